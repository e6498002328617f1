#!/bin/bash
# block size of the split (policy) P2 / Maxwell kernels, 2^21 .. 2^28
OUT=${OUT:-gpurun_out/splitthr}
mkdir -p $OUT
export PYTHONPATH=$PWD
SPLIT_THREADS=2097152,16777216,67108864 ROUNDS=7 K=10 timeout 900 python scripts/tune_ab.py > $OUT/tune_ab_split_threads.jsonl 2> $OUT/tune_ab_split_threads.err
SPLIT_THREADS=268435456 ROUNDS=5 K=3 timeout 900 python scripts/tune_ab.py >> $OUT/tune_ab_split_threads.jsonl 2>> $OUT/tune_ab_split_threads.err
echo done > $OUT/DONE
