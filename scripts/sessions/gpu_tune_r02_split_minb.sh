#!/bin/bash
# register caps for the split P2 kernel (89 registers uncapped)
OUT=${OUT:-gpurun_out/minb}
mkdir -p $OUT
export PYTHONPATH=$PWD
SPLIT_MINB=16777216,67108864 ROUNDS=7 K=10 timeout 900 python scripts/tune_ab.py > $OUT/tune_ab_split_minb.jsonl 2> $OUT/err.txt
SPLIT_MINB=268435456 ROUNDS=5 K=3 timeout 900 python scripts/tune_ab.py >> $OUT/tune_ab_split_minb.jsonl 2>> $OUT/err.txt
echo done > $OUT/DONE
