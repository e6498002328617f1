#!/bin/bash
# independent statement parts (Variant.split) A/B: P2 and Maxwell, 2^18 .. 2^28
OUT=${OUT:-gpurun_out/splitab}
mkdir -p $OUT
export PYTHONPATH=$PWD
SPLITS=262144,2097152,16777216,67108864 ROUNDS=7 K=10 timeout 900 python scripts/tune_ab.py > $OUT/tune_ab_split.jsonl 2> $OUT/tune_ab_split.err
SPLITS=268435456 ROUNDS=7 K=3 timeout 900 python scripts/tune_ab.py >> $OUT/tune_ab_split.jsonl 2>> $OUT/tune_ab_split.err
echo done > $OUT/DONE
