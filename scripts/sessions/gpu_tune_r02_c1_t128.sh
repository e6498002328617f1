#!/bin/bash
# does the dt g part (C1's statement) lose by running in P2's 128-thread blocks?
OUT=${OUT:-gpurun_out/c1t128}
mkdir -p $OUT
export PYTHONPATH=$PWD
CASES="$(cat scripts/sessions/c1_t128_cases.json)" ROUNDS=7 K=10 timeout 900 python scripts/tune_ab.py > $OUT/tune_ab_c1_t128.jsonl 2> $OUT/err.txt
echo done > $OUT/DONE
