#!/bin/bash
# statement parts with a tiny part (Gamma + a 2/6/18-array copy): split vs fused
OUT=${OUT:-gpurun_out/splittiny}
mkdir -p $OUT
export PYTHONPATH=$PWD
CASES="$(cat scripts/sessions/split_tiny_cases.json)" ROUNDS=7 K=10 timeout 900 python scripts/tune_ab.py > $OUT/tune_ab_split_tiny.jsonl 2> $OUT/err.txt
echo done > $OUT/DONE
