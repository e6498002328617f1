#!/bin/bash
# light-kernel code (hoisted ld.global.cs) for P2's light statement part
OUT=${OUT:-gpurun_out/partlight}
mkdir -p $OUT
export PYTHONPATH=$PWD
CASES="$(cat scripts/sessions/part_light_cases.json)" ROUNDS=7 K=10 timeout 900 python scripts/tune_ab.py > $OUT/tune_ab_part_light.jsonl 2> $OUT/err.txt
CASES="$(cat scripts/sessions/part_light_cases_2e28.json)" ROUNDS=7 K=3 timeout 900 python scripts/tune_ab.py >> $OUT/tune_ab_part_light.jsonl 2>> $OUT/err.txt
echo done > $OUT/DONE
