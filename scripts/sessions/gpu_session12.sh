#!/bin/bash
# staged share of the read slots: per-program sweep + P2 bench at 2^28
TAG=${1:-r01s}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1500 python scripts/tune_stage.py frac > $OUT/tune_stage_frac.jsonl 2> $OUT/tune_stage_frac.err
for i in 1 2; do
  for cfg in "0 128 0" "3 128 26" "3 128 28" "3 128 30" "3 128 32" "3 128 34" "4 128 26" "4 128 28"; do
    set -- $cfg
    TLK_STAGE=$1 TLK_STAGE_THREADS=$2 TLK_STAGE_READS=$3 timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 20 > $OUT/bench_g$1x$2r$3_$i.json 2>> $OUT/bench_ab.err
  done
done
echo done > $OUT/DONE
