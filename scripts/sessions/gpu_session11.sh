#!/bin/bash
# P2 at 2^28: partially staged rings (some reads through TMA, the rest direct)
TAG=${1:-r01r}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tma_staged or stage" > $OUT/pytest_stage.log 2>&1
for i in 1 2; do
  for cfg in "0 128 0" "3 128 16" "3 128 24" "3 128 30" "3 128 36" "4 128 24" "2 256 24" "3 256 12" "2 128 40"; do
    set -- $cfg
    TLK_STAGE=$1 TLK_STAGE_THREADS=$2 TLK_STAGE_READS=$3 timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 20 > $OUT/bench_g$1x$2r$3_$i.json 2>> $OUT/bench_ab.err
  done
done
echo done > $OUT/DONE
