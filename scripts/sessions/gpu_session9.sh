#!/bin/bash
# P2 at 2^28 (the bench line): plain entry vs staged ring shapes, eager launches
TAG=${1:-r01o}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
for i in 1 2; do
  for cfg in "0 128" "2 128" "2 256" "3 128" "3 64" "4 64" "6 64" "2 192"; do
    set -- $cfg
    TLK_STAGE=$1 TLK_STAGE_THREADS=$2 timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 20 > $OUT/bench_g$1x$2_$i.json 2>> $OUT/bench_ab.err
  done
done
echo done > $OUT/DONE
