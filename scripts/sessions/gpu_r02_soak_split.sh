#!/bin/bash
# soak under the default policy (statement parts included): random programs x sizes
OUT=${OUT:-gpurun_out/soaksplit}
mkdir -p $OUT
export PYTHONPATH=$PWD:$PWD/tests
timeout 900 python scripts/soak.py --mode default --seconds 480 --seed 11 > $OUT/soak_default_split.json 2> $OUT/soak.err
echo done > $OUT/DONE
