#!/bin/bash
# final soak under the default policy (statement parts with the size guard)
OUT=${OUT:-gpurun_out/soakfinal}
mkdir -p $OUT
export PYTHONPATH=$PWD:$PWD/tests
timeout 1200 python scripts/soak.py --mode default --seconds 900 --seed 23 > $OUT/soak_default_final.json 2> $OUT/soak.err
echo done > $OUT/DONE
