#!/bin/bash
# ncu --set full of every BASELINE config's kernel under the final policy; new parity tests
TAG=${1:-r01za}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "without_reads or size_classes" > $OUT/pytest_new.log 2>&1
for cfg in c1 c3 c2 c4_p2 c4_p3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tlk_ -s 1 -c 1 \
    -o $OUT/prof_$cfg python scripts/ncu_configs.py $cfg > $OUT/ncu_$cfg.log 2>&1
done
echo done > $OUT/DONE
