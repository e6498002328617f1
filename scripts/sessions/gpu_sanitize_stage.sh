#!/bin/bash
# compute-sanitizer over the TMA-staged entry (memcheck, racecheck, synccheck)
TAG=${1:-r01q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all python -m pytest tests/test_gpu_parity.py -q -x \
    -k "tma_staged_entry_bitwise and (c3_christoffel or p3) and 2-" > $OUT/sanitizer_stage_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitizer_stage_$tool.log
done
echo done > $OUT/DONE
