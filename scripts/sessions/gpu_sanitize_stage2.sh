#!/bin/bash
# compute-sanitizer over the staged batch entry (warp-specialised, prefetching
# producer) and the partially staged flat entry
TAG=${1:-r01zj}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all python -m pytest tests/test_gpu_parity.py -q -x \
    -k "(tma_staged_batch_entry_bitwise and 128-7 and c4_p2) or (tma_staged_entry_bitwise and 3-5 and p2)" > $OUT/sanitizer_stage2_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitizer_stage2_$tool.log
done
echo done > $OUT/DONE
