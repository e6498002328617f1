#!/bin/bash
# compute-sanitizer memcheck + racecheck over the output-group kernels
# (Variant.vn: non-inlined group functions, __grid_constant__ parameter
# blocks), the grouped batch entry, and the host-staged bounce ring / concurrent
# host-staged threads (pageable and pinned host fields)
OUT=${OUT:-gpurun_out/sanitize_groups}
mkdir -p $OUT
export PYTHONPATH=$PWD
SEL="output_groups_are_bit_exact or grouped_program_in_a_multi_domain_batch"
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all python -m pytest tests/test_gpu_parity.py -q -x \
    -k "$SEL" > $OUT/sanitizer_groups_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitizer_groups_$tool.log
done
timeout 1500 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests -q -x -m gpu \
  -k "pageable or concurrent_host or host_staged" > $OUT/sanitizer_host_memcheck.log 2>&1
echo "rc=$?" >> $OUT/sanitizer_host_memcheck.log
echo done > $OUT/DONE
