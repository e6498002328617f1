#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over the
# warp-specialised staged entry (policy 2): full and partial rings, ring
# wrap-around, ragged tails, 2- and 3-deep rings, and the contraction-class
# 128-point ring, all through the parity tests
OUT=${OUT:-gpurun_out/sanitize_ws}
mkdir -p $OUT
export PYTHONPATH=$PWD
SEL="(tma_staged_entry_bitwise and (2-0-1 or 3-5-1) and (p2 or c3_christoffel or c1_dtg)) or (codegen_variant and stage_ws and (c4_p2 or suite_contract1 or c1_dtg))"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all python -m pytest tests/test_gpu_parity.py -q -x \
    -k "$SEL" > $OUT/sanitizer_ws_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitizer_ws_$tool.log
done
