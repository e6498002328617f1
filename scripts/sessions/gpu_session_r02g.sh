#!/bin/bash
# Round-2 session g: e2e host-slab size, the unchanged tl_harness on C3
# 128^3 (pageable / registered / pinned), compute-sanitizer over the policy-3
# one-shot launches (incl. the small-launch block shrink).
set -u
OUT=${OUT:-gpurun_out/r02g}
mkdir -p "$OUT"
for slab in 16777216 33554432 67108864; do
  timeout 900 python bench.py --no-configs --no-cpu --steps 5 --warmup 3 --e2e-steps 3 \
      --e2e-slab $slab > "$OUT/bench_e2e_slab_$slab.json" 2> "$OUT/bench_e2e_slab_$slab.err"
done
timeout 900 python scripts/harness_timing.py > "$OUT/harness_timing.jsonl" 2> "$OUT/harness_timing.err"
export PYTHONPATH=$PWD
SEL="one_shot_block_shrink or (fused_program_matches and (c4_p2 or c1_dtg or suite_outer3 or suite_assign3)) or (suite_statements and (add1 or outer2 or contract1))"
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all python -m pytest tests/test_gpu_parity.py -q -x \
    -k "$SEL" > "$OUT/sanitizer_policy3_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitizer_policy3_$tool.log"
done
