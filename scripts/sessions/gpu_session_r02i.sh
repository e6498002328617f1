#!/bin/bash
# Round-2 session i: one-shot stream-mix ceilings; the paper's GPU design vs
# the policy-3 kernels on the same B200.
set -u
OUT=${OUT:-gpurun_out/r02i}
mkdir -p "$OUT"
timeout 600 python scripts/stream_probe.py > "$OUT/stream_probe.jsonl" 2> "$OUT/stream_probe.err"
PYTHONPATH=$PWD timeout 900 python scripts/compare_reference_design.py > "$OUT/reference_design_comparator.jsonl" 2> "$OUT/compare.err"
