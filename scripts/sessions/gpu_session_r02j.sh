#!/bin/bash
# Round-2 rehearsal of the driver's round-end commands (final policy):
# pytest -m gpu, smoke, bench (ours + reference arm), each wall-timed.
set -u
OUT=${OUT:-gpurun_out/r02j}
mkdir -p "$OUT"
s=$(date +%s); timeout 1800 python -m pytest tests -x -q -m gpu -rs -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$? wall_s=$(( $(date +%s) - s ))" >> "$OUT/pytest_gpu.log"
s=$(date +%s); timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke rc=$? wall_s=$(( $(date +%s) - s ))" >> "$OUT/smoke.log"
s=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench rc=$? wall_s=$(( $(date +%s) - s ))" >> "$OUT/bench.err"
s=$(date +%s); timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
echo "ref rc=$? wall_s=$(( $(date +%s) - s ))" >> "$OUT/bench_ref.err"
