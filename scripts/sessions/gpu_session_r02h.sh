#!/bin/bash
# Round-2 session h: pinned bounce ring for pageable host fields — parity of
# every host-staged / harness path, the harness timing on C3 128^3, e2e.
set -u
OUT=${OUT:-gpurun_out/r02h}
mkdir -p "$OUT"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_harness_b200.py tests/test_cli.py -m gpu -q -rs -p no:cacheprovider \
    -k "host or harness or bounce or eval or staged_through" > "$OUT/pytest_host.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_host.log"
timeout 900 python scripts/harness_timing.py > "$OUT/harness_timing.jsonl" 2> "$OUT/harness_timing.err"
timeout 900 python bench.py --no-configs --no-cpu --steps 5 --warmup 3 --e2e-steps 3 > "$OUT/bench_e2e.json" 2> "$OUT/bench_e2e.err"
