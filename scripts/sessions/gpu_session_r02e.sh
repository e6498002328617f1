#!/bin/bash
# Round-2 session e: policy 3 (one-shot flat grids) — full GPU parity suite,
# smoke, bench, and the interleaved policy-2-vs-3 A/B over every program.
set -u
OUT=${OUT:-gpurun_out/r02e}
mkdir -p "$OUT"
timeout 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
POLICY_AB=1000,100000,262144,2097152,16777216,67108864 POLICY_PAIR=2,3 ROUNDS=5 timeout 2400 \
    python scripts/tune_ab.py > "$OUT/tune_ab_policy2_vs_3.jsonl" 2> "$OUT/tune_ab.err"
