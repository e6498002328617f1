#!/bin/bash
# Round-2 session c: full GPU parity suite, smoke, bench (both arms), the
# streaming-ceiling probes, launch list + one ncu --set full of the bench
# kernel (P2, current policy variant) at 2^25 points.
set -u
OUT=${OUT:-gpurun_out/r02c}
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia_smi.txt" 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 600 python scripts/stream_probe.py > "$OUT/stream_probe.jsonl" 2> "$OUT/stream_probe.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file "$OUT/ncu_launches_p2_2e25.csv" python bench.py --points 33554432 --steps 3 --warmup 3 \
    --no-e2e --no-cpu --no-configs > "$OUT/ncu_launches_bench.out" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tlk_stage -s 2 -c 1 \
    -o "$OUT/ncu_full_p2_2e25" python scripts/ncu_target.py p2 25 > "$OUT/ncu_full.out" 2>&1
