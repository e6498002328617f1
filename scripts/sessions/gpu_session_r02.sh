#!/bin/bash
# Round-2 GPU session: parity suite, smoke, both bench arms, launch list and
# one ncu --set full capture of the bench kernel.  Usage: OUT=gpurun_out/x bash scripts/sessions/gpu_session_r02.sh
set -u
OUT=${OUT:-gpurun_out/r02}
mkdir -p "$OUT"
nproc > "$OUT/nproc.txt"; lscpu >> "$OUT/nproc.txt" 2>/dev/null; free -g >> "$OUT/nproc.txt"
nvidia-smi > "$OUT/nvidia_smi.txt" 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -rs -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file "$OUT/ncu_launches_p2_2e25.csv" python bench.py --points 33554432 --steps 3 --warmup 3 \
      --no-e2e --no-cpu --no-configs > "$OUT/ncu_launches_bench.out" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tlk_stage -s 2 -c 1 \
      -o "$OUT/ncu_full_p2_2e25" python scripts/ncu_target.py p2 25 > "$OUT/ncu_full.out" 2>&1
fi
