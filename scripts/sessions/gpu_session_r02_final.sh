#!/bin/bash
# Round-2 final record: memcheck over the statement-part kernels, then exactly
# what the driver runs (pytest -m gpu, smoke, bench both arms), the launch
# list of the bench command
set -u
OUT=${OUT:-gpurun_out/r02final}
mkdir -p "$OUT"
export PYTHONPATH=$PWD
timeout 900 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_gpu_parity.py -q -x \
  -k "statement_parts or fuzzed or pageable" > "$OUT/sanitizer_parts_memcheck.log" 2>&1
echo "rc=$?" >> "$OUT/sanitizer_parts_memcheck.log"
( time timeout 2400 python -m pytest tests -q -rs -m gpu -p no:cacheprovider ) > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
( time timeout 1200 python bench.py ) > "$OUT/bench.json" 2> "$OUT/bench.err"
( time timeout 900 python bench.py --impl reference ) > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread \
    --clock-control none -c 60 --csv --log-file "$OUT/ncu_launches_p2_2e25.csv" \
    python bench.py --points 33554432 --steps 3 --warmup 3 --no-e2e --no-cpu --no-configs > "$OUT/ncu_launches_bench.out" 2>&1
nvidia-smi > "$OUT/nvidia_smi.txt" 2>&1; free -g >> "$OUT/nvidia_smi.txt" 2>&1
echo done > "$OUT/DONE"
