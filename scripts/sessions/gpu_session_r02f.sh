#!/bin/bash
# Round-2 session f (policy 3 + batch bounds): full GPU parity suite, smoke,
# bench (both arms), launch list of the bench command, ncu --set full of the
# bench kernel at 2^25 and of the C1 / C3 / C4 config kernels.
set -u
OUT=${OUT:-gpurun_out/r02f}
mkdir -p "$OUT"
nproc > "$OUT/nproc.txt"; lscpu >> "$OUT/nproc.txt" 2>/dev/null
timeout 1800 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 300 python scripts/c4_check.py > "$OUT/c4_check.jsonl" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread \
    --clock-control none -c 60 --csv --log-file "$OUT/ncu_launches_p2_2e25.csv" \
    python bench.py --points 33554432 --steps 3 --warmup 3 --no-e2e --no-cpu --no-configs > "$OUT/ncu_launches_bench.out" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tlk_flat -s 2 -c 1 \
    -o "$OUT/ncu_full_p2_2e25" python scripts/ncu_target.py p2 25 > "$OUT/ncu_full.out" 2>&1
for c in c1 c3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tlk_ -s 2 -c 1 \
      -o "$OUT/ncu_full_$c" python scripts/ncu_configs.py $c > "$OUT/ncu_full_$c.out" 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tlk_batch -s 2 -c 1 \
    -o "$OUT/ncu_full_c4_p2" python scripts/ncu_configs.py c4_p2 > "$OUT/ncu_full_c4_p2.out" 2>&1
