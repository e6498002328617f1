#!/bin/bash
# Statement parts (Variant.split) adopted by policy 3: full GPU parity suite,
# smoke, bench (both arms), launch list of the bench command, ncu --set full
# of the (split) bench kernel at 2^25 and of C2 Maxwell at 10^8-class size.
set -u
OUT=${OUT:-gpurun_out/r02s}
mkdir -p "$OUT"
export PYTHONPATH=$PWD
timeout 2400 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 900 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread \
    --clock-control none -c 60 --csv --log-file "$OUT/ncu_launches_p2_2e25.csv" \
    python bench.py --points 33554432 --steps 3 --warmup 3 --no-e2e --no-cpu --no-configs > "$OUT/ncu_launches_bench.out" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tlk_flat -s 2 -c 1 \
    -o "$OUT/ncu_full_p2_2e25" python scripts/ncu_target.py p2 25 > "$OUT/ncu_full.out" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tlk_flat -s 2 -c 1 \
    -o "$OUT/ncu_full_c2_2e26" python scripts/ncu_target.py c2_maxwell 26 > "$OUT/ncu_full_c2.out" 2>&1
echo done > "$OUT/DONE"
