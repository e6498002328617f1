#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), ncu launch list + full capture.
# Usage (under gpurun): bash scripts/sessions/gpu_session.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/nvidia_smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | head -20 >> $OUT/nproc.txt
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --points 33554432 --steps 3 --warmup 1 --no-e2e --no-cpu --no-configs > $OUT/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tlk_flat -s 1 -c 1 \
    -o $OUT/prof_p2 python bench.py --points 33554432 --steps 2 --warmup 1 --no-e2e --no-cpu --no-configs > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
