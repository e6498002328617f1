#!/bin/bash
# policy with the staged entry: parity suite, smoke, bench line, sweep, ncu of staged kernels
TAG=${1:-r01p}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 python bench.py --sweep > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 python scripts/small_latency.py > $OUT/small_latency.jsonl 2> $OUT/small_latency.err
for pc in "p3 24" "c3_christoffel 24" "c2_maxwell 24"; do
  set -- $pc
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tlk_stage -s 1 -c 1 \
    -o $OUT/prof_$1 python scripts/ncu_target.py $1 $2 > $OUT/ncu_$1.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tlk_ --csv \
  --log-file $OUT/ncu_launches_small.csv python scripts/small_configs.py > $OUT/ncu_small.log 2>&1
echo done > $OUT/DONE
