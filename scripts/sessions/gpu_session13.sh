#!/bin/bash
# partially staged policy: parity suite, smoke, bench (both arms), sweep, small-N, ncu of the bench kernel
TAG=${1:-r01final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 python bench.py --sweep > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 900 python scripts/tune_smalln.py > $OUT/tune_smalln.jsonl 2> $OUT/tune_smalln.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/ncu_launches_p2_2e25.csv python bench.py --points 33554432 --steps 3 --warmup 1 --no-e2e --no-cpu --no-configs > $OUT/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tlk_ -s 1 -c 1 \
  -o $OUT/prof_p2 python bench.py --points 33554432 --steps 2 --warmup 1 --no-e2e --no-cpu --no-configs > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
