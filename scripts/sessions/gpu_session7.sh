#!/bin/bash
# size-class dispatch: parity suite, small-N timings, bench line with configs
TAG=${1:-r01k}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python scripts/small_latency.py > $OUT/small_latency.jsonl 2> $OUT/small_latency.err
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --sweep > $OUT/sweep.jsonl 2> $OUT/sweep.err
echo done > $OUT/DONE
