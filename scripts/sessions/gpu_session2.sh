#!/bin/bash
TAG=${1:-r01b}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --sweep > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 python scripts/compare_reference_design.py > $OUT/refdesign.jsonl 2> $OUT/refdesign.err
timeout 900 python bench.py --no-cpu > $OUT/bench.json 2> $OUT/bench.err
echo done > $OUT/DONE
