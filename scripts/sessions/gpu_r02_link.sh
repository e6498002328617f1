#!/bin/bash
# bench contract GPU test + a full bench run with the e2e link floor
OUT=${OUT:-gpurun_out/link}
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_bench_contract.py -q -m gpu -p no:cacheprovider > $OUT/pytest_bench_contract.log 2>&1
echo "rc=$?" >> $OUT/pytest_bench_contract.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo done > $OUT/DONE
