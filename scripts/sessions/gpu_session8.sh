#!/bin/bash
# staged (TMA) policy: full parity suite, policy vs no-stage timings, bench A/B
TAG=${1:-r01n}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python scripts/tune_stage.py > $OUT/tune_stage.jsonl 2> $OUT/tune_stage.err
for i in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --no-configs > $OUT/bench_policy_$i.json 2>> $OUT/bench_ab.err
  TLK_STAGE=0 timeout 300 python bench.py --no-e2e --no-cpu --no-configs > $OUT/bench_nostage_$i.json 2>> $OUT/bench_ab.err
done
echo done > $OUT/DONE
