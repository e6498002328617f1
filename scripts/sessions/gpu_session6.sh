#!/bin/bash
# re-validation of a fresh build + small-N timing methodology study + cold
# per-kernel device times (ncu launch list) of the small configs
TAG=${1:-r01i}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
nvidia-smi > $OUT/nvidia_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python scripts/small_latency.py > $OUT/small_latency.jsonl 2> $OUT/small_latency.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tlk_ --csv \
  --log-file $OUT/ncu_launches_small.csv python scripts/small_configs.py > $OUT/ncu_small.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo done > $OUT/DONE
