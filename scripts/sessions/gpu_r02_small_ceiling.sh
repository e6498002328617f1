#!/bin/bash
# small-size stream-mix ceilings beside C1 64^3 / C3 128^3 (scripts/small_ceiling.py)
OUT=${OUT:-gpurun_out/ceil}
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 600 python scripts/small_ceiling.py > $OUT/small_ceiling.jsonl 2> $OUT/small_ceiling.err
REPS=3 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:'tlk_|probe_' --csv --log-file $OUT/ncu_small_ceiling.csv \
  python scripts/small_ceiling.py > $OUT/ncu_run.log 2>&1
echo done > $OUT/DONE
