#!/bin/bash
# C1 64^3 vs TMA bulk reads of its inputs and its TMA-staged entry (events + ncu)
OUT=${OUT:-gpurun_out/smalltma}
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 600 python scripts/small_ceiling_tma.py > $OUT/small_ceiling_tma.jsonl 2> $OUT/err.txt
REPS=3 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:'tlk_|probe_' --csv --log-file $OUT/ncu_small_tma.csv \
  python scripts/small_ceiling_tma.py > $OUT/ncu_run.log 2>&1
echo done > $OUT/DONE
