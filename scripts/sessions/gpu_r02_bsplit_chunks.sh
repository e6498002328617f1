#!/bin/bash
# C4 P2: batch entry over statement parts with several chunks per block
OUT=${OUT:-gpurun_out/bschunks}
mkdir -p $OUT
export PYTHONPATH=$PWD
for r in 1 2; do
  timeout 300 python scripts/c4_check.py > /dev/null 2>&1  # warm the box
  timeout 300 python scripts/c4_check.py >> $OUT/fused_c1.jsonl 2>&1
  TLB_BATCH_CHUNKS=2 timeout 300 python scripts/c4_check.py >> $OUT/fused_c2.jsonl 2>&1
  TLK_BATCH_SPLIT=1 TLB_BATCH_CHUNKS=2 timeout 300 python scripts/c4_check.py >> $OUT/split_c2.jsonl 2>&1
  TLK_BATCH_SPLIT=1 TLB_BATCH_CHUNKS=4 timeout 300 python scripts/c4_check.py >> $OUT/split_c4.jsonl 2>&1
  TLK_BATCH_SPLIT=1 TLB_BATCH_CHUNKS=8 timeout 300 python scripts/c4_check.py >> $OUT/split_c8.jsonl 2>&1
done
echo done > $OUT/DONE
