#!/bin/bash
# batch entry over statement parts (TLK_BATCH_SPLIT=1) vs the fused batch body:
# C4 timing alternated 3x, and the batch parity subset under the split batch entry
OUT=${OUT:-gpurun_out/bsplit}
mkdir -p $OUT
export PYTHONPATH=$PWD
for r in 1 2 3; do
  timeout 300 python scripts/c4_check.py >> $OUT/c4_fused_body.jsonl 2>&1
  TLK_BATCH_SPLIT=1 timeout 300 python scripts/c4_check.py >> $OUT/c4_batch_split.jsonl 2>&1
done
TLK_BATCH_SPLIT=1 timeout 1200 python -m pytest tests -m gpu -q -rs -p no:cacheprovider -k "batch or c4" > $OUT/pytest_batch_split.log 2>&1
echo "rc=$?" >> $OUT/pytest_batch_split.log
echo done > $OUT/DONE
