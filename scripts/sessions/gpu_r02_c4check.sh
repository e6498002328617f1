#!/bin/bash
# batch / split parity subset + C4 timing after the fused-tlk_point fix
OUT=${OUT:-gpurun_out/c4fix}
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider -k "batch or c4 or parts or split or fuzz or program" > $OUT/pytest_subset.log 2>&1
echo "rc=$?" >> $OUT/pytest_subset.log
timeout 300 python scripts/c4_check.py > $OUT/c4_check.jsonl 2>&1
echo done > $OUT/DONE
