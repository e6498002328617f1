#!/bin/bash
# harness bindings load build_shared's precompiled cubins (no NVRTC in the
# harness process): harness GPU tests + whole-process harness timing on C3 128^3
OUT=${OUT:-gpurun_out/hcache}
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -q -rs -p no:cacheprovider -k "harness or default_launch" > $OUT/pytest_harness.log 2>&1
echo "rc=$?" >> $OUT/pytest_harness.log
timeout 900 python scripts/harness_timing.py > $OUT/harness_timing.jsonl 2> $OUT/harness_timing.err
echo done > $OUT/DONE
