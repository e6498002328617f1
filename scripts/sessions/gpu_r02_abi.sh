#!/bin/bash
# C-ABI default launch parity + harness tests after the symbol-visibility change
OUT=${OUT:-gpurun_out/abi}
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -q -rs -p no:cacheprovider -k "default_launch or harness or library or smoke or multirank" > $OUT/pytest_abi.log 2>&1
echo "rc=$?" >> $OUT/pytest_abi.log
echo done > $OUT/DONE
