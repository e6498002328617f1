#!/bin/bash
# ncu --set full of the final bench kernel (statement parts, fused tlk_point beside)
# at 2^25 + the new protocol GPU test
OUT=${OUT:-gpurun_out/ncufinal}
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_make_env.py -q -m gpu -p no:cacheprovider > $OUT/pytest_protocol.log 2>&1
echo "rc=$?" >> $OUT/pytest_protocol.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tlk_flat -s 2 -c 1 \
    -o "$OUT/ncu_full_p2_2e25" python scripts/ncu_target.py p2 25 > "$OUT/ncu_full.out" 2>&1
echo done > $OUT/DONE
