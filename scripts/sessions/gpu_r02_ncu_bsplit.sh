#!/bin/bash
# ncu --set full of C4 P2's batch entry: fused body vs statement-part rows
OUT=${OUT:-gpurun_out/ncubs}
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tlk_batch -s 2 -c 1 \
    -o "$OUT/ncu_c4_p2_fused" python scripts/ncu_configs.py c4_p2 > "$OUT/fused.out" 2>&1
TLK_BATCH_SPLIT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tlk_batch -s 2 -c 1 \
    -o "$OUT/ncu_c4_p2_split" python scripts/ncu_configs.py c4_p2 > "$OUT/split.out" 2>&1
echo done > $OUT/DONE
