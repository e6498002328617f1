#!/bin/bash
# Round-2 tuning session: warp-specialised staged
# entry parity, P2 knobs + streaming ceilings at 2^28, component-pitch
# padding, C1 64^3 / C3 128^3 launch shapes.
# Usage: OUT=gpurun_out/x bash scripts/sessions/gpu_tune_r02.sh
set -u
OUT=${OUT:-gpurun_out/tune_r02}
mkdir -p "$OUT"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/clocks_before.txt" 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -rs -p no:cacheprovider \
    -k "staged or codegen_variant" > "$OUT/pytest_ws.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_ws.log"
timeout 1200 python scripts/tune_p2b.py $((1 << 28)) 10 > "$OUT/tune_p2b.jsonl" 2> "$OUT/tune_p2b.err"
PADS=0,32,256,264,1040 SHAPES=policy,t128_r34 timeout 900 python scripts/tune_pitch.py \
    $((1 << 28)) 8 > "$OUT/tune_pitch.jsonl" 2> "$OUT/tune_pitch.err"
timeout 900 python scripts/tune_small2.py > "$OUT/tune_small2.jsonl" 2> "$OUT/tune_small2.err"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/clocks_after.txt" 2>&1
