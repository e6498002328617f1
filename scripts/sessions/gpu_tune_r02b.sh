#!/bin/bash
# Round-2 tuning session b: warp-specialised vs barrier ring per program/size,
# streaming ceilings, and ncu kernel durations of the C1 64^3 launch shapes.
set -u
OUT=${OUT:-gpurun_out/tune_r02b}
mkdir -p "$OUT"
timeout 900 python scripts/tune_ws.py > "$OUT/tune_ws.jsonl" 2> "$OUT/tune_ws.err"
timeout 600 python scripts/stream_probe.py > "$OUT/stream_probe.jsonl" 2> "$OUT/stream_probe.err"
NCU=1 ONLY_C1=1 timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:tlk_ --csv --log-file "$OUT/ncu_c1_shapes.csv" \
    python scripts/tune_small2.py > "$OUT/ncu_c1_shapes.out" 2>&1
