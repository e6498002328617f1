#!/bin/bash
# e2e pipeline stage size sweep (TLB_HOST_SLAB points per H2D/kernel/D2H stage)
OUT=${OUT:-gpurun_out/hostslab}
mkdir -p $OUT
export PYTHONPATH=$PWD
for sl in 0 524288 1048576 2097152 4194304 0; do
  TLB_HOST_SLAB=$sl timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 3 --no-cpu --no-configs > $OUT/bench_slab_$sl.json 2> $OUT/bench_slab_$sl.err
  python -c "import json,sys;d=json.loads(open('$OUT/bench_slab_$sl.json').read().strip().splitlines()[-1]);print($sl, d['e2e']['s_per_step'], d['e2e']['link'])" >> $OUT/summary.txt
done
echo done > $OUT/DONE
