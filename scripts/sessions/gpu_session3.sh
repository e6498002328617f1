#!/bin/bash
TAG=${1:-r01e}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
   bench.py --gpus 2 --dist-backend gloo --same-device --points 67108864 --steps 10 --warmup 3 --e2e-steps 1 \
   > $OUT/bench_2rank_samegpu.json 2> $OUT/bench_2rank.err
for w in 0 4 16; do
  TLB_BATCH_WAVES=$w timeout 300 python -c "
import json, statistics, torch
from paper_1804_10120_b200 import bench as tb, eval_batch, capture_graph
from paper_1804_10120_b200.evaluator import plan_for
prog, vs = tb.load(tb.P2)
envs = []
for d in range(512):
    e = tb.make_env(prog, '__none__', 0, tb.DEFAULT_SEED + d)
    for f in e.values():
        f.resize(16**3)
        if f.name not in ('Gamma', 'dtg'): f.data.uniform_()
    envs.append(e)
g = capture_graph(lambda: eval_batch(vs, envs))
flush = torch.empty(1 << 28, dtype=torch.uint8, device='cuda')
ts = []
for _ in range(31):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
print(json.dumps({'batch_waves': $w, 'us': statistics.median(ts[1:]) * 1e3}))
" >> $OUT/batch_waves.jsonl 2>> $OUT/batch_waves.err
done
echo done > $OUT/DONE
