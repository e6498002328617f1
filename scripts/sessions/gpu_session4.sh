#!/bin/bash
TAG=${1:-r01g}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# ncu: the light-kernel variant (Maxwell, 1 point/thread) and the C4 batch kernel
cat > /tmp/ncu_cfg.py <<'PY'
import sys, torch
from paper_1804_10120_b200 import bench as tb, eval_program, eval_batch
which = sys.argv[1]
if which == "maxwell":
    prog, vs = tb.load(tb.MAXWELL)
    env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
    tg = {v.stmt.lhs.field for v in vs}
    for f in env.values():
        f.resize(10**8)
        if f.name not in tg: f.data.uniform_()
    for _ in range(3): eval_program(vs, env)
else:
    prog, vs = tb.load(tb.P2)
    envs = []
    for d in range(512):
        e = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED + d)
        for f in e.values():
            f.resize(16**3)
            if f.name not in ("Gamma", "dtg"): f.data.uniform_()
        envs.append(e)
    for _ in range(3): eval_batch(vs, envs)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tlk_ -s 1 -c 1 -o $OUT/prof_maxwell python /tmp/ncu_cfg.py maxwell > $OUT/ncu_maxwell.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tlk_batch -s 1 -c 1 -o $OUT/prof_c4batch python /tmp/ncu_cfg.py c4 > $OUT/ncu_c4.log 2>&1
echo done > $OUT/DONE
