"""Mid/small-N variant tuning (graph replay, L2 flushed): C1 64^3, C3 128^3,
P2 2^21, C4 batch 512 x 16^3 under launch/codegen variants.
Usage: PYTHONPATH=. python scripts/tune_small.py"""

import json
import os
import subprocess
import sys

VARIANTS = {
    "policy": {},
    "waves1": {"TLK_WAVES": "1"},
    "waves2": {"TLK_WAVES": "2"},
    "waves4": {"TLK_WAVES": "4"},
    "waves8": {"TLK_WAVES": "8"},
    "vec1": {"TLK_VEC": "1"},
    "vec2": {"TLK_VEC": "2"},
    "t128": {"TLK_THREADS": "128"},
    "t512": {"TLK_THREADS": "512"},
    "vec1_t128_w8": {"TLK_VEC": "1", "TLK_THREADS": "128", "TLK_WAVES": "8"},
}

CHILD = r"""
import json, statistics, torch
from paper_1804_10120_b200 import bench as tb, eval_program, eval_batch, capture_graph
from paper_1804_10120_b200.evaluator import plan_for
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
def timed(fn, reps=31):
    g = capture_graph(fn)
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts[1:])
for name, n in (("c1_dtg", 64**3), ("c1_dtg", 2**21), ("c3_christoffel", 128**3),
                ("p2", 2**21), ("c2_maxwell", 10**6)):
    prog, vs = tb.load(tb.PROGRAMS[name])
    targets = {v.stmt.lhs.field for v in vs}
    env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
    for f in env.values():
        f.resize(n)
        if f.name not in targets:
            f.data.uniform_()
    plan = plan_for(vs, env)
    t = timed(lambda: eval_program(vs, env))
    print(json.dumps({"program": name, "n": n, "us": t * 1e6,
                      "gbs": plan.bytes_per_point * n / t / 1e9,
                      "variant": plan.variant.tag()}), flush=True)
prog, vs = tb.load(tb.P2)
envs = []
for d in range(512):
    e = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED + d)
    for f in e.values():
        f.resize(16**3)
        if f.name not in ("Gamma", "dtg"):
            f.data.uniform_()
    envs.append(e)
plan = plan_for(vs, envs[0])
t = timed(lambda: eval_batch(vs, envs))
print(json.dumps({"program": "c4_batch", "n": 512 * 16**3, "us": t * 1e6,
                  "gbs": plan.bytes_per_point * 512 * 16**3 / t / 1e9,
                  "variant": plan.variant.tag()}), flush=True)
"""

for vname, knobs in VARIANTS.items():
    env = dict(os.environ, **knobs)
    res = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                         timeout=600)
    if res.returncode != 0:
        print(json.dumps({"knobs": vname, "error": res.stderr[-800:]}), flush=True)
        continue
    for line in res.stdout.splitlines():
        d = json.loads(line)
        d["knobs"] = vname
        print(json.dumps(d), flush=True)
