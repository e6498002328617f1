"""The reference's 14-statement suite (bench.builtin_suite, reference
bench.py:98-199) plus C1-C3/P2/P3 at 2^22 points: default policy against
the plain entries (TLK_STAGE=0), one graph replay after a clean L2 flush and
20 back-to-back launches — a check that the staging policy generalises.
Usage: PYTHONPATH=. python scripts/tune_suite.py > tune_suite.jsonl"""

import json
import os
import subprocess
import sys

CHILD = r"""
import json, statistics, torch
from paper_1804_10120_b200 import bench as tb, eval_program, capture_graph
from paper_1804_10120_b200.evaluator import plan_for
wbuf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(1 << 25, dtype=torch.float64, device="cuda")
def single(fn, reps=11):
    g = capture_graph(fn); ts = []
    for _ in range(reps):
        wbuf.zero_(); rbuf.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts[1:])
def b2b(fn, k=20):
    g = capture_graph(lambda: [fn() for _ in range(k)]); ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / k)
    return statistics.median(ts[1:])
n = 1 << 22
items = [(e.name, e.source) for e in tb.builtin_suite()] + [(k, v) for k, v in tb.PROGRAMS.items()]
for name, text in items:
    prog, vs = tb.load(text)
    targets = {v.stmt.lhs.field for v in vs}
    env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
    for f in env.values():
        f.resize(n)
        if f.name not in targets:
            f.data.uniform_()
    plan = plan_for(vs, env)
    fn = lambda: eval_program(vs, env)
    ts, tb2 = single(fn), b2b(fn)
    gb = plan.bytes_per_point * n / 1e9
    print(json.dumps({"program": name, "n": n, "reads": plan.reads, "writes": plan.writes,
                      "us_single_clean": ts * 1e6, "us_b2b": tb2 * 1e6,
                      "gbs_single": gb / ts, "gbs_b2b": gb / tb2,
                      "variant": plan.variant.tag()}), flush=True)
    del env
    torch.cuda.empty_cache()
"""

for vname, knobs in (("policy", {}), ("plain", {"TLK_STAGE": "0"})):
    env = dict(os.environ, **knobs)
    res = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                         timeout=1500)
    if res.returncode != 0:
        print(json.dumps({"knobs": vname, "error": res.stderr[-800:]}), flush=True)
        continue
    for line in res.stdout.splitlines():
        d = json.loads(line)
        d["knobs"] = vname
        print(json.dumps(d), flush=True)
