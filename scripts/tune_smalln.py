"""Small-N variant tuning: every (program, N) below under code-generation /
launch variants, timed as one graph replay after a clean L2 flush (256 MB
write, then 256 MB read) and as 20 back-to-back launches in one graph.
Usage: PYTHONPATH=. python scripts/tune_smalln.py [sizes] > tune_smalln.jsonl
(sizes: "small" (default) or "cross": 2^20..2^26 to locate variant crossovers)"""

import json
import os
import subprocess
import sys

CROSS = len(sys.argv) > 1 and sys.argv[1] == "cross"
VARIANTS_CROSS = {
    "policy": {},
    "v1w4": {"TLK_VEC": "1", "TLK_WAVES": "4"},
    "h1v1w4": {"TLK_HOIST": "1", "TLK_VEC": "1", "TLK_WAVES": "4"},
    "l1v1w4": {"TLK_LDMODE": "1", "TLK_VEC": "1", "TLK_WAVES": "4"},
    "h1l1v1w4": {"TLK_HOIST": "1", "TLK_LDMODE": "1", "TLK_VEC": "1", "TLK_WAVES": "4"},
    "h1l1v1w1": {"TLK_HOIST": "1", "TLK_LDMODE": "1", "TLK_VEC": "1", "TLK_WAVES": "1"},
    "h1l1v2w1": {"TLK_HOIST": "1", "TLK_LDMODE": "1", "TLK_VEC": "2", "TLK_WAVES": "1"},
}
VARIANTS = {
    "policy": {},
    "nosmall": {"TLK_SMALL_N": "0"},  # the large-N choice (staged entry) at every size
    "h1": {"TLK_HOIST": "1"},
    "l1": {"TLK_LDMODE": "1"},
    "h1l1": {"TLK_HOIST": "1", "TLK_LDMODE": "1"},
    "h1l1v2": {"TLK_HOIST": "1", "TLK_LDMODE": "1", "TLK_VEC": "2"},
    "h1l1v1": {"TLK_HOIST": "1", "TLK_LDMODE": "1", "TLK_VEC": "1"},
    "h1l1v1w1": {"TLK_HOIST": "1", "TLK_LDMODE": "1", "TLK_VEC": "1", "TLK_WAVES": "1"},
    "h1l1v2w4": {"TLK_HOIST": "1", "TLK_LDMODE": "1", "TLK_VEC": "2", "TLK_WAVES": "4"},
    "v2": {"TLK_VEC": "2"},
    "t128": {"TLK_THREADS": "128"},
    "h1l1t128": {"TLK_HOIST": "1", "TLK_LDMODE": "1", "TLK_THREADS": "128"},
}

CHILD = r"""
import json, statistics, torch
from paper_1804_10120_b200 import bench as tb, eval_program, capture_graph
from paper_1804_10120_b200.evaluator import plan_for
wbuf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(1 << 25, dtype=torch.float64, device="cuda")
def clean():
    wbuf.zero_(); rbuf.sum()
def single(fn, reps=25):
    g = capture_graph(fn); ts = []
    for _ in range(reps):
        clean()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts[1:])
def b2b(fn, k=20):
    g = capture_graph(lambda: [fn() for _ in range(k)]); ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / k)
    return statistics.median(ts[1:])
import sys
if sys.argv[1] == "cross":
    CASES = [(p, 1 << e) for p in ("c2_maxwell", "c1_dtg", "c3_christoffel", "p2", "p3")
             for e in (20, 22, 23, 24, 26)]
else:
    CASES = (("c2_maxwell", 10**3), ("c2_maxwell", 10**4), ("c2_maxwell", 10**5),
             ("c2_maxwell", 10**6), ("c1_dtg", 64**3), ("c3_christoffel", 64**3),
             ("c3_christoffel", 128**3), ("p2", 128**3), ("p3", 128**3))
for name, n in CASES:
    prog, vs = tb.load(tb.PROGRAMS[name])
    targets = {v.stmt.lhs.field for v in vs}
    env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
    for f in env.values():
        f.resize(n)
        if f.name not in targets:
            f.data.uniform_()
    plan = plan_for(vs, env)
    fn = lambda: eval_program(vs, env)
    ts, tb2 = single(fn, 9 if n >= 1 << 24 else 25), b2b(fn)
    print(json.dumps({"program": name, "n": n, "us_single_clean": ts * 1e6, "us_b2b": tb2 * 1e6,
                      "gbs_single": plan.bytes_per_point * n / ts / 1e9,
                      "gbs_b2b": plan.bytes_per_point * n / tb2 / 1e9,
                      "variant": plan.variant.tag()}), flush=True)
    del env
    torch.cuda.empty_cache()
"""

for vname, knobs in (VARIANTS_CROSS if CROSS else VARIANTS).items():
    env = dict(os.environ, **knobs)
    res = subprocess.run([sys.executable, "-c", CHILD, "cross" if CROSS else "small"], env=env, capture_output=True, text=True,
                         timeout=900)
    if res.returncode != 0:
        print(json.dumps({"knobs": vname, "error": res.stderr[-800:]}), flush=True)
        continue
    for line in res.stdout.splitlines():
        d = json.loads(line)
        d["knobs"] = vname
        print(json.dumps(d), flush=True)
