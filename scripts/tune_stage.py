"""TMA-staged entry (tlk_stage_v1) against the policy kernels: each program
at 2^21 and 2^24 points under stage depths / block sizes, timed as one graph
replay after a clean L2 flush and 20 back-to-back launches in one graph.
Usage: PYTHONPATH=. python scripts/tune_stage.py [grid|frac|light] > tune_stage.jsonl"""

import json
import os
import subprocess
import sys

VARIANTS = {"policy": {}, "nostage": {"TLK_STAGE": "0"},
            "nostage_h0": {"TLK_STAGE": "0", "TLK_HOIST": "0"}}
if len(sys.argv) > 1 and sys.argv[1] == "frac":
    VARIANTS = {"policy": {}}
    for th in (128, 256):
        for fr in ("0.5", "0.625", "0.75", "0.875", "1.0"):
            VARIANTS[f"g3x{th}f{fr}"] = {"TLK_STAGE": "3", "TLK_STAGE_THREADS": str(th),
                                         "TLK_STAGE_FRAC": fr}
if len(sys.argv) > 1 and sys.argv[1] == "light":
    VARIANTS = {"policy": {}}
    for depth in (3, 4):
        for r in (4, 6, 8, 10, 12, 14, 16):
            VARIANTS[f"g{depth}x256r{r}"] = {"TLK_STAGE": str(depth), "TLK_STAGE_THREADS": "256",
                                            "TLK_STAGE_READS": str(r)}
if len(sys.argv) > 1 and sys.argv[1] == "grid":
    for st in (2, 3, 4, 6):
        for th in (128, 256):
            VARIANTS[f"g{st}x{th}"] = {"TLK_STAGE": str(st), "TLK_STAGE_THREADS": str(th)}

CHILD = r"""
import json, statistics, sys, torch
from paper_1804_10120_b200 import bench as tb, eval_program, capture_graph
from paper_1804_10120_b200.evaluator import plan_for, kernel_for
wbuf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(1 << 25, dtype=torch.float64, device="cuda")
def clean():
    wbuf.zero_(); rbuf.sum()
def single(fn, reps):
    g = capture_graph(fn); ts = []
    for _ in range(reps):
        clean()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts[1:])
def b2b(fn, k=20):
    g = capture_graph(lambda: [fn() for _ in range(k)]); ts = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / k)
    return statistics.median(ts[1:])
for name in (("c1_dtg", "c2_maxwell") if len(sys.argv) > 1 and sys.argv[1] == "light"
             else ("c3_christoffel", "p2", "p3", "c1_dtg", "c2_maxwell")):
    for n in ((1 << 24, 1 << 26) if len(sys.argv) > 1 and sys.argv[1] in ("frac", "light")
              else (1 << 21, 1 << 24, 1 << 26)):
        prog, vs = tb.load(tb.PROGRAMS[name])
        targets = {v.stmt.lhs.field for v in vs}
        env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
        for f in env.values():
            f.resize(n)
            if f.name not in targets:
                f.data.uniform_()
        plan = plan_for(vs, env)
        kern = kernel_for(vs, env)
        fn = lambda: eval_program(vs, env)
        try:
            ts, tb2 = single(fn, 7 if n >= 1 << 24 else 21), b2b(fn, 10 if n >= 1 << 26 else 20)
        except Exception as e:
            print(json.dumps({"program": name, "n": n, "error": str(e)[:300]}), flush=True)
            continue
        entry = "tlk_stage_v1" if kern.vec == 3 else "tlk_flat_v2"
        try:
            attrs = kern.attrs(entry)
        except Exception:
            attrs = {}
        print(json.dumps({"program": name, "n": n, "us_single_clean": ts * 1e6,
                          "us_b2b": tb2 * 1e6,
                          "gbs_single": plan.bytes_per_point * n / ts / 1e9,
                          "gbs_b2b": plan.bytes_per_point * n / tb2 / 1e9,
                          "variant": plan.variant.tag(), "entry": entry, **attrs}), flush=True)
        del env
        torch.cuda.empty_cache()
"""

for vname, knobs in VARIANTS.items():
    env = dict(os.environ, **knobs)
    res = subprocess.run([sys.executable, "-c", CHILD, *sys.argv[1:2]], env=env, capture_output=True, text=True,
                         timeout=900)
    if res.returncode != 0:
        print(json.dumps({"knobs": vname, "error": res.stderr[-800:]}), flush=True)
        continue
    for line in res.stdout.splitlines():
        d = json.loads(line)
        d["knobs"] = vname
        print(json.dumps(d), flush=True)
