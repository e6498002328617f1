"""C4 (512 subdomains of 16^3 points, one launch) through the plain batch
entry and the TMA-staged batch entry under ring shapes: one graph replay
after a clean L2 flush, and 20 back-to-back launches in one graph.
Usage: PYTHONPATH=. python scripts/tune_batch_stage.py [threads] > out.jsonl"""

import json
import os
import subprocess
import sys

VARIANTS = {"policy": {}, "staged": {"TLK_BATCH_VEC": "3"}}
if len(sys.argv) > 1 and sys.argv[1] == "threads":
    VARIANTS = {"policy": {}}
    for th in (64, 128, 192):
        VARIANTS[f"bt{th}"] = {"TLK_BATCH_THREADS": str(th)}
        VARIANTS[f"bt{th}_v2"] = {"TLK_BATCH_THREADS": str(th), "TLK_BATCH_VEC": "2"}
    VARIANTS["bptrs1_bt128"] = {"TLK_BATCH_THREADS": "128", "TLK_BATCH_PTRS": "1"}
else:
    for th in (128, 256):
        for fr in ("0.5", "0.75", "1.0"):
            VARIANTS[f"staged_x{th}f{fr}"] = {"TLK_BATCH_VEC": "3",
                                              "TLK_STAGE_THREADS": str(th),
                                              "TLK_STAGE_FRAC": fr}

CHILD = r"""
import json, statistics, torch
from paper_1804_10120_b200 import bench as tb, eval_batch, capture_graph
from paper_1804_10120_b200.evaluator import plan_for, kernel_for
wbuf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(1 << 25, dtype=torch.float64, device="cuda")
def single(fn, reps=21):
    g = capture_graph(fn); ts = []
    for _ in range(reps):
        wbuf.zero_(); rbuf.sum()
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
for name in ("p2", "p3"):
    prog, vs = tb.load(tb.PROGRAMS[name])
    targets = {v.stmt.lhs.field for v in vs}
    envs = []
    for d in range(512):
        e = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED + d)
        for f in e.values():
            f.resize(16**3)
            if f.name not in targets:
                f.data.uniform_()
        envs.append(e)
    plan = plan_for(vs, envs[0])
    kern = kernel_for(vs, envs[0])
    fn = lambda: eval_batch(vs, envs)
    ts, tb2 = single(fn), b2b(fn)
    gb = plan.bytes_per_point * 512 * 16**3 / 1e9
    print(json.dumps({"program": name, "n": 512 * 16**3, "us_single_clean": ts * 1e6,
                      "us_b2b": tb2 * 1e6, "gbs_single": gb / ts, "gbs_b2b": gb / tb2,
                      "variant": plan.variant.tag(), "batch_vec": kern.batch_vec}), flush=True)
    del envs
    torch.cuda.empty_cache()
"""

for vname, knobs in VARIANTS.items():
    env = dict(os.environ, **knobs)
    res = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True,
                         timeout=900)
    if res.returncode != 0:
        print(json.dumps({"knobs": vname, "error": res.stderr[-800:]}), flush=True)
        continue
    for line in res.stdout.splitlines():
        d = json.loads(line)
        d["knobs"] = vname
        print(json.dumps(d), flush=True)
