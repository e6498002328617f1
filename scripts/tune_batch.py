"""C4 multi-domain batch variants (512 x 16^3, P2 and the P3 chain), graph
replay with L2 flush.  Usage: PYTHONPATH=. python scripts/tune_batch.py"""
import json
import os
import subprocess
import sys

VARIANTS = {
    "smem_v2": {},
    "smem_v1": {"TLK_BATCH_VEC": "1"},
    "table_v2": {"TLK_BATCH_PTRS": "1"},
    "table_v1": {"TLK_BATCH_PTRS": "1", "TLK_BATCH_VEC": "1"},
    "table_v2_t128": {"TLK_BATCH_PTRS": "1", "TLK_THREADS": "128"},
    "table_v1_t128": {"TLK_BATCH_PTRS": "1", "TLK_BATCH_VEC": "1", "TLK_THREADS": "128"},
    "smem_v2_t512": {"TLK_THREADS": "512"},
    "table_v2_t512": {"TLK_BATCH_PTRS": "1", "TLK_THREADS": "512"},
}

CHILD = r"""
import json, statistics, torch
from paper_1804_10120_b200 import bench as tb, eval_batch, capture_graph
from paper_1804_10120_b200.evaluator import plan_for
flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
for name, text in (("p2", tb.P2), ("p3", tb.P3)):
    prog, vs = tb.load(text)
    tg = {v.stmt.lhs.field for v in vs}
    envs = []
    for d in range(512):
        e = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED + d)
        for f in e.values():
            f.resize(16**3)
            if f.name not in tg: f.data.uniform_()
        envs.append(e)
    g = capture_graph(lambda: eval_batch(vs, envs))
    ts = []
    for _ in range(31):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) / 1e3)
    t = statistics.median(ts[1:])
    plan = plan_for(vs, envs[0])
    print(json.dumps({"program": name, "us": t * 1e6,
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
