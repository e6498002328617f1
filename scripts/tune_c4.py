"""C4 batch launch shapes, interleaved A/B: block size x chunks per block
(TLB_BATCH_CHUNKS is read once per process, so each shape runs in its own
subprocess; rounds alternate shapes).  Usage: python scripts/tune_c4.py"""
import json
import os
import subprocess
import sys

CHILD = r"""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200.evaluator import _batch_plan
name, threads = sys.argv[1], int(sys.argv[2])
text = {"p2": tb.P2, "p3": tb.P3}[name]
prog, vs = tb.load(text)
targets = {v.stmt.lhs.field for v in vs}
envs = []
for d in range(512):
    env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED + d)
    for f in env.values():
        f.resize(16**3)
        if f.name not in targets:
            f.data.uniform_()
    envs.append(env)
kern, key, dev = _batch_plan(vs, envs)
from paper_1804_10120_b200.evaluator import _batches
stream = torch.cuda.current_stream().cuda_stream
batch = _batches.get(kern, key, stream)
fn = lambda: batch.launch(stream, threads=threads)
for _ in range(5):
    fn()
torch.cuda.synchronize()
ts = []
for _ in range(7):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record(); b.synchronize()
    ts.append(a.elapsed_time(b) / 20 * 1e3)
ts.sort()
print(json.dumps({"us_median": ts[3], "us_min": ts[0]}))
"""

shapes = [(t, c) for t in (64, 128, 256) for c in (1, 2, 4)]
for name in ("p2", "p3"):
    res = {s: [] for s in shapes}
    for _ in range(3):
        for t, c in shapes:
            env = dict(os.environ, TLB_BATCH_CHUNKS=str(c))
            out = subprocess.run([sys.executable, "-c", CHILD, name, str(t)], env=env,
                                 capture_output=True, text=True, timeout=600)
            if out.returncode:
                print(json.dumps({"program": name, "threads": t, "chunks": c,
                                  "error": out.stderr[-400:]}), flush=True)
                continue
            res[(t, c)].append(json.loads(out.stdout.strip().splitlines()[-1])["us_median"])
    for (t, c), v in res.items():
        if v:
            v.sort()
            print(json.dumps({"program": "c4_" + name, "threads": t, "chunks": c,
                              "us_median_of_rounds": v[len(v) // 2], "us_all": v}), flush=True)
