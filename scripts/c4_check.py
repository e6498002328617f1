"""C4 (512 subdomains x 16^3, P2 and the P3 chain) as one bound batched
launch: mean of 20 back-to-back launches x 5, CUDA events (a quick check of
the batch entry's code under the current lowering policy).
Usage: python scripts/c4_check.py -> JSON lines"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_10120_b200 import bench as tb  # noqa: E402
from paper_1804_10120_b200 import bind_batch  # noqa: E402
from paper_1804_10120_b200.evaluator import plan_for  # noqa: E402

for name, text in (("c4_p2", tb.P2), ("c4_p3", tb.P3)):
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
    fn = bind_batch(vs, envs)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 20 * 1e3)
    plan = plan_for(vs, envs[0])
    print(json.dumps({"config": name, "variant": plan.variant.tag(), "us_min": round(min(ts), 2),
                      "us_all": [round(t, 2) for t in ts],
                      "tbs": round(plan.bytes_per_point * 512 * 16**3 / min(ts) / 1e6, 4)}),
          flush=True)
    del envs, fn
    torch.cuda.empty_cache()
