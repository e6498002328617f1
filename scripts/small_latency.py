"""Small/mid-N timing methodology study (graph replay, CUDA events).

For each config: the event-bracketed time of one graph replay after
  (a) a 256 MB write flush       (L2 left full of dirty lines: their
                                  write-back lands inside the timed kernel)
  (b) a write + 256 MB read flush (L2 cold AND clean)
  (c) no flush                    (inputs L2-resident when they fit)
plus the floor of the method itself (a graph holding one 1-element torch
kernel) and the per-launch time of 20 back-to-back launches in one graph.
Usage: PYTHONPATH=. python scripts/small_latency.py"""

import json
import statistics

import torch

from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200 import capture_graph, eval_batch, eval_program
from paper_1804_10120_b200.evaluator import plan_for

wbuf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(1 << 25, dtype=torch.float64, device="cuda")  # 256 MB


def flush(mode):
    if mode in ("write", "clean"):
        wbuf.zero_()
    if mode == "clean":
        rbuf.sum()


def timed(fn, mode, reps=25):
    g = capture_graph(fn)
    ts = []
    for _ in range(reps):
        flush(mode)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts[1:])


def per_launch(fn, k=20):
    g = capture_graph(lambda: [fn() for _ in range(k)])
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / k)
    return statistics.median(ts[1:])


tiny = torch.zeros(1, device="cuda")
for mode in ("write", "clean", "none"):
    print(json.dumps({"config": "floor_1elem_kernel", "flush": mode,
                      "us": timed(lambda: tiny.add_(1.0), mode) * 1e6}), flush=True)


def env_for(text, n, seed=tb.DEFAULT_SEED):
    prog, vs = tb.load(text)
    targets = {v.stmt.lhs.field for v in vs}
    env = tb.make_env(prog, "__none__", 0, seed)
    for f in env.values():
        f.resize(n)
        if f.name not in targets:
            f.data.uniform_()
    return vs, env


for name, text, n in (("C1_dtg", tb.DTG, 64**3), ("C3_christoffel", tb.CHRISTOFFEL, 128**3),
                      ("C2_maxwell", tb.MAXWELL, 10**5), ("C2_maxwell", tb.MAXWELL, 10**6),
                      ("C1_dtg", tb.DTG, 1 << 21), ("P2", tb.P2, 1 << 21)):
    vs, env = env_for(text, n)
    plan = plan_for(vs, env)
    fn = lambda: eval_program(vs, env)  # noqa: E731
    row = {"config": name, "N": n, "MB": plan.bytes_per_point * n / 1e6,
           "variant": plan.variant.tag()}
    for mode in ("write", "clean", "none"):
        row["us_" + mode] = timed(fn, mode) * 1e6
    row["us_b2b"] = per_launch(fn) * 1e6
    print(json.dumps(row), flush=True)
    del env
    torch.cuda.empty_cache()

for name, text in (("C4_p2", tb.P2), ("C4_p3", tb.P3)):
    envs = []
    vs = None
    for d in range(512):
        vs, e = env_for(text, 16**3, tb.DEFAULT_SEED + d)
        envs.append(e)
    plan = plan_for(vs, envs[0])
    fn = lambda: eval_batch(vs, envs)  # noqa: E731
    row = {"config": name, "N": 512 * 16**3, "MB": plan.bytes_per_point * 512 * 16**3 / 1e6,
           "variant": plan.variant.tag()}
    for mode in ("write", "clean", "none"):
        row["us_" + mode] = timed(fn, mode) * 1e6
    row["us_b2b"] = per_launch(fn) * 1e6
    print(json.dumps(row), flush=True)
    del envs
