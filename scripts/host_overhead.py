"""Host-side cost per call (eager, no graph) of the public entry points at
small sizes, where the host can dominate: eval_program on C1 64^3,
eval_batch on C4 (512 x 16^3) cold-path / steady-state, and the bound
launches.  Each figure is wall time per call over 200 calls with a final
synchronize (GPU time per launch is the floor).
Usage: PYTHONPATH=. python scripts/host_overhead.py"""
import json
import time

import torch

from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200 import bind_batch, bind_program, eval_batch, eval_program
from paper_1804_10120_b200.evaluator import _BATCH_FAST


def per_call(fn, k=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k


prog, vs = tb.load(tb.DTG)
env = tb.make_env(prog, "dtg", 64**3, tb.DEFAULT_SEED, device="cuda")
out = {"c1_eval_program_us": per_call(lambda: eval_program(vs, env)) * 1e6}
b = bind_program(vs, env)
out["c1_bound_program_us"] = per_call(b) * 1e6

prog, vs = tb.load(tb.P2)
envs = [tb.make_env(prog, "Gamma", 16**3, tb.DEFAULT_SEED + d, device="cuda") for d in range(512)]


def cold():
    _BATCH_FAST.clear()
    eval_batch(vs, envs)


out["c4_eval_batch_cold_us"] = per_call(cold, 20) * 1e6
out["c4_eval_batch_steady_us"] = per_call(lambda: eval_batch(vs, envs)) * 1e6
bb = bind_batch(vs, envs)
out["c4_bound_batch_us"] = per_call(bb) * 1e6
print(json.dumps(out))
