"""BASELINE configs as ncu targets (final policy): C1 64^3, C3 128^3,
C2 Maxwell 10^8, C4 P2 and P3 chain (512 x 16^3, one batched launch).
Usage: python scripts/ncu_configs.py CONFIG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200 import eval_batch, eval_program


def env_for(name, n, seed=tb.DEFAULT_SEED):
    prog, vs = tb.load(tb.PROGRAMS[name])
    targets = {v.stmt.lhs.field for v in vs}
    env = tb.make_env(prog, "__none__", 0, seed)
    for f in env.values():
        f.resize(n)
        if f.name not in targets:
            f.data.uniform_()
    return vs, env


which = sys.argv[1]
if which.startswith("c4_"):
    name = which[3:]
    envs = []
    for d in range(512):
        vs, e = env_for(name, 16**3, tb.DEFAULT_SEED + d)
        envs.append(e)
    for _ in range(3):
        eval_batch(vs, envs)
else:
    name, n = {"c1": ("c1_dtg", 64**3), "c3": ("c3_christoffel", 128**3),
               "c2": ("c2_maxwell", 10**8)}[which]
    vs, env = env_for(name, n)
    for _ in range(3):
        eval_program(vs, env)
torch.cuda.synchronize()
