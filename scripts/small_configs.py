"""Launch each small/mid BASELINE config a few times (for an ncu launch list:
gpu__time_duration per kernel = device time without the host/graph floor)."""
import torch

from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200 import eval_batch, eval_program

for name, text, n in (("C1", tb.DTG, 64**3), ("C3", tb.CHRISTOFFEL, 128**3),
                      ("C2", tb.MAXWELL, 10**3), ("C2", tb.MAXWELL, 10**4),
                      ("C2", tb.MAXWELL, 10**5), ("C2", tb.MAXWELL, 10**6)):
    prog, vs = tb.load(text)
    tg = {v.stmt.lhs.field for v in vs}
    env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
    for f in env.values():
        f.resize(n)
        if f.name not in tg:
            f.data.uniform_()
    torch.cuda.synchronize()
    for _ in range(5):
        eval_program(vs, env)
    torch.cuda.synchronize()
prog, vs = tb.load(tb.P2)
envs = []
for d in range(512):
    e = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED + d)
    for f in e.values():
        f.resize(16**3)
        if f.name not in ("Gamma", "dtg"):
            f.data.uniform_()
    envs.append(e)
for _ in range(5):
    eval_batch(vs, envs)
torch.cuda.synchronize()
