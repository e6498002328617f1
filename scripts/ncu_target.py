"""One program at one size, launched a few times (an ncu target).
Usage: python scripts/ncu_target.py PROGRAM LOG2N"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200 import eval_program

name, n = sys.argv[1], 1 << int(sys.argv[2])
prog, vs = tb.load(tb.PROGRAMS[name])
targets = {v.stmt.lhs.field for v in vs}
env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
for f in env.values():
    f.resize(n)
    if f.name not in targets:
        f.data.uniform_()
for _ in range(3):
    eval_program(vs, env)
torch.cuda.synchronize()
