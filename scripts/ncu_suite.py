"""A suite statement (bench.builtin_suite) at 2^22 points as an ncu target:
3 launches of the default policy's kernel.
Usage: python scripts/ncu_suite.py NAME"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1804_10120_b200 import bench as tb  # noqa: E402
from paper_1804_10120_b200 import eval_program  # noqa: E402

src = {e.name: e.source for e in tb.builtin_suite()}[sys.argv[1]]
prog, vs = tb.load(src)
targets = {v.stmt.lhs.field for v in vs}
env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
for f in env.values():
    f.resize(1 << 22)
    if f.name not in targets:
        f.data.uniform_()
for _ in range(3):
    eval_program(vs, env)
torch.cuda.synchronize()
