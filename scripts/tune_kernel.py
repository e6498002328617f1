"""Launch/code-generation variants of the fused kernel, timed on one B200.

Each variant runs in a fresh subprocess with its knobs in the environment:
  TLK_DEFINES  e.g. "-DTLK_LDMODE=1" (load flavour), "-DTLK_STMODE=1"
  TLK_THREADS  block size (also __launch_bounds__)
  TLK_WAVES    grid = waves x SMs x resident blocks (0 = one wave)
  TLK_HOIST    1 = all loads first in the generated body
Prints one JSON line per (variant, program).
Usage: PYTHONPATH=. python scripts/tune_kernel.py [points]
"""

import json
import os
import subprocess
import sys

POINTS = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26

VARIANTS = {
    "base": {},
    "norestrict": {"TLK_RESTRICT": "0"},
    "vec1": {"TLK_VEC": "1"},
    "vec1_norestrict": {"TLK_VEC": "1", "TLK_RESTRICT": "0"},
    "vec1_waves4": {"TLK_VEC": "1", "TLK_WAVES": "4"},
    "norestrict_waves4": {"TLK_RESTRICT": "0", "TLK_WAVES": "4"},
    "ldnc": {"TLK_DEFINES": "-DTLK_LDMODE=1"},
    "ldnc_vec1": {"TLK_DEFINES": "-DTLK_LDMODE=1", "TLK_VEC": "1"},
    "hoist_ldnc": {"TLK_HOIST": "1", "TLK_DEFINES": "-DTLK_LDMODE=1"},
    "hoist_ldnc_vec1": {"TLK_HOIST": "1", "TLK_DEFINES": "-DTLK_LDMODE=1", "TLK_VEC": "1"},
    "hoist_ldnc_waves4": {"TLK_HOIST": "1", "TLK_DEFINES": "-DTLK_LDMODE=1", "TLK_WAVES": "4"},
    "hoist_waves4": {"TLK_HOIST": "1", "TLK_WAVES": "4"},
}

CHILD = r"""
import json, os, statistics, sys, torch
from paper_1804_10120_b200 import bench as tb, eval_program
from paper_1804_10120_b200.evaluator import plan_for, kernel_for
n = int(sys.argv[1])
suite = {e.name: e.source for e in tb.builtin_suite()}
progs = dict(tb.PROGRAMS)
progs.update({"contract1": suite["contract1"], "outer3": suite["outer3"], "kij": suite["kij"]})
n0 = n
for name in ("p2", "c3_christoffel", "c1_dtg", "c2_maxwell", "p3", "contract1", "outer3", "kij"):
    n = n0 // 4 if name in ("contract1", "outer3") else n0
    prog, vs = tb.load(progs[name])
    targets = {v.stmt.lhs.field for v in vs}
    env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
    for f in env.values():
        f.resize(n)
        if f.name not in targets:
            f.data.uniform_()
    plan = plan_for(vs, env)
    for _ in range(3):
        eval_program(vs, env)
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); eval_program(vs, env); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    t = statistics.median(ts[1:])
    k = kernel_for(vs, env)
    print(json.dumps({"program": name, "t_ms": t * 1e3, "n": n,
                      "gbs": plan.bytes_per_point * n / t / 1e9,
                      "regs": k.attrs("tlk_flat_v2")["registers"]}), flush=True)
    del env
    torch.cuda.empty_cache()
"""

for vname, knobs in VARIANTS.items():
    env = dict(os.environ, **knobs)
    res = subprocess.run([sys.executable, "-c", CHILD, str(POINTS)], env=env,
                         capture_output=True, text=True, timeout=600)
    if res.returncode != 0:
        print(json.dumps({"variant": vname, "error": res.stderr[-500:]}), flush=True)
        continue
    for line in res.stdout.splitlines():
        d = json.loads(line)
        d["variant"] = vname
        d["points"] = POINTS
        print(json.dumps(d), flush=True)
