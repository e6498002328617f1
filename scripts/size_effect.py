"""Why does P2 reach 99 % of the measured copy bandwidth at 2^28 points but
~95 % at 2^24?  Times P2 at several sizes with the bench's field builder
(counter-RNG fill) and with make_env (torch uniform_), as an eager launch
loop (the bench's method) and as 20 launches in one CUDA graph, plus a
torch copy of the same byte count for the bandwidth reference.
Usage: PYTHONPATH=. python scripts/size_effect.py"""

import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1804_10120_b200 import bench as tb  # noqa: E402
from paper_1804_10120_b200 import capture_graph, eval_program  # noqa: E402
from paper_1804_10120_b200.evaluator import plan_for  # noqa: E402


def eager(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / k


def graphed(fn, k=20):
    g = capture_graph(lambda: [fn() for _ in range(k)])
    ts = []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / k)
    return statistics.median(ts[1:])


for e in (22, 24, 26, 28):
    n = 1 << e
    for builder in ("bench", "make_env"):
        if builder == "bench":
            prog, vs, env = bench.build_p2_env(n, 0, "cuda")
        else:
            prog, vs = tb.load(tb.P2)
            env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
            for f in env.values():
                f.resize(n)
                if f.name not in ("Gamma", "dtg"):
                    f.data.uniform_()
        plan = plan_for(vs, env)
        fn = lambda: eval_program(vs, env)  # noqa: E731
        k = 20 if e < 28 else 8
        te, tg = eager(fn, k), graphed(fn, k)
        gb = plan.bytes_per_point * n / 1e9
        print(json.dumps({"log2n": e, "builder": builder, "us_eager": te * 1e6,
                          "us_graph": tg * 1e6, "gbs_eager": gb / te, "gbs_graph": gb / tg}),
              flush=True)
        del env
        torch.cuda.empty_cache()
    # copy of the same byte count (half read, half written)
    half = plan.bytes_per_point * n // 2
    src = torch.empty(half // 8, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    tc = eager(lambda: dst.copy_(src), 10)
    print(json.dumps({"log2n": e, "builder": "torch_copy", "us_eager": tc * 1e6,
                      "gbs_eager": 2 * half / 1e9 / tc}), flush=True)
    del src, dst
    torch.cuda.empty_cache()
