"""Warp-specialised staged entry (Variant.stage_ws) vs the policy's block-
barrier ring, per BASELINE program and size, on one B200.

For each (program, N): the policy variant and the same variant with
stage_ws=1 (and, for the heavier programs, a couple of ring shapes), timed
as the mean of 20 eager launches back to back (CUDA events; kernels of
>= 100 us, so the ~2 us event tick is noise) and as the mean of 15 single
launches queued behind a cold-and-clean L2 flush.  Every variant's output
is compared bitwise with the policy's.

Usage: python scripts/tune_ws.py  -> JSON lines
"""

from __future__ import annotations

import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1804_10120_b200 import bench as tb  # noqa: E402
from paper_1804_10120_b200.lowering import Variant, lower_program  # noqa: E402
from paper_1804_10120_b200.runtime import fill_uniform, get_kernel  # noqa: E402

wbuf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(1 << 25, dtype=torch.float64, device="cuda")


def flush():
    wbuf.zero_()
    rbuf.sum()


def b2b(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / k)
    return min(ts)


def single(fn, reps=15):
    ts = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.mean(ts)


def run(name, n):
    prog, vs = tb.load(tb.PROGRAMS[name])
    base = lower_program(vs)
    v0 = base.variant
    if base.variant.small_n and n <= base.variant.small_n:
        return
    shapes = {"policy": v0, "ws": Variant(**{**v0.__dict__, "stage_ws": 1})}
    if not v0.stage:
        return
    if v0.stage_reads >= 12:
        shapes["ws_s2"] = Variant(**{**v0.__dict__, "stage_ws": 1, "stage": 2})
        shapes["ws_t128"] = Variant(**{**v0.__dict__, "stage_ws": 1, "stage_threads": 128})
    bufs = []
    for k, info in enumerate(base.fields):
        b = torch.zeros(info.n_components, n, dtype=torch.float64, device="cuda")
        if k not in base.lhs_fields:
            for c in range(info.n_components):
                fill_uniform(b[c], 0xC0FFEE, (k << 8) | c)
        bufs.append(b)
    bases = [b.data_ptr() for b in bufs]
    pitches = [n if info.n_components > 1 else 0 for info in base.fields]
    want = None
    for sname, var in shapes.items():
        plan = lower_program(vs, variant=var)
        kern = get_kernel(plan)
        fn = lambda: kern.launch(n, bases, pitches,  # noqa: E731
                                 torch.cuda.current_stream().cuda_stream)
        fn()
        torch.cuda.synchronize()
        out = torch.cat([bufs[k][:, ::997].flatten() for k in base.lhs_fields])
        if want is None:
            want = out.clone()
        same = bool(torch.equal(out.view(torch.int64), want.view(torch.int64)))
        t_b2b = b2b(fn)
        t_one = single(fn)
        mb = plan.bytes_per_point * n
        print(json.dumps({"program": name, "N": n, "shape": sname, "variant": plan.variant.tag(),
                          "us_b2b": round(t_b2b * 1e6, 2), "us_single": round(t_one * 1e6, 2),
                          "tbs_b2b": round(mb / t_b2b / 1e12, 4),
                          "tbs_single": round(mb / t_one / 1e12, 4), "bitwise_same": same}),
              flush=True)
    del bufs
    torch.cuda.empty_cache()


def main():
    sizes = [int(x) for x in os.environ.get("SIZES", f"{1 << 21},{1 << 24},{1 << 26}").split(",")]
    progs = os.environ.get("PROGS", "c1_dtg,c2_maxwell,c3_christoffel,p2,p3").split(",")
    for name in progs:
        for n in sizes:
            run(name, n)


if __name__ == "__main__":
    main()
