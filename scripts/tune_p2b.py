"""P2 bench kernel at 2^28 on one B200: staging/caching knobs A/B, plus the
device's own streaming ceilings for the same byte mix.

Knobs (compile-time defines of csrc/tlk_template.cuh, via TLK_DEFINES):
TLK_STMODE (store flavour), TLK_L2HINT (evict-first L2 policy on the
read-once inputs), TLK_TILE_ORDER (interleaved vs contiguous tile runs per
persistent block), and the staged read share.  Ceilings: torch read-only
(sum), copy (read+write 1:1) and write-only (fill) over 8.6 GB, and a
5:3 read:write mix like P2's (40 reads, 24 writes) built from copies.

Usage: python scripts/tune_p2b.py [points] [reps]   -> JSON lines
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
from paper_1804_10120_b200.runtime import Kernel, fill_uniform  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 10


def timeit(fn, reps=REPS, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return statistics.median(ts), min(ts)


def ceilings():
    n = 1 << 30  # 8.6 GB of doubles
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    x.uniform_()
    t, _ = timeit(lambda: x.sum())
    print(json.dumps({"ceiling": "read_only_sum", "tbs": round(8 * n / t / 1e12, 4)}), flush=True)
    t, _ = timeit(lambda: y.copy_(x))
    print(json.dumps({"ceiling": "copy_1to1", "tbs": round(16 * n / t / 1e12, 4)}), flush=True)
    t, _ = timeit(lambda: y.fill_(1.5))
    print(json.dumps({"ceiling": "write_only_fill", "tbs": round(8 * n / t / 1e12, 4)}),
          flush=True)
    # 5:3 read:write: out[:3/5 n] = a + b style via torch.add over halves
    m = (n // 5) * 1
    a, b2, c = x[:m], x[m:2 * m], y[:m]
    t, _ = timeit(lambda: torch.add(a, b2, out=c))
    print(json.dumps({"ceiling": "add_2to1", "tbs": round(24 * m / t / 1e12, 4)}), flush=True)
    del x, y
    torch.cuda.empty_cache()


def main():
    prog, vs = tb.load(tb.P2)
    base = lower_program(vs)
    v0 = base.variant
    shapes = [
        ("policy", v0, ""),
        ("stmode1", v0, "-DTLK_STMODE=1"),
        ("stmode2", v0, "-DTLK_STMODE=2"),
        ("l2hint", v0, "-DTLK_L2HINT=1"),
        ("tile_chunked", v0, "-DTLK_TILE_ORDER=1"),
        ("r32", Variant(**{**v0.__dict__, "stage_reads": 32}), ""),
        ("r36", Variant(**{**v0.__dict__, "stage_reads": 36}), ""),
        ("r36_s3x256_l2hint", Variant(**{**v0.__dict__, "stage_reads": 36}), "-DTLK_L2HINT=1"),
        ("stmode1_l2hint", v0, "-DTLK_STMODE=1 -DTLK_L2HINT=1"),
        ("ws", Variant(**{**v0.__dict__, "stage_ws": 1}), ""),
        ("ws_r36", Variant(**{**v0.__dict__, "stage_ws": 1, "stage_reads": 36}), ""),
        ("ws_r40_s4x128", Variant(**{**v0.__dict__, "stage_ws": 1, "stage_reads": 40,
                                     "stage": 4, "stage_threads": 128}), ""),
        ("ws_r40_s2x256", Variant(**{**v0.__dict__, "stage_ws": 1, "stage_reads": 40,
                                     "stage": 2}), ""),
        ("ws_l2hint", Variant(**{**v0.__dict__, "stage_ws": 1}), "-DTLK_L2HINT=1"),
        ("policy_again", v0, ""),
    ]
    only = os.environ.get("SHAPES")
    if only:
        shapes = [s for s in shapes if s[0] in only.split(",")]
    bufs = []
    for k, info in enumerate(base.fields):
        b = torch.zeros(info.n_components, N, dtype=torch.float64, device="cuda")
        if k not in base.lhs_fields:
            for c in range(info.n_components):
                fill_uniform(b[c], 0xC0FFEE, (k << 8) | c)
        bufs.append(b)
    torch.cuda.synchronize()
    bases = [b.data_ptr() for b in bufs]
    pitches = [N if info.n_components > 1 else 0 for info in base.fields]
    stream = torch.cuda.current_stream().cuda_stream
    ref = None
    for sname, var, defines in shapes:
        os.environ["TLK_DEFINES"] = defines
        plan = lower_program(vs, variant=var)
        kern = Kernel(plan)
        for k in base.lhs_fields:
            bufs[k].zero_()
        t, tmin = timeit(lambda: kern.launch(N, bases, pitches, stream))
        # bitwise check of the written arrays against the first variant (sampled)
        sig = torch.cat([bufs[k][:, :: 4099].flatten() for k in base.lhs_fields])
        same = True
        if ref is None:
            ref = sig.clone()
        else:
            same = bool(torch.equal(sig.view(torch.int64), ref.view(torch.int64)))
        print(json.dumps({"shape": sname, "defines": defines, "variant": plan.variant.tag(),
                          "N": N, "ms": round(t * 1e3, 4), "min_ms": round(tmin * 1e3, 4),
                          "tbs": round(plan.bytes_per_point * N / t / 1e12, 4),
                          "bitwise_same": same}), flush=True)
        del kern
    os.environ["TLK_DEFINES"] = ""
    del bufs
    torch.cuda.empty_cache()
    ceilings()


if __name__ == "__main__":
    main()
