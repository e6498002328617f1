"""Streaming ceilings of this B200 (see scripts/stream_probe.cu): pure reads
(LDG.128 at several unrolls/occupancies, and TMA bulk copies), pure writes,
a 1:1 copy-like mix, and P2's 40:24 read:write stream mix with no
arithmetic.  Each line: best of 3 rounds of 10 back-to-back launches over
>= 8 GB (far beyond L2), CUDA events.

Usage: python scripts/stream_probe.py  -> JSON lines"""

from __future__ import annotations

import ctypes
import json
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_probe", "stream_probe.so")


def timeit(fn, k=10):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            fn()
        b.record()
        b.synchronize()
        t = a.elapsed_time(b) / 1e3 / k
        best = t if best is None else min(best, t)
    return best


def main():
    lib = ctypes.CDLL(LIB)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    n = 1 << 30  # doubles: 8.6 GB
    a = torch.rand(n, dtype=torch.float64, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    n2 = ctypes.c_longlong(n // 2)
    res = []

    def rec(name, bytes_, t, **kw):
        d = {"probe": name, "tbs": round(bytes_ / t / 1e12, 4), "ms": round(t * 1e3, 3), **kw}
        res.append(d)
        print(json.dumps(d), flush=True)

    for unroll in (1, 2, 4, 8):
        for bps in (4, 8):
            t = timeit(lambda: lib.sp_read(ctypes.c_void_p(a.data_ptr()), n2,
                                           ctypes.c_void_p(out.data_ptr()), unroll, bps, st))
            rec("read_ldg128", 8 * n, t, unroll=unroll, blocks_per_sm=bps)
    for chunk, bps in ((4096, 4), (4096, 7), (16384, 2), (16384, 3), (32768, 1)):
        t = timeit(lambda: lib.sp_bulk(ctypes.c_void_p(a.data_ptr()), ctypes.c_longlong(8 * n),
                                       chunk, bps, st))
        rec("read_tma_bulk", 8 * n, t, chunk=chunk, blocks_per_sm=bps)
    modes = {0: "st.global.cs", 1: "st.global", 2: "st.global.L1::no_allocate", 4: "st.global.wt"}
    for width in (16, 8):
        for mode, mname in modes.items():
            for bps in (4, 8):
                t = timeit(lambda: lib.sp_write(ctypes.c_void_p(a.data_ptr()), n2, bps, st, mode,
                                                width))
                rec("write", 8 * n, t, store=mname, width=width, blocks_per_sm=bps)
    for bps in (2, 4, 8):
        t = timeit(lambda: lib.sp_bulk_store(ctypes.c_void_p(a.data_ptr()),
                                             ctypes.c_longlong(8 * n), bps, st))
        rec("write_tma_bulk_store", 8 * n, t, chunk=8192, blocks_per_sm=bps)
    t = timeit(lambda: a.fill_(1.5))
    rec("write_torch_fill", 8 * n, t)
    for bps in (4, 8):
        t = timeit(lambda: lib.sp_write_v4(ctypes.c_void_p(a.data_ptr()), ctypes.c_longlong(n),
                                           bps, st))
        rec("write", 8 * n, t, store="st.global.v4.f64 (256-bit)", width=32, blocks_per_sm=bps)
    for w in (1, 2, 4):
        t = timeit(lambda: lib.sp_write_np(ctypes.c_void_p(a.data_ptr()), ctypes.c_longlong(n),
                                           w, st))
        rec("write_nonpersistent_grid", 8 * n, t, width=8 * w)
    half = n // 2
    src, dst = a[:half], a[half:2 * half]
    for mode, mname in modes.items():
        for bps in (4, 8):
            t = timeit(lambda: lib.sp_copy1(ctypes.c_void_p(src.data_ptr()),
                                            ctypes.c_void_p(dst.data_ptr()),
                                            ctypes.c_longlong(half), bps, st, mode))
            rec("copy_8B_per_thread", 16 * half, t, store=mname, blocks_per_sm=bps)
    t = timeit(lambda: dst.copy_(src))
    rec("copy_torch", 16 * half, t)
    for w in (1, 2, 4):
        t = timeit(lambda: lib.sp_copy_np(ctypes.c_void_p(src.data_ptr()),
                                          ctypes.c_void_p(dst.data_ptr()),
                                          ctypes.c_longlong(half), w, st))
        rec("copy_nonpersistent_grid", 16 * half, t, width=8 * w)
    for bps in (4, 8):
        t = timeit(lambda: lib.sp_copy_v4(ctypes.c_void_p(src.data_ptr()),
                                          ctypes.c_void_p(dst.data_ptr()),
                                          ctypes.c_longlong(half), bps, st))
        rec("copy_v4_persistent", 16 * half, t, width=32, blocks_per_sm=bps)
    del a
    torch.cuda.empty_cache()
    # stream mixes: m points per stream, nr + nw streams
    for nr, nw in ((1, 1), (5, 3), (40, 24)):
        m = (1 << 34) // (8 * (nr + nw))  # ~17 GB in total
        m -= m % 512
        rs = [torch.rand(m, dtype=torch.float64, device="cuda") for _ in range(nr)]
        ws = [torch.empty(m, dtype=torch.float64, device="cuda") for _ in range(nw)]
        rp = (ctypes.c_void_p * nr)(*[x.data_ptr() for x in rs])
        wp = (ctypes.c_void_p * nw)(*[x.data_ptr() for x in ws])
        for bps in (2, 4, 8):
            t = timeit(lambda: lib.sp_mix(rp, nr, wp, nw, ctypes.c_longlong(m // 2), bps, st))
            rec("mix_ldg128_stcs128", 8 * m * (nr + nw), t, reads=nr, writes=nw,
                blocks_per_sm=bps)
        for threads in (128, 256):
            t = timeit(lambda: lib.sp_mix1(rp, nr, wp, nw, ctypes.c_longlong(m), 0, threads, st))
            rec("mix_ldg64_stcs64_oneshot", 8 * m * (nr + nw), t, reads=nr, writes=nw,
                threads=threads)
        del rs, ws
        torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    sys.exit(0 if main() else 1)
