"""Small-size streaming ceiling: is C1 64^3 (and C3 128^3) at the floor of
THIS part for its byte mix at its size?

For each config, the fused kernel and stream-mix probe kernels with the
SAME number of read and write streams at the SAME point count and no
arithmetic (scripts/stream_probe.cu: probe_mix1 one point per thread in a
one-shot grid of 128/256-thread blocks, or persistent; probe_mix two points per thread
in a persistent grid).  Each kernel is launched REPS times (mean reported) with a 256 MB
write + read flush before every launch (L2 cold and clean), CUDA events
around the launch alone; the floor of the method (a 1-element kernel after
the same flush) is reported beside.  Run under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`
the same script gives per-kernel device times with ncu's own cache flush.

Usage: PYTHONPATH=. python scripts/small_ceiling.py  -> JSON lines"""

from __future__ import annotations

import ctypes
import json
import os
import statistics

import torch

from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200 import bind_program
from paper_1804_10120_b200.evaluator import plan_for

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "_probe", "stream_probe.so"))
REPS = int(os.environ.get("REPS", "15"))
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

wbuf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(1 << 25, dtype=torch.float64, device="cuda")
tiny = torch.zeros(1, device="cuda")


def cold(fn):
    ts = []
    for _ in range(REPS):
        wbuf.zero_()
        rbuf.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    # event timestamps tick in ~2 us steps on this part: the mean, not the median
    return round(statistics.mean(ts[1:]), 2), round(min(ts), 2)


def env_for(text, n):
    prog, vs = tb.load(text)
    targets = {v.stmt.lhs.field for v in vs}
    env = tb.make_env(prog, "__none__", 0, tb.DEFAULT_SEED)
    for f in env.values():
        f.resize(n)
        if f.name not in targets:
            f.data.uniform_()
    return vs, env


def main():
    floor = cold(lambda: tiny.add_(1.0))
    print(json.dumps({"kernel": "floor_1elem", "us_mean": floor[0], "us_min": floor[1]}),
          flush=True)
    for name, text, n, nr, nw in (("C1_dtg_64^3", tb.DTG, 64**3, 16, 6),
                                  ("C3_christoffel_128^3", tb.CHRISTOFFEL, 128**3, 24, 18)):
        mb = 8 * n * (nr + nw) / 1e6
        vs, env = env_for(text, n)
        plan = plan_for(vs, env)
        run = bind_program(vs, env)
        run()
        med, mn = cold(run)
        print(json.dumps({"config": name, "kernel": "fused", "variant": plan.variant.tag(),
                          "MB": mb, "us_mean": med, "us_min": mn,
                          "tbs_mean": round(mb / med, 3)}), flush=True)
        del env, run
        torch.cuda.empty_cache()
        rs = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(nr)]
        ws = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(nw)]
        rp = (ctypes.c_void_p * nr)(*[x.data_ptr() for x in rs])
        wp = (ctypes.c_void_p * nw)(*[x.data_ptr() for x in ws])
        shapes = [("mix1_oneshot", 0, t) for t in (128, 256)]
        shapes += [("mix1_persistent", b, 256) for b in (4, 8)]
        for label, bps, threads in shapes:
            fn = lambda: lib.sp_mix1(rp, nr, wp, nw, ctypes.c_longlong(n), bps, threads, st)  # noqa
            assert fn() == 0
            med, mn = cold(fn)
            print(json.dumps({"config": name, "kernel": label, "threads": threads,
                              "blocks_per_sm": bps, "MB": mb, "us_mean": med, "us_min": mn,
                              "tbs_mean": round(mb / med, 3)}), flush=True)
        if (nr, nw) == (16, 6):
            for bps in (4, 8):
                fn = lambda: lib.sp_mix(rp, nr, wp, nw, ctypes.c_longlong(n // 2), bps, st)  # noqa
                assert fn() == 0
                med, mn = cold(fn)
                print(json.dumps({"config": name, "kernel": "mix_2pt_persistent",
                                  "blocks_per_sm": bps, "MB": mb, "us_mean": med,
                                  "us_min": mn, "tbs_mean": round(mb / med, 3)}),
                      flush=True)
        # the same bytes as reads only, and the inputs alone (no writes)
        for rr in ((nr + nw, 0), (nr, 0)):
            if rr not in ((22, 0), (16, 0)):
                continue
            xs = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(rr[0])]
            xp = (ctypes.c_void_p * rr[0])(*[x.data_ptr() for x in xs])
            fn = lambda: lib.sp_mix1(xp, rr[0], wp, 0, ctypes.c_longlong(n), 0, 128, st)  # noqa
            assert fn() == 0
            med, mn = cold(fn)
            mbr = 8 * n * rr[0] / 1e6
            print(json.dumps({"config": name, "kernel": f"read_only_{rr[0]}_streams",
                              "threads": 128, "MB": mbr, "us_mean": med, "us_min": mn,
                              "tbs_mean": round(mbr / med, 3)}), flush=True)
            del xs
        # the dispatch floor of the one-shot grid alone (no memory traffic)
        fn = lambda: lib.sp_mix1(rp, 0, wp, 0, ctypes.c_longlong(n), 0, 128, st)  # noqa
        assert fn() == 0
        med, mn = cold(fn)
        print(json.dumps({"config": name, "kernel": "empty_oneshot_grid", "threads": 128,
                          "us_mean": med, "us_min": mn}), flush=True)
        del rs, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
