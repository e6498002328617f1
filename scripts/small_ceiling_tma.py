"""C1 64^3 against TMA: (1) the cold read of C1's 33.5 MB of inputs by TMA
bulk copies (scripts/stream_probe.cu probe_bulk: one elected thread per
block keeps 4-8 chunks in flight), (2) C1's own TMA-staged entry
(tlk_stage_v1; ring depth x tile), beside the policy kernel.  Each launch
follows a 256 MB write + read flush (cold, clean L2); under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum` the same
launches give device times with ncu's own flush.
Usage: PYTHONPATH=. python scripts/small_ceiling_tma.py -> JSON lines"""

from __future__ import annotations

import ctypes
import json
import os
import statistics

import torch

from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200.evaluator import _bind
from paper_1804_10120_b200.lowering import Variant, lower_program
from paper_1804_10120_b200.runtime import Kernel

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "_probe", "stream_probe.so"))
REPS = int(os.environ.get("REPS", "15"))
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
wbuf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(1 << 25, dtype=torch.float64, device="cuda")


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
    return round(statistics.mean(ts[1:]), 2), round(min(ts), 2)


def main():
    n = 64**3
    buf = torch.rand(16 * n, dtype=torch.float64, device="cuda")  # C1's 16 input arrays
    for chunk, bps in ((4096, 4), (4096, 7), (16384, 2), (16384, 3), (32768, 1)):
        fn = lambda: lib.sp_bulk(ctypes.c_void_p(buf.data_ptr()),  # noqa: E731
                                 ctypes.c_longlong(buf.numel() * 8), chunk, bps, st)
        assert fn() == 0
        mean, mn = cold(fn)
        print(json.dumps({"kernel": "tma_bulk_read_inputs", "chunk": chunk, "blocks_per_sm": bps,
                          "MB": buf.numel() * 8 / 1e6, "us_mean": mean, "us_min": mn}), flush=True)
    del buf
    prog, vs = tb.load(tb.DTG)
    env = tb.make_env(prog, "__none__", 0)
    for f in env.values():
        f.resize(n)
        if f.name != "dtg":
            f.data.uniform_()
    _, _, stores = _bind(vs, env)
    bases, pitches = [s.base for s in stores], [s.pitch for s in stores]
    shapes = {"policy": None}
    for depth in (2, 3):
        for tile in (64, 128, 256):
            shapes[f"staged_d{depth}_t{tile}"] = Variant(stage=depth, stage_threads=tile,
                                                         vec=1, waves=1)
    want = None
    for label, var in shapes.items():
        plan = lower_program(vs) if var is None else lower_program(vs, variant=var)
        k = Kernel(plan)
        fn = lambda: k.launch(n, bases, pitches, st.value)  # noqa: E731
        fn()
        torch.cuda.synchronize()
        got = env["dtg"].data.clone()
        want = got if want is None else want
        mean, mn = cold(fn)
        print(json.dumps({"kernel": "c1_" + label, "variant": plan.variant.tag(),
                          "us_mean": mean, "us_min": mn,
                          "bitwise_same": bool(torch.equal(got.view(torch.int64),
                                                           want.view(torch.int64)))}),
              flush=True)


if __name__ == "__main__":
    main()
