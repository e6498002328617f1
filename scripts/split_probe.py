"""Fused P2 (one launch: 40 read + 24 write streams at once) against the same
program as its two independent statements launched back to back (Γ: 24 R +
18 W streams, then ∂t g: 16 R + 6 W) over the SAME device fields —
interleaved rounds, K back-to-back launches (or launch pairs) per round,
CUDA events.  Measures what fewer concurrent DRAM streams are worth.

Usage: PYTHONPATH=. python scripts/split_probe.py  -> JSON lines"""

from __future__ import annotations

import json
import os
import statistics

import torch

from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200 import bind_program

ROUNDS = int(os.environ.get("ROUNDS", "7"))
SIZES = [int(x) for x in os.environ.get("SIZES", f"{1 << 25},{1 << 28}").split(",")]


def main():
    prog, vs = tb.load(tb.P2)
    for n in SIZES:
        env = tb.make_env(prog, "__none__", 0)
        for f in env.values():
            f.resize(n)
            if f.name not in ("Gamma", "dtg"):
                f.data.uniform_()
        k = max(2, min(20, (1 << 30) // n))
        fused = bind_program(vs, env)
        g1, g2 = bind_program([vs[0]], env), bind_program([vs[1]], env)
        shapes = {"fused": [fused], "split": [g1, g2]}
        outs = {}
        for label, fns in shapes.items():
            env["Gamma"].data.zero_()
            env["dtg"].data.zero_()
            for fn in fns:
                fn()
            torch.cuda.synchronize()
            outs[label] = torch.cat([env["Gamma"].data[:, 0, ::4099].flatten(),
                                     env["dtg"].data[:, 0, ::4099].flatten()]).clone()
        same = bool(torch.equal(outs["fused"].view(torch.int64), outs["split"].view(torch.int64)))
        ts = {label: [] for label in shapes}
        for _ in range(ROUNDS):
            for label, fns in shapes.items():
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(k):
                    for fn in fns:
                        fn()
                b.record()
                b.synchronize()
                ts[label].append(a.elapsed_time(b) / 1e3 / k)
        for label, t in ts.items():
            med = statistics.median(t)
            print(json.dumps({"program": "p2", "N": n, "shape": label,
                              "us_median": round(med * 1e6, 2), "us_min": round(min(t) * 1e6, 2),
                              "tbs_median": round(512 * n / med / 1e12, 4),
                              "bitwise_same": same}), flush=True)
        del env, fused, g1, g2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
