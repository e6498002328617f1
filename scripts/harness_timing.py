"""The reference's unchanged tl_harness driving the b200 bindings on C3
(Christoffel, 128^3 points) — VERDICT r01 "what's next" #7.

1. Whole-process wall time of `tl_harness <so> <manifest> in.tldf out.tldf`
   with our bindings (pageable host arrays: TLB_HOST_REGISTER=0, and
   page-locked for the call: =1) and with the reference's own emitted C
   (oracle/_ref/c3_christoffel.so), same fixture; outputs compared bitwise
   with the reference's tl_compare.
2. The bindings' `call` alone through ctypes (oracle/refc, the harness's
   wiring) on pageable numpy arrays, host-registered arrays and pinned
   (cudaHostAlloc) arrays: seconds per call, and the reference C on all
   cores for scale.

Usage: python scripts/harness_timing.py [n]   -> JSON lines
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path


ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import refc  # noqa: E402
from paper_1804_10120_b200 import bench as tb  # noqa: E402
from paper_1804_10120_b200 import tldf  # noqa: E402
from paper_1804_10120_b200.registry import Registry  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128**3


def main():
    work = Path(tempfile.mkdtemp(prefix="tlb_harness_"))
    prog, vs = tb.load(tb.CHRISTOFFEL)
    reg = Registry()
    for v in vs:
        reg.register(v)
    so = reg.build_shared(work / "b200")
    man = work / "b200" / "tloops_manifest.tsv"
    env = tb.make_env(prog, "Gamma", N, tb.DEFAULT_SEED, device="cpu")
    fin = work / "in.tldf"
    tldf.write(fin, env)
    harness = refc.REF_DIR / "tl_harness"
    compare = refc.REF_DIR / "tl_compare"
    runs = [("b200_pageable", so, man, {"TLB_HOST_REGISTER": "0"}),
            ("b200_registered", so, man, {"TLB_HOST_REGISTER": "1"}),
            ("reference_c", refc.REF_DIR / "c3_christoffel.so",
             refc.REF_DIR / "c3_christoffel.manifest.tsv", {})]
    outs = {}
    for name, lib, manifest, extra in runs:
        out = work / f"{name}.tldf"
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            res = subprocess.run([str(harness), str(lib), str(manifest), str(fin), str(out)],
                                 capture_output=True, text=True,
                                 env={**os.environ, **extra, "TLB_CACHE_DIR": str(work)})
            dt = time.perf_counter() - t0
            if res.returncode != 0:
                print(json.dumps({"run": name, "rc": res.returncode, "stderr": res.stderr[-500:]}))
                break
            best = dt if best is None else min(best, dt)
        outs[name] = out
        print(json.dumps({"run": name, "N": N, "harness_wall_s": best,
                          "fixture_MB": fin.stat().st_size / 1e6}), flush=True)
    for name in ("b200_pageable", "b200_registered"):
        res = subprocess.run([str(compare), "--bitwise", str(outs["reference_c"]),
                              str(outs[name])], capture_output=True, text=True)
        print(json.dumps({"compare": name, "vs": "reference_c", "bitwise_rc": res.returncode,
                          "out": (res.stdout + res.stderr)[-300:]}), flush=True)

    # the call alone, through the harness's own wiring (ctypes)
    import torch

    host = {k: f.data.numpy() for k, f in env.items()}
    ours = refc.RefProgram("c3", so_path=so, manifest_path=man)
    ref = refc.RefProgram("c3_christoffel")
    pinned = {k: torch.from_numpy(a).pin_memory().numpy() for k, a in host.items()}

    def per_call(go, reps=5):
        go()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            go()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    for name, prog_, arrays, extra, threads in (
            ("b200_call_pageable", ours, host, "0", 1),
            ("b200_call_registered", ours, host, "1", 1),
            ("b200_call_pinned", ours, pinned, "0", 1),
            ("reference_c_call_all_cores", ref, host, "0", os.cpu_count())):
        os.environ["TLB_HOST_REGISTER"] = extra  # read by libtlb200 at every staged run
        t = per_call(lambda: prog_.run(arrays, N, threads=threads))
        print(json.dumps({"run": name, "N": N, "s_per_call": t, "gridpoints_per_s": N / t,
                          "host_bytes_moved": 336 * N}), flush=True)


if __name__ == "__main__":
    main()
