"""In-tree build of libtlb200.so (nvcc, sm_100a) and kernel pre-compilation.

``build_library()`` compiles csrc/tlb_runtime.cpp (driver/NVRTC host
runtime, C-ABI of include/tlb200.h) and csrc/tlb_static.cu (statically
compiled sm_100a helper kernels) into ``paper_1804_10120_b200/libtlb200.so``.
``precompile(programs)`` JIT-compiles the fused kernels of the given
programs with NVRTC into the in-tree cubin cache (``_kcache/``) so a fresh
GPU box does not pay NVRTC latency on first use.  Neither step needs a GPU.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libtlb200.so"
GENCODE = "arch=compute_100a,code=sm_100a"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def build_library(force: bool = False, verbose: bool = False) -> Path:
    srcs = [CSRC / "tlb_runtime.cpp", CSRC / "tlb_static.cu"]
    deps = srcs + [ROOT / "include" / "tlb200.h"]
    if LIB.exists() and not force:
        newest = max(p.stat().st_mtime for p in deps)
        if LIB.stat().st_mtime >= newest:
            return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), "-std=c++17", "-O2", "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
           "-gencode", GENCODE, "-lineinfo", "-Xptxas", "-v",
           *[str(s) for s in srcs], "-o", str(tmp), "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"building libtlb200.so failed:\n{' '.join(cmd)}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, LIB)
    return LIB


def precompile(sources: dict[str, str]) -> dict[str, dict]:
    """NVRTC-compile every statement program of `sources` (name -> .tl text)
    as one fused program kernel and as per-statement kernels; returns
    per-program info (slots, bytes/point, cubin path)."""
    from .parser import parse_program
    from .ir import validate_statement
    from .lowering import lower_program
    from .runtime import Kernel, get_kernel

    out = {}
    for name, text in sources.items():
        res = parse_program(text)
        if res.diagnostics:
            raise RuntimeError(f"{name}: {res.diagnostics}")
        prog = res.program
        vs = [validate_statement(s, prog.decls) for s in prog.statements]
        try:
            plans = [lower_program(vs)] + ([lower_program([v]) for v in vs] if len(vs) > 1
                                           else [])
        except ArithmeticError:
            continue  # a literal `1/0` (raises at run time, like the reference): nothing to build
        for p in plans:
            k: Kernel = get_kernel(p)
        out[name] = {"slots": plans[0].n_slots, "bytes_per_point": plans[0].bytes_per_point,
                     "flops_per_point": plans[0].flops_per_point,
                     "cubin": str(get_kernel(plans[0]).cubin_path)}
    return out
