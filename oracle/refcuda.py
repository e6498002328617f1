"""Drive the reference's own emitted CUDA (the paper's GPU design) on the B200
— COMPARATOR INFRASTRUCTURE ONLY (scripts/compare_reference_design.py).

The reference emits, per statement, ``g_NNNN`` (one thread per (grid point,
LHS component), components reached through device pointer arrays,
pkg/src/tlang/codegen_cuda.py:135-180) and ``CUDAWrapper_g_NNNN`` (its fixed
launch geometry, codegen_cuda.py:182-204), wired into the bindings table
``tloops_entries`` (registry.py:183-270).  The emitted ``tl_call_NNNN``
passes its ``T[k]`` pointer arrays straight to the kernel, so here ``T[k]``
holds *device* pointer arrays (what the never-wired GPUPointers cache,
codegen_cuda.py:219-291, would have produced): ``flat[f] = base +
alias[f]*N`` uploaded once per field.  The kernels launch on the legacy
default stream.  A wrapper refuses N > 65535*blocksize_x
(codegen_cuda.py:187-189); callers keep N below that.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .refc import P_DOUBLE, P_P_DOUBLE, REF_DIR, TlEntry


def available(program: str) -> bool:
    return (REF_DIR / f"{program}_cuda.so").exists()


class RefCudaProgram:
    def __init__(self, program: str):
        so = REF_DIR / f"{program}_cuda.so"
        if not so.exists():
            raise FileNotFoundError(f"{so} missing: run python oracle/build_ref.py")
        self.lib = ctypes.CDLL(str(so))
        count = ctypes.c_int.in_dll(self.lib, "tloops_entry_count").value
        self.entries = (TlEntry * count).in_dll(self.lib, "tloops_entries")
        manifest = (REF_DIR / f"{program}.manifest.tsv").read_text().splitlines()
        self.order = [int(line.split("\t")[0]) for line in manifest if line.strip()]
        self.by_ordinal = {e.ordinal: e for e in self.entries}
        self._bound = None

    def bind(self, env: dict) -> None:
        """env: name -> CUDA float64 torch tensor, tensors (outer, inner, N)
        contiguous, scalars (N,).  Builds the device pointer arrays."""
        import torch

        calls = []
        keep = []
        for ordinal in self.order:
            e = self.by_ordinal[ordinal]
            tensors, scalars, numbers = [], [], []
            n = None
            for a in range(e.n_args):
                d = e.args[a]
                if d.kind == 3:
                    numbers.append(d.value)
                    continue
                t = env[d.name.decode()]
                n = t.shape[-1]
                if d.kind == 2:
                    scalars.append(ctypes.cast(t.data_ptr(), P_DOUBLE))
                    continue
                addrs = [t.data_ptr() + 8 * d.alias[f] * n for f in range(d.n_flat)]
                dev = torch.tensor(np.array(addrs, dtype=np.int64), device=t.device)
                keep.append(dev)
                tensors.append(ctypes.cast(dev.data_ptr(), P_P_DOUBLE))
            t_arr = (P_P_DOUBLE * max(1, len(tensors)))(*tensors)
            s_arr = (P_DOUBLE * max(1, len(scalars)))(*scalars)
            d_arr = (ctypes.c_double * max(1, len(numbers)))(*numbers)
            keep += [t_arr, s_arr, d_arr]
            calls.append((e.call, n, t_arr, s_arr, d_arr))
        self._bound = (calls, keep)

    def run(self) -> None:
        for call, n, t_arr, s_arr, d_arr in self._bound[0]:
            call(n, t_arr, s_arr, d_arr)
