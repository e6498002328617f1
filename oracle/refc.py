"""Run the reference's own compiled C kernels (oracle/_ref/<program>.so) —
TEST/BASELINE INFRASTRUCTURE ONLY (bench.py cpu_baseline, --impl reference).

Binds the emitted bindings table exactly as the reference harness does
(pkg/harness/tl_harness.c:24-48 struct mirror, :113-124 dlsym,
:188-217 argument wiring): per tensor argument a flattened aliased pointer
array ``flat[f] = data + alias[f]*N`` (symmetric images share a buffer),
scalar fields by pointer, numbers by value, then ``entry->call(N, T, S, D)``
for every manifest entry in order.

Parallel execution follows BASELINE.md §2: each statement's grid is split
into contiguous slabs by pointer offset, one thread per host core (ctypes
releases the GIL during the foreign call), statements one after another.
"""

from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

REF_DIR = Path(__file__).resolve().parent / "_ref"

c_long, c_int, c_double = ctypes.c_long, ctypes.c_int, ctypes.c_double
P_DOUBLE = ctypes.POINTER(c_double)
P_P_DOUBLE = ctypes.POINTER(P_DOUBLE)


class TlArgDesc(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("kind", c_int), ("dim", c_int),
                ("outer_rank", c_int), ("inner_rank", c_int), ("n_outer_pairs", c_int),
                ("outer_pairs", ctypes.POINTER(ctypes.c_ubyte)), ("n_inner_pairs", c_int),
                ("inner_pairs", ctypes.POINTER(ctypes.c_ubyte)), ("n_components", c_long),
                ("n_flat", c_long), ("alias", ctypes.POINTER(c_long)), ("value", c_double)]


CALL = ctypes.CFUNCTYPE(None, c_long, ctypes.POINTER(P_P_DOUBLE), ctypes.POINTER(P_DOUBLE),
                        P_DOUBLE)


class TlEntry(ctypes.Structure):
    _fields_ = [("ordinal", c_int), ("signature", ctypes.c_char_p), ("n_args", c_int),
                ("args", ctypes.POINTER(TlArgDesc)), ("call", CALL)]


def available(program: str) -> bool:
    return (REF_DIR / f"{program}.so").exists()


class RefProgram:
    """One compiled reference program (all its statements, manifest order)."""

    def __init__(self, program: str, so_path=None, manifest_path=None):
        """``program``'s compiled reference C (oracle/_ref/<program>.so), or
        any .so exporting the same bindings table (``so_path`` +
        ``manifest_path``, e.g. the b200 bindings of registry.build_shared)."""
        so = Path(so_path) if so_path else REF_DIR / f"{program}.so"
        if not so.exists():
            raise FileNotFoundError(f"{so} missing: run python oracle/build_ref.py")
        self.lib = ctypes.CDLL(str(so))
        count = c_int.in_dll(self.lib, "tloops_entry_count").value
        self.entries = (TlEntry * count).in_dll(self.lib, "tloops_entries")
        man = Path(manifest_path) if manifest_path else REF_DIR / f"{program}.manifest.tsv"
        manifest = man.read_text().splitlines()
        self.order = [int(line.split("\t")[0]) for line in manifest if line.strip()]
        self.by_ordinal = {e.ordinal: e for e in self.entries}

    def run(self, env: dict, n: int, threads: int | None = None, min_slab: int = 1024) -> None:
        """Execute every manifest entry over ``env`` (name -> float64 numpy
        array, tensors (outer, inner, N) C-contiguous, scalars (N,))."""
        threads = threads or os.cpu_count() or 1
        slabs = _slabs(n, threads, min_slab)
        pool = ThreadPoolExecutor(max_workers=len(slabs)) if len(slabs) > 1 else None
        try:
            for ordinal in self.order:
                entry = self.by_ordinal[ordinal]
                calls = [self._bind(entry, env, lo, hi) for lo, hi in slabs]
                if pool is None:
                    for c in calls:
                        c()
                else:
                    list(pool.map(lambda c: c(), calls))
        finally:
            if pool is not None:
                pool.shutdown()

    def slab_runner(self, env: dict, n: int, threads: int, min_slab: int = 1024):
        """A callable running every entry over ``env`` split into per-thread
        slabs (as ``run``), with all pointer tables bound once up front so
        that repeated calls time only the kernels."""
        slabs = _slabs(n, threads, min_slab)
        calls = [[self._bind(self.by_ordinal[o], env, lo, hi) for lo, hi in slabs]
                 for o in self.order]
        pool = ThreadPoolExecutor(max_workers=len(slabs)) if len(slabs) > 1 else None

        def go():
            for per_entry in calls:
                if pool is None:
                    for c in per_entry:
                        c()
                else:
                    list(pool.map(lambda c: c(), per_entry))

        return go

    def domain_runner(self, envs: list, threads: int):
        """A callable running the program over many subdomains, one task per
        subdomain (its entries in manifest order) on ``threads`` workers —
        how a multi-domain CPU code parallelises (multi-domain
        loops live outside TLoops)."""
        tasks = []
        for env in envs:
            npts = next(iter(env.values())).shape[-1]
            tasks.append([self._bind(self.by_ordinal[o], env, 0, npts) for o in self.order])
        pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None

        def one(task):
            for c in task:
                c()

        def go():
            if pool is None:
                for t in tasks:
                    one(t)
            else:
                list(pool.map(one, tasks))

        return go

    def _bind(self, entry: TlEntry, env: dict, lo: int, hi: int):
        tensors, scalars, numbers, keep = [], [], [], []
        for a in range(entry.n_args):
            d = entry.args[a]
            name = d.name.decode()
            if d.kind == 3:
                numbers.append(d.value)
                continue
            arr = env[name]
            assert arr.dtype == np.float64 and arr.flags.c_contiguous, name
            base = arr.ctypes.data
            npts = arr.shape[-1]
            if d.kind == 2:
                scalars.append(ctypes.cast(base + 8 * lo, P_DOUBLE))
                continue
            flat = (P_DOUBLE * d.n_flat)(*[
                ctypes.cast(base + 8 * (d.alias[f] * npts + lo), P_DOUBLE)
                for f in range(d.n_flat)])
            keep.append(flat)
            tensors.append(ctypes.cast(flat, P_P_DOUBLE))
        t_arr = (P_P_DOUBLE * max(1, len(tensors)))(*tensors)
        s_arr = (P_DOUBLE * max(1, len(scalars)))(*scalars)
        d_arr = (c_double * max(1, len(numbers)))(*numbers)
        keep += [t_arr, s_arr, d_arr]
        call, count = entry.call, hi - lo

        def go(keep=keep):
            call(count, t_arr, s_arr, d_arr)

        return go


def _slabs(n: int, parts: int, min_slab: int = 1024) -> list[tuple[int, int]]:
    parts = max(1, min(parts, n // min_slab or 1))
    step = -(-n // parts)
    return [(lo, min(lo + step, n)) for lo in range(0, n, step)]
