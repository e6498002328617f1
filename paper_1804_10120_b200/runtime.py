"""ctypes binding of libtlb200.so (include/tlb200.h) and the kernel cache.

The shared library is built in-tree by ``paper_1804_10120_b200.build`` and
loaded from this package directory.  There is no fallback: if the library
or NVRTC or the GPU is missing, the calls below raise ``TlbError``.
"""

from __future__ import annotations

import atexit
import ctypes
import hashlib
import os
import threading
from collections import OrderedDict
from pathlib import Path
from typing import Sequence

from .lowering import KernelPlan

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libtlb200.so"
DEFAULT_CACHE_DIR = PKG_DIR / "_kcache"

ARCH = "sm_100a"
BASE_OPTIONS = (
    f"--gpu-architecture={ARCH}",
    "--fmad=false",  # bit-exact parity: no DFMA contraction
    "--prec-div=true",
    "--prec-sqrt=true",
    "-std=c++17",
    "-lineinfo",
)

EXPORTED = (
    "tlb_abi_version", "tlb_init", "tlb_last_error", "tlb_nvrtc_version", "tlb_device_sm_count",
    "tlb_compile", "tlb_kernel_log", "tlb_kernel_cubin", "tlb_kernel_destroy",
    "tlb_kernel_set_slots", "tlb_kernel_attrs", "tlb_launch", "tlb_launch_default",
    "tlb_batch_create",
    "tlb_batch_launch", "tlb_batch_destroy", "tlb_exec_host", "tlb_fill_uniform",
    "tlb_fp64_probe",
    "tlb_harness_call", "tlb_release_staging",
)


class TlbError(RuntimeError):
    """A libtlb200 call failed (message from tlb_last_error)."""


_lib = None
_lib_lock = threading.Lock()
_exiting = False


def _at_exit() -> None:
    # the CUDA context may already be gone at interpreter shutdown: modules
    # are released with the process there, not one by one
    global _exiting
    _exiting = True


atexit.register(_at_exit)

c_ll = ctypes.c_longlong
c_vp = ctypes.c_void_p
c_int = ctypes.c_int


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise TlbError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(str(LIB_PATH))
            sig = {
                "tlb_abi_version": (c_int, []),
                "tlb_init": (c_int, [c_int]),
                "tlb_last_error": (ctypes.c_char_p, []),
                "tlb_nvrtc_version": (c_int, [ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
                "tlb_device_sm_count": (c_int, [ctypes.POINTER(c_int)]),
                "tlb_compile": (c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p), c_int,
                                        ctypes.c_char_p, ctypes.POINTER(c_vp)]),
                "tlb_kernel_log": (ctypes.c_char_p, [c_vp]),
                "tlb_kernel_cubin": (c_int, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_ll)]),
                "tlb_kernel_destroy": (None, [c_vp]),
                "tlb_kernel_set_slots": (c_int, [c_vp, c_int, c_int, ctypes.POINTER(c_int),
                                                 ctypes.POINTER(c_ll), ctypes.POINTER(c_int)]),
                "tlb_kernel_attrs": (c_int, [c_vp, ctypes.c_char_p, ctypes.POINTER(c_int),
                                             ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
                "tlb_launch": (c_int, [c_vp, c_ll, ctypes.POINTER(c_vp), ctypes.POINTER(c_ll),
                                       c_int, c_int, c_ll, c_vp]),
                "tlb_launch_default": (c_int, [c_vp, c_ll, ctypes.POINTER(c_vp),
                                               ctypes.POINTER(c_ll), c_vp]),
                "tlb_batch_create": (c_int, [c_vp, c_int, ctypes.POINTER(c_vp),
                                             ctypes.POINTER(c_ll), ctypes.POINTER(c_ll), c_vp,
                                             ctypes.POINTER(c_vp)]),
                "tlb_batch_launch": (c_int, [c_vp, c_int, c_int, c_vp]),
                "tlb_batch_destroy": (None, [c_vp]),
                "tlb_exec_host": (c_int, [c_vp, c_ll, ctypes.POINTER(ctypes.POINTER(c_vp)),
                                          c_ll, c_vp]),
                "tlb_fill_uniform": (c_int, [c_vp, c_ll, ctypes.c_ulonglong, ctypes.c_ulonglong,
                                             c_ll, c_vp]),
                "tlb_release_staging": (c_int, []),
                "tlb_fp64_probe": (c_int, [c_vp, c_int, c_int, c_vp]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().tlb_last_error().decode(errors="replace")
        raise TlbError(f"{what}: {msg}" if what else msg)


def nvrtc_version() -> tuple[int, int]:
    a, b = c_int(), c_int()
    check(lib().tlb_nvrtc_version(ctypes.byref(a), ctypes.byref(b)), "nvrtc version")
    return a.value, b.value


def compile_options() -> list[str]:
    # the block size (TLK_THREADS) is part of the source: lowering.Variant.threads
    opts = list(BASE_OPTIONS)
    extra = os.environ.get("TLK_DEFINES", "").split()
    opts += extra
    return opts


def cache_dir() -> Path:
    d = Path(os.environ.get("TLB_CACHE_DIR", str(DEFAULT_CACHE_DIR)))
    try:
        d.mkdir(parents=True, exist_ok=True)
    except OSError:
        pass
    return d


def _arr(ctype, values):
    return (ctype * len(values))(*values)


# ------------------------------------------------------- graph capture pins
# A CUDA graph bakes in kernel handles and batch-table addresses.  While a
# pin scope is open on this thread (evaluator.capture_graph), every Kernel
# and Batch that launches is recorded, and the graph keeps that list, so
# neither the module nor the table can be freed under a later replay.

_pins = threading.local()


class pin_scope:
    def __enter__(self) -> list:
        self.prev = getattr(_pins, "cur", None)
        _pins.cur = []
        return _pins.cur

    def __exit__(self, *exc) -> None:
        _pins.cur = self.prev


_launch_count = [0]


def _pin(obj) -> None:
    _launch_count[0] += 1
    cur = getattr(_pins, "cur", None)
    if cur is not None:
        cur.append(obj)


class Kernel:
    """A compiled fused kernel (cubin + slot map); modules load per context."""

    def __init__(self, plan: KernelPlan, options: Sequence[str] | None = None):
        self.plan = plan
        self.options = list(options) if options is not None else compile_options()
        L = lib()
        maj, mnr = nvrtc_version()
        h = hashlib.sha256()
        h.update(plan.source.encode())
        h.update("\0".join(self.options).encode())
        h.update(f"nvrtc{maj}.{mnr}".encode())
        self.cache_key = h.hexdigest()
        path = cache_dir() / f"{self.cache_key}.cubin"
        opts = _arr(ctypes.c_char_p, [o.encode() for o in self.options])
        handle = c_vp()
        check(L.tlb_compile(plan.source.encode(), opts, len(self.options), str(path).encode(),
                            ctypes.byref(handle)), "tlb_compile")
        self.handle = handle
        self.cubin_path = path
        check(L.tlb_kernel_set_slots(handle, len(plan.fields), plan.n_slots,
                                     _arr(c_int, plan.slot_field), _arr(c_ll, plan.slot_comp),
                                     _arr(c_int, plan.slot_flags)), "tlb_kernel_set_slots")
        self.nfields = len(plan.fields)
        self.launches = 0
        var = plan.variant
        # block size = the compiled TLK_THREADS; grid = one wave unless the
        # variant asks for more (lowering.choose_variant / TLK_WAVES)
        self.threads = var.threads if var is not None else 256
        self.max_blocks = 0
        # vec 2 = auto (128-bit when every slot is 16-byte aligned), 1 = forced
        # scalar, 3 = the TMA-staged entry
        self.vec = 1 if (var is not None and var.vec == 1) else 0
        if var is not None and var.stage:
            self.vec = 3  # the staged entry (its tile ring size is read from the source)
        if var is not None and self.max_blocks == 0:
            self.max_blocks = _grid_cap(var.waves)
        # batch entry: 0 = 2-point when aligned, 1 = 1-point, 3 = TMA-staged
        self.batch_vec = 1 if (var is not None and var.batch_vec == 1) else 0
        if var is not None and var.batch_vec == 3:
            self.batch_vec = 3 if var.stage else 1
        self.batch_threads = (var.batch_threads if var is not None and var.batch_threads
                              else self.threads)
        # size class (Variant.small_class): launches of <= small_n points run
        # `small` (a second cubin when the code differs, else this one) with
        # its own vec/waves; set by get_kernel
        self.small_n = 0
        self.small: "Kernel | None" = None
        self.small_vec, self.small_max_blocks = self.vec, self.max_blocks

    def _attach_small(self, small_n: int, sv, small: "Kernel | None") -> None:
        self.small_n = small_n
        self.small = small
        self.small_vec = 1 if sv.vec == 1 else 0
        self.small_max_blocks = _grid_cap(sv.waves)

    @property
    def log(self) -> str:
        return lib().tlb_kernel_log(self.handle).decode(errors="replace")

    def cubin(self) -> bytes:
        p, n = c_vp(), c_ll()
        check(lib().tlb_kernel_cubin(self.handle, ctypes.byref(p), ctypes.byref(n)))
        return ctypes.string_at(p.value, n.value)

    def attrs(self, entry: str = "tlk_flat_v2") -> dict:
        r, lb, mt = c_int(), c_int(), c_int()
        check(lib().tlb_kernel_attrs(self.handle, entry.encode(), ctypes.byref(r),
                                     ctypes.byref(lb), ctypes.byref(mt)), "tlb_kernel_attrs")
        return {"registers": r.value, "local_bytes": lb.value, "max_threads": mt.value}

    def launch(self, n: int, bases: Sequence[int], pitches: Sequence[int], stream: int,
               vec: int | None = None, threads: int | None = None,
               max_blocks: int | None = None) -> None:
        handle = self.handle
        if n <= self.small_n and vec is None and max_blocks is None:
            handle = (self.small or self).handle
            vec, max_blocks = self.small_vec, self.small_max_blocks
        vec = self.vec if vec is None else vec
        threads = self.threads if threads is None else threads
        max_blocks = self.max_blocks if max_blocks is None else max_blocks
        check(lib().tlb_launch(handle, n, _arr(c_vp, bases), _arr(c_ll, pitches), vec,
                               threads, max_blocks, stream), "tlb_launch")
        self.launches += 1
        _pin(self)

    def launch_arrays(self, n: int, bases, pitches, stream: int) -> None:
        """Launch with prebuilt ctypes address arrays (bound-launch fast path)."""
        if n <= self.small_n:
            rc = _lib.tlb_launch((self.small or self).handle, n, bases, pitches, self.small_vec,
                                 self.threads, self.small_max_blocks, stream)
        else:
            rc = _lib.tlb_launch(self.handle, n, bases, pitches, self.vec, self.threads,
                                 self.max_blocks, stream)
        if rc:
            check(rc, "tlb_launch")
        self.launches += 1
        _pin(self)

    def __del__(self):
        # unloads the module from every context it was loaded into (after
        # the context's pending work); evicted kernels only ever reach this
        # once nothing — plan cache, bound launch, batch, graph — holds them
        try:
            if getattr(self, "handle", None) and _lib is not None and not _exiting:
                _lib.tlb_kernel_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def exec_host(self, n: int, comp_ptrs: Sequence[Sequence[int]], stream: int,
                  slab: int = 0) -> None:
        if not slab:  # tuning: TLB_HOST_SLAB points per pipeline stage (0 = the runtime's)
            slab = int(os.environ.get("TLB_HOST_SLAB", "0"))
        rows = [_arr(c_vp, list(r)) for r in comp_ptrs]
        outer = (ctypes.POINTER(c_vp) * len(rows))(
            *[ctypes.cast(r, ctypes.POINTER(c_vp)) for r in rows])
        check(lib().tlb_exec_host(self.handle, n, outer, slab, stream), "tlb_exec_host")
        self.launches += 1
        _pin(self)


# tlb_launch's max_blocks for a one-shot grid: a cap no launch reaches, so the
# grid is one block per `threads` points (pairs) — the runtime clamps it to
# the 2^31-1 grid limit, beyond which the grid-stride loop covers the rest
ONE_SHOT = 1 << 62


def _grid_cap(waves: int) -> int:
    """tlb_launch max_blocks for Variant.waves: 0 one-shot, 1 one wave at
    occupancy, w > 1 w waves."""
    if waves == 0:
        return ONE_SHOT
    return -waves if waves > 1 else 0


def address_arrays(bases: Sequence[int], pitches: Sequence[int]):
    return _arr(c_vp, list(bases)), _arr(c_ll, list(pitches))


class Batch:
    """Uploaded multi-domain table for one kernel (tlb_batch_*)."""

    def __init__(self, kernel: Kernel, bases: Sequence[Sequence[int]],
                 pitches: Sequence[Sequence[int]], ns: Sequence[int], stream: int):
        self.kernel = kernel
        flat_b = [b for row in bases for b in row]
        flat_p = [p for row in pitches for p in row]
        h = c_vp()
        check(lib().tlb_batch_create(kernel.handle, len(ns), _arr(c_vp, flat_b),
                                     _arr(c_ll, flat_p), _arr(c_ll, list(ns)), stream,
                                     ctypes.byref(h)),
              "tlb_batch_create")
        self.handle = h
        self.ndom = len(ns)

    def launch(self, stream: int, threads: int | None = None) -> None:
        threads = self.kernel.batch_threads if threads is None else threads
        check(lib().tlb_batch_launch(self.handle, self.kernel.batch_vec, threads, stream),
              "tlb_batch_launch")
        self.kernel.launches += 1
        _pin(self)

    def __del__(self):
        try:
            if self.handle and _lib is not None and not _exiting:
                _lib.tlb_batch_destroy(self.handle)
        except Exception:
            pass


KERNEL_CACHE_SIZE = 256
_kernels: "OrderedDict[str, Kernel]" = OrderedDict()
_kernels_lock = threading.Lock()


def get_kernel(plan: KernelPlan) -> Kernel:
    """Compiled kernel for `plan`, cached in memory by source (LRU, at most
    KERNEL_CACHE_SIZE; on disk by source + options + NVRTC version)."""
    key = plan.key + "|" + " ".join(compile_options())
    with _kernels_lock:
        k = _kernels.get(key)
        if k is not None:
            _kernels.move_to_end(key)
            return k
        k = Kernel(plan)
        if plan.small_variant is not None:
            small = Kernel(plan.small_plan) if plan.small_plan is not None else None
            k._attach_small(plan.variant.small_n, plan.small_variant, small)
        _kernels[key] = k
        while len(_kernels) > KERNEL_CACHE_SIZE:
            _kernels.popitem(last=False)
    return k


def all_kernels() -> list[Kernel]:
    with _kernels_lock:
        return list(_kernels.values())


def total_launches() -> int:
    """Fused-kernel launches (plain, staged, batched, host-staged) issued by
    this process so far, whichever kernel objects are still cached."""
    return _launch_count[0]


def release_staging() -> None:
    """Free the device staging buffers used for host-resident fields."""
    check(lib().tlb_release_staging(), "tlb_release_staging")


def fill_uniform(t, seed: int, stream_id: int, offset: int = 0, stream: int | None = None):
    """Fill a contiguous CUDA float64 tensor with counter-based uniform [0,1)
    values (tlb_fill_uniform; host twin: oracle/counter_rng.py)."""
    import torch

    assert t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
    if stream is None:
        stream = torch.cuda.current_stream(t.device).cuda_stream
    with torch.cuda.device(t.device):
        check(lib().tlb_fill_uniform(t.data_ptr(), t.numel(), seed, stream_id, offset, stream),
              "tlb_fill_uniform")


def fp64_peak_gflops(iters: int = 4096, reps: int = 5) -> float:
    """Measured uncontracted fp64 throughput (DMUL + DADD, GFLOP/s) of the
    current device: the flop side of the roofline (tlb_fp64_probe)."""
    import torch

    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(out.device).multi_processor_count
    blocks = sms * 8
    stream = torch.cuda.current_stream().cuda_stream
    check(lib().tlb_fp64_probe(out.data_ptr(), blocks, 64, stream), "tlb_fp64_probe")
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        check(lib().tlb_fp64_probe(out.data_ptr(), blocks, iters, stream), "tlb_fp64_probe")
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return blocks * 256 * iters * 16 / best / 1e9
