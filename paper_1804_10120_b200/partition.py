"""Multi-GPU partitioner: grid points (or whole subdomains) across GPUs.

Every statement reads and writes only at its own grid point (derivatives are
precomputed inputs, reference evaluator.py:116-161), so a grid
splits into independent contiguous slabs, one per GPU, with no exchange on
the data path — the reference's "chunking is invisible" property
(test_evaluator.py:200-211) becomes "partitioning is invisible": the bits of
every slab equal the bits of a single-GPU run.

The only collective is optional: ``global_norm`` reduces one fp64 partial per
GPU with NCCL (8 bytes over NVLink) for monitoring-style diagnostics.
"""

from __future__ import annotations

from typing import Sequence


def slab_bounds(n_total: int, rank: int, world: int, align: int = 256) -> tuple[int, int]:
    """[lo, hi) of `rank`'s contiguous slab.  Interior boundaries are
    multiples of `align` points (keeps 128-bit accesses aligned); slabs
    differ by at most `align` points; an empty slab is possible when
    n_total < world*align."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if n_total < 0:
        raise ValueError("negative point count")
    units = -(-n_total // align)
    base, extra = divmod(units, world)
    lo_u = rank * base + min(rank, extra)
    hi_u = lo_u + base + (1 if rank < extra else 0)
    return min(lo_u * align, n_total), min(hi_u * align, n_total)


def all_slabs(n_total: int, world: int, align: int = 256) -> list[tuple[int, int]]:
    return [slab_bounds(n_total, r, world, align) for r in range(world)]


def domain_bounds(n_domains: int, rank: int, world: int) -> tuple[int, int]:
    """Whole subdomains per GPU for multi-domain batches (C4)."""
    return slab_bounds(n_domains, rank, world, 1)


def local_fields(program, n_total: int, rank: int, world: int, device=None,
                 align: int = 256) -> tuple[dict, tuple[int, int]]:
    """Allocate this rank's slab of every declared field (zero-filled)."""
    from .fields import ScalarField, TensorField

    lo, hi = slab_bounds(n_total, rank, world, align)
    env = {}
    for name, shape in program.decls.tensors.items():
        env[name] = TensorField(name, shape, hi - lo, device=device)
    for name in program.decls.scalar_fields:
        env[name] = ScalarField(name, hi - lo, device=device)
    return env, (lo, hi)


def global_norm(fields: Sequence, group=None) -> float:
    """sqrt(sum of squares) over the components of `fields` on every rank:
    a per-GPU fp64 partial, then one 8-byte all-reduce (NCCL for CUDA
    tensors, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    partial = None
    for f in fields:
        if f.data.numel() == 0:
            continue
        # one component array at a time (a dot product reduces in place: no
        # full-size temporary, which a 2^28-point Gamma could not afford)
        for row in f.data.to(torch.float64).reshape(-1, f.data.shape[-1]):
            s = torch.dot(row, row)
            partial = s if partial is None else partial + s
    if partial is None:  # no fields on this rank: a zero on the backend's device
        nccl = dist.is_available() and dist.is_initialized() and dist.get_backend(group) == "nccl"
        partial = torch.zeros((), dtype=torch.float64,
                              device="cuda" if nccl else "cpu")
    partial = partial.reshape(1)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return float(partial.sqrt().item())
