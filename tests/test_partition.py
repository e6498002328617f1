"""Multi-GPU partition logic on CPU: slab arithmetic, and a world_size-2
gloo run showing the sharded grid covers every point exactly once and the
optional global-norm collective reduces correctly (the data path has no
collective)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_10120_b200.partition import all_slabs, domain_bounds


@pytest.mark.parametrize("n", [0, 1, 255, 256, 257, 1000, 1 << 20, (1 << 28) + 3])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_slabs_tile_the_grid(n, world):
    slabs = all_slabs(n, world)
    assert slabs[0][0] == 0 and slabs[-1][1] == n
    for (a, b), (c, d) in zip(slabs, slabs[1:]):
        assert b == c and a <= b
        assert b % 256 == 0 or b == n
    sizes = [b - a for a, b in slabs]
    assert max(sizes) - min(sizes) <= 2 * 256 or n < 256 * world


def test_domains_split_whole():
    got = [domain_bounds(512, r, 8) for r in range(8)]
    assert got[0] == (0, 64) and got[-1] == (448, 512)


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1804_10120_b200.bench import P2, load
    from paper_1804_10120_b200.partition import global_norm, local_fields
    from oracle import counter_rng, numpy_eval

    prog, vs = load(P2)
    env, (lo, hi) = local_fields(prog, n, rank, world, device="cpu")
    host = {}
    for sid, name in enumerate(list(prog.decls.tensors) + sorted(prog.decls.scalar_fields)):
        f = env[name]
        if name in ("Gamma", "dtg"):
            host[name] = f.data.numpy().copy()
            continue
        flat = f.data.view(-1, hi - lo)
        for c in range(flat.shape[0]):
            flat[c] = torch.from_numpy(counter_rng.uniform(7, (sid << 8) | c, lo, hi - lo))
        host[name] = f.data.numpy().copy()
    numpy_eval.eval_program(vs, host)  # CPU stand-in for the per-rank kernel
    for name in ("Gamma", "dtg"):
        env[name].data.copy_(torch.from_numpy(host[name]))
    norm = global_norm([env["Gamma"], env["dtg"]])
    cover = torch.zeros(n, dtype=torch.int64)
    cover[lo:hi] += 1
    dist.all_reduce(cover)
    out[rank] = (norm, int(cover.min()), int(cover.max()), hi - lo)
    dist.destroy_process_group()


def test_two_rank_gloo_partition_and_norm():
    n = 3000
    port = 29500 + os.getpid() % 2000
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, n, out), nprocs=2, join=True)
        res = dict(out)
    (n0, lo0, hi0, s0), (n1, lo1, hi1, s1) = res[0], res[1]
    assert n0 == pytest.approx(n1, rel=0, abs=0)
    assert (lo0, hi0, lo1, hi1) == (1, 1, 1, 1)  # every point owned exactly once
    assert s0 + s1 == n
    # single-process reference of the same norm
    from paper_1804_10120_b200.bench import P2, load
    from oracle import counter_rng, numpy_eval

    prog, vs = load(P2)
    host = {}
    for sid, name in enumerate(list(prog.decls.tensors) + sorted(prog.decls.scalar_fields)):
        if name in prog.decls.tensors:
            s = prog.decls.tensors[name]
            shape = (s.outer_count, s.inner_count, n)
        else:
            shape = (n,)
        if name in ("Gamma", "dtg"):
            host[name] = np.zeros(shape)
            continue
        flat = np.stack([counter_rng.uniform(7, (sid << 8) | c, 0, n)
                         for c in range(int(np.prod(shape[:-1])) if len(shape) > 1 else 1)])
        host[name] = flat.reshape(shape)
    numpy_eval.eval_program(vs, host)
    want = np.sqrt((host["Gamma"] ** 2).sum() + (host["dtg"] ** 2).sum())
    assert n0 == pytest.approx(want, rel=1e-12)


def test_batch_subdomains_grouped_per_device():
    # eval_batch issues one batched launch per GPU of the process; the
    # grouping keeps first-appearance order and each device's domain order
    from collections import namedtuple
    from types import SimpleNamespace

    from paper_1804_10120_b200.evaluator import _device_groups

    Dev = namedtuple("Dev", "type index")  # hashable like torch.device

    def env(dev):
        dv = Dev("cuda", dev) if dev is not None else Dev("cpu", None)
        return {"T": SimpleNamespace(data=SimpleNamespace(device=dv))}

    v = SimpleNamespace(stmt=SimpleNamespace(lhs=SimpleNamespace(field="T")))
    envs = [env(1), env(0), env(1), env(None), env(0)]
    groups = _device_groups([v], envs)
    assert list(groups.values()) == [[0, 2], [1, 4], [3]]
    assert len(_device_groups([v], [env(0), env(0)])) == 1
