"""Parity at BASELINE.json's full sizes: whole-grid bitwise
checks where the oracle finishes in seconds (C1 64^3, C3 128^3, C4
512 x 16^3), slab-sampled bitwise checks where it cannot hold the grid (C2 at
10^8, C5 at 2^28: first, last and 16 random slabs of 2^12 points regenerated
on the host from the counter RNG)."""

import numpy as np
import pytest
import torch

from helpers import same_bits
from oracle import counter_rng, numpy_eval
from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200 import eval_batch, eval_program
from paper_1804_10120_b200.fields import ScalarField, TensorField
from paper_1804_10120_b200.runtime import fill_uniform

pytestmark = pytest.mark.gpu
SEED = 0xC0FFEE


def _host_env(prog, n, seed):
    return {k: f.data.cpu().numpy().copy() for k, f in tb.make_env(
        prog, "__none__", n, seed, device="cpu").items()}


@pytest.mark.parametrize("name,n", [("c1_dtg", 64**3), ("c3_christoffel", 128**3)])
def test_whole_grid_bitwise(name, n):
    prog, vs = tb.load(tb.PROGRAMS[name])
    targets = [v.stmt.lhs.field for v in vs]
    env = tb.make_env(prog, targets[0], n, SEED)  # the reference's exact inputs
    host = {k: f.data.cpu().numpy().copy() for k, f in env.items()}
    eval_program(vs, env)
    numpy_eval.eval_program(vs, host)
    for t in targets:
        assert same_bits(env[t].data.cpu().numpy(), host[t]), t


def test_c4_multidomain_batch_bitwise():
    prog, vs = tb.load(tb.P2)
    envs = [tb.make_env(prog, "Gamma", 16**3, SEED + d) for d in range(512)]
    for e in envs:
        e["dtg"].data.zero_()
    hosts = [{k: f.data.cpu().numpy().copy() for k, f in e.items()} for e in envs]
    eval_batch(vs, envs)
    for e, h in zip(envs, hosts):
        numpy_eval.eval_program(vs, h)
        for t in ("Gamma", "dtg"):
            assert same_bits(e[t].data.cpu().numpy(), h[t]), t


def _counter_env(prog, targets, n):
    env, sids = {}, {}
    for sid, it in enumerate(it for it in prog.items if getattr(it, "name", None) in
                             set(prog.decls.tensors) | prog.decls.scalar_fields):
        name = it.name
        if name in prog.decls.tensors:
            f = TensorField(name, prog.decls.tensors[name], n)
            comps = f.data.view(-1, n)
        else:
            f = ScalarField(name, n)
            comps = f.data.view(1, n)
        if name not in targets:
            for c in range(comps.shape[0]):
                fill_uniform(comps[c], SEED, (sid << 8) | c)
        env[name], sids[name] = f, sid
    return env, sids


def _slab_check(prog, vs, env, sids, n, slab=4096, count=16):
    rng = np.random.default_rng(1)
    starts = [0, n - slab] + list(rng.integers(0, n - slab, count))
    targets = {v.stmt.lhs.field for v in vs}
    for lo in starts:
        lo = int(lo)
        host = {}
        for name, f in env.items():
            shape = tuple(f.data.shape[:-1]) + (slab,)
            if name in targets:
                host[name] = np.zeros(shape)
                continue
            ncomp = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
            vals = np.stack([counter_rng.uniform(SEED, (sids[name] << 8) | c, lo, slab)
                             for c in range(ncomp)])
            host[name] = vals.reshape(shape)
        numpy_eval.eval_program(vs, host)
        for t in targets:
            got = env[t].data[..., lo:lo + slab].cpu().numpy()
            assert same_bits(got, host[t]), (t, lo)


def test_c5_p2_at_2e28_slab_sampled():
    torch.cuda.empty_cache()
    n = 1 << 28
    prog, vs = tb.load(tb.P2)
    env, sids = _counter_env(prog, {"Gamma", "dtg"}, n)
    eval_program(vs, env)
    torch.cuda.synchronize()
    _slab_check(prog, vs, env, sids, n)
    del env
    torch.cuda.empty_cache()


def test_c2_maxwell_at_1e8_slab_sampled():
    torch.cuda.empty_cache()
    n = 10**8
    prog, vs = tb.load(tb.MAXWELL)
    env, sids = _counter_env(prog, {v.stmt.lhs.field for v in vs}, n)
    eval_program(vs, env)
    torch.cuda.synchronize()
    _slab_check(prog, vs, env, sids, n)
    del env
    torch.cuda.empty_cache()
