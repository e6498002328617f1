"""The N>1 path on the one GPU a test box has: two ranks (processes) share
cuda:0 over a gloo process group, each evaluating its own slab (or its own
whole subdomains) exactly as bench.py does under torchrun.  Partitioning
must be invisible in the bits (the reference's "chunking is invisible",
pkg/tests/test_evaluator.py:200-211, across processes — SURVEY.md 8e), and
the optional global-norm collective runs over NCCL at world size 1."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import same_bits

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
SEED = 0x5EED


def _fill_env(prog, env, lo, hi):
    """Inputs keyed by GLOBAL point index (counter RNG), targets zeroed."""
    from paper_1804_10120_b200.runtime import fill_uniform

    targets = {"Gamma", "dtg"}
    names = list(prog.decls.tensors) + sorted(prog.decls.scalar_fields)
    for sid, name in enumerate(names):
        f = env[name]
        if name in targets:
            f.data.zero_()
            continue
        flat = f.data.view(-1, hi - lo)
        for c in range(flat.shape[0]):
            fill_uniform(flat[c], SEED, (sid << 8) | c, offset=lo)


def _rank_worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1804_10120_b200 import eval_batch, eval_program
    from paper_1804_10120_b200.bench import P2, load
    from paper_1804_10120_b200.partition import domain_bounds, global_norm, local_fields

    prog, vs = load(P2)
    env, (lo, hi) = local_fields(prog, n, rank, world, device="cuda")
    _fill_env(prog, env, lo, hi)
    eval_program(vs, env)
    torch.cuda.synchronize()
    norm = global_norm([env["Gamma"], env["dtg"]])  # gloo: host partials
    res = {"slab": (lo, hi), "norm": norm,
           "Gamma": env["Gamma"].data.cpu().numpy(), "dtg": env["dtg"].data.cpu().numpy()}
    # C4-style: whole subdomains per rank, one batched launch each
    d0, d1 = domain_bounds(12, rank, world)
    doms = []
    for d in range(d0, d1):
        e, _ = local_fields(prog, 4096, 0, 1, device="cuda")
        _fill_env(prog, e, d * 4096, (d + 1) * 4096)
        doms.append(e)
    eval_batch(vs, doms)
    torch.cuda.synchronize()
    res["domains"] = (d0, d1)
    res["dom_Gamma"] = [e["Gamma"].data.cpu().numpy() for e in doms]
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_partition_is_invisible():
    from oracle import counter_rng, numpy_eval
    from paper_1804_10120_b200 import eval_batch, eval_program
    from paper_1804_10120_b200.bench import P2, load
    from paper_1804_10120_b200.partition import local_fields

    n = 300_001  # odd: the second slab is ragged
    port = 29600 + os.getpid() % 2000
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        mp.start_processes(_rank_worker, args=(2, port, n, out), nprocs=2, join=True,
                           start_method="spawn")
        res = dict(out)
    prog, vs = load(P2)
    # one rank over the whole grid
    env, _ = local_fields(prog, n, 0, 1, device="cuda")
    _fill_env(prog, env, 0, n)
    eval_program(vs, env)
    whole = {t: env[t].data.cpu().numpy() for t in ("Gamma", "dtg")}
    assert res[0]["slab"][0] == 0 and res[0]["slab"][1] == res[1]["slab"][0]
    assert res[1]["slab"][1] == n
    for r in (0, 1):
        lo, hi = res[r]["slab"]
        for t in ("Gamma", "dtg"):
            assert same_bits(res[r][t], whole[t][..., lo:hi]), (r, t)
    # the oracle on a window straddling the slab boundary
    cut = res[0]["slab"][1]
    lo, hi = cut - 300, cut + 300
    host = {}
    names = list(prog.decls.tensors) + sorted(prog.decls.scalar_fields)
    for sid, name in enumerate(names):
        if name in prog.decls.tensors:
            s = prog.decls.tensors[name]
            shape = (s.outer_count, s.inner_count, hi - lo)
        else:
            shape = (hi - lo,)
        if name in ("Gamma", "dtg"):
            host[name] = np.zeros(shape)
            continue
        k = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
        host[name] = np.stack([counter_rng.uniform(SEED, (sid << 8) | c, lo, hi - lo)
                               for c in range(k)]).reshape(shape)
    numpy_eval.eval_program(vs, host)
    for t in ("Gamma", "dtg"):
        got = np.concatenate([res[0][t][..., lo:], res[1][t][..., :hi - cut]], axis=-1)
        assert same_bits(got, host[t]), t
    # both ranks agree on the global norm, and it is the whole grid's
    want = float(np.sqrt((whole["Gamma"] ** 2).sum() + (whole["dtg"] ** 2).sum()))
    assert res[0]["norm"] == res[1]["norm"]
    assert res[0]["norm"] == pytest.approx(want, rel=1e-12)
    # subdomains split across ranks == all subdomains in one batched launch
    doms = []
    for d in range(12):
        e, _ = local_fields(prog, 4096, 0, 1, device="cuda")
        _fill_env(prog, e, d * 4096, (d + 1) * 4096)
        doms.append(e)
    eval_batch(vs, doms)
    for r in (0, 1):
        d0, d1 = res[r]["domains"]
        for k, d in enumerate(range(d0, d1)):
            assert same_bits(res[r]["dom_Gamma"][k], doms[d]["Gamma"].data.cpu().numpy())


def _nccl_worker(rank, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_1804_10120_b200.fields import TensorField
    from paper_1804_10120_b200.partition import global_norm
    from paper_1804_10120_b200.symmetry import SymmetrySpec
    from paper_1804_10120_b200.fields import TensorShape

    f = TensorField("g", TensorShape(3, 2, SymmetrySpec(((0, 1),))), 1000)
    f.data.copy_(torch.arange(f.data.numel(), dtype=torch.float64).view_as(f.data))
    out["norm"] = global_norm([f])
    out["backend"] = dist.get_backend()
    out["want"] = float(torch.sqrt((f.data ** 2).sum()).item())
    dist.destroy_process_group()


def test_global_norm_over_nccl_world_size_one():
    port = 31600 + os.getpid() % 2000
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        mp.start_processes(_nccl_worker, args=(port, out), nprocs=1, join=True,
                           start_method="spawn")
        res = dict(out)
    assert res["backend"] == "nccl"
    assert res["norm"] == pytest.approx(res["want"], rel=1e-15)


def test_bench_line_at_two_ranks_on_one_gpu():
    # the driver's N>1 launch (torchrun, one process per rank), with both
    # ranks mapped to cuda:0 over gloo: the full line, cpu_baseline included
    port = 32600 + os.getpid() % 2000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--gpus", "2", "--points", str(1 << 22), "--steps", "3", "--warmup", "3",
           "--dist-backend", "gloo", "--same-device", "--no-e2e", "--no-configs",
           "--cpu-sample", "65536", "--cpu-seconds", "0.5"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpu_launches"] == 6  # 3 steps x 2 ranks
    assert d["config"]["points_per_gpu"] == 1 << 21
    assert d["cpu_baseline"]["value"] > 0
