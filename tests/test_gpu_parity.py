"""Device parity: the fused sm_100a kernels against the reference's own
outputs (golden vectors) and against the CPU oracle.  Bar: bit-exact
(NaN payloads aside) — the kernels run the reference's exact operation
order with --fmad=false."""

import numpy as np
import pytest
import torch

from helpers import (case_names, device_env, env_to_host, golden_io, manifest, numpy_env,
                     program, random_host_env, random_program, run_case, same_bits)
from oracle import counter_rng, numpy_eval
from paper_1804_10120_b200 import (EvalError, capture_graph, eval_batch, eval_program,
                                   eval_statement, eval_statement_per_component)
from paper_1804_10120_b200.runtime import all_kernels, fill_uniform, total_launches

pytestmark = pytest.mark.gpu

CASES = case_names()


def _check(case, env_host, want):
    for t in case["targets"]:
        assert same_bits(env_host[t], want[t]), t


@pytest.mark.parametrize("name", CASES)
def test_fused_program_matches_reference_bitwise(name):
    case = manifest()["cases"][name]
    prog, vs = program(case["source"])
    host, want = golden_io(name)
    env = device_env(prog, host)
    run_case(case, lambda: eval_program(vs, env))
    _check(case, env_to_host(env), want)


@pytest.mark.parametrize("name", CASES)
def test_statement_by_statement_matches_reference_bitwise(name):
    case = manifest()["cases"][name]
    prog, vs = program(case["source"])
    host, want = golden_io(name)
    env = device_env(prog, host)

    def go():
        for v in vs:
            eval_statement(v, env)

    run_case(case, go)
    _check(case, env_to_host(env), want)


@pytest.mark.parametrize("name", [n for n in CASES if len(manifest()["cases"][n]["statements"]) == 1])
def test_per_component_arrays_mode_bitwise(name):
    case = manifest()["cases"][name]
    prog, (v,) = program(case["source"])
    host, want = golden_io(name)
    env = device_env(prog, host)
    eval_statement_per_component(v, env)
    _check(case, env_to_host(env), want)


@pytest.mark.parametrize("name", ["c1_dtg", "c1_dtg_odd", "c3_christoffel", "c4_p3",
                                  "seq_augmented", "special_values", "aliased_write_order"])
def test_host_fields_staged_through_gpu_bitwise(name):
    # the reference's own numpy-backed fields: drop-in, computed on the GPU
    case = manifest()["cases"][name]
    prog, vs = program(case["source"])
    host, want = golden_io(name)
    env = numpy_env(prog, host)
    eval_program(vs, env)
    _check(case, env_to_host(env), want)
    env = device_env(prog, host, device="cpu")  # this package's host fields
    eval_program(vs, env)
    _check(case, env_to_host(env), want)


@pytest.mark.parametrize("register", ["0", "1"])
@pytest.mark.parametrize("name", ["p2", "p3"])
def test_pageable_host_fields_through_the_bounce_ring(name, register, monkeypatch):
    # pageable (numpy) host fields large enough for many bounce slabs: the
    # pinned ring wraps several times, the last slab is ragged, and outputs
    # drain oldest-first; TLB_HOST_REGISTER=1 takes the page-locking path
    from paper_1804_10120_b200 import bench as tb

    monkeypatch.setenv("TLB_HOST_REGISTER", register)
    prog, vs = tb.load(tb.PROGRAMS[name])
    n = 131072 * 7 + 333  # P2: 64 slots -> 131072-point bounce slabs
    host = random_host_env(prog, n, 23)
    want = {k: a.copy() for k, a in host.items()}
    numpy_eval.eval_program(vs, want)
    env = numpy_env(prog, host)
    eval_program(vs, env)
    got = env_to_host(env)
    for k in want:
        assert same_bits(got[k], want[k]), k


@pytest.mark.parametrize("name", ["c1_dtg_odd", "c3_christoffel", "suite_contract3"])
@pytest.mark.parametrize("chunk", [1, 7, 32])
def test_chunking_is_invisible(name, chunk):
    case = manifest()["cases"][name]
    prog, (v,) = program(case["source"])
    host, want = golden_io(name)
    env = device_env(prog, host)
    eval_statement(v, env, chunk=chunk, threads=4)
    _check(case, env_to_host(env), want)


@pytest.mark.parametrize("name", ["c4_p2", "c4_p3", "c2_maxwell", "suite_kij"])
def test_multi_domain_batch_one_launch(name):
    case = manifest()["cases"][name]
    prog, vs = program(case["source"])
    host, want = golden_io(name)
    envs = [device_env(prog, host) for _ in range(5)]
    before = total_launches()
    eval_batch(vs, envs)
    assert total_launches() == before + 1
    for env in envs:
        _check(case, env_to_host(env), want)


def test_cuda_graph_replay():
    case = manifest()["cases"]["c4_p2"]
    prog, vs = program(case["source"])
    host, want = golden_io("c4_p2")
    env = device_env(prog, host)
    g = capture_graph(lambda: eval_program(vs, env))
    for t in case["targets"]:
        env[t].data.zero_()
    g.replay()
    torch.cuda.synchronize()
    _check(case, env_to_host(env), want)


@pytest.mark.parametrize("seed", range(24))
def test_random_programs_match_oracle(seed):
    rng = np.random.default_rng(seed)
    src = random_program(rng, n_statements=1 + seed % 3)
    prog, vs = program(src)
    n = [1, 2, 3, 255, 256, 1001][seed % 6]
    host = random_host_env(prog, n, seed)
    want = {k: a.copy() for k, a in host.items()}
    numpy_eval.eval_program(vs, want)
    env = device_env(prog, host)
    eval_program(vs, env)
    got = env_to_host(env)
    for t in ("T", "U", "A"):
        assert same_bits(got[t], want[t]), (src, t)


def test_large_grid_slab_parity_and_partition_invisibility():
    # Christoffel + dt g (P2) at 2^22+6 points, counter-RNG inputs; check
    # three slabs bitwise against the oracle, and that evaluating two slab
    # views of the same fields gives the same bits as one launch
    case = manifest()["cases"]["c4_p2"]
    prog, vs = program(case["source"])
    n = (1 << 22) + 6
    env = device_env(prog, {k: np.zeros(a.shape[:-1] + (n,)) for k, a in
                            golden_io("c4_p2")[0].items()})
    names = list(prog.decls.tensors) + sorted(prog.decls.scalar_fields)
    for sid, nm in enumerate(names):
        fill_uniform(env[nm].data.view(-1), 0xC0FFEE, sid)
    eval_program(vs, env)
    got = env_to_host(env)
    for lo, hi in [(0, 4096), (n // 2 - 1000, n // 2 + 1000), (n - 4096, n)]:
        host = {}
        for sid, nm in enumerate(names):
            full = counter_rng.uniform(0xC0FFEE, sid, 0, env[nm].data.numel())
            host[nm] = full.reshape(env[nm].data.shape)[..., lo:hi].copy()
        for t in case["targets"]:
            host[t][:] = 0.0
        numpy_eval.eval_program(vs, host)
        for t in case["targets"]:
            assert same_bits(got[t][..., lo:hi], host[t]), (t, lo)
    # partition invisibility: two slab views
    from paper_1804_10120_b200.fields import ScalarField, TensorField

    def view(f, lo, hi):
        g = (TensorField if hasattr(f, "shape") else ScalarField)(f.name, *(
            (f.shape, 0) if hasattr(f, "shape") else (0,)))
        g.data = f.data[..., lo:hi]
        return g

    for t in case["targets"]:
        env[t].data.zero_()
    cut = (n // 3) & ~1
    for lo, hi in [(0, cut), (cut, n)]:
        eval_program(vs, {k: view(f, lo, hi) for k, f in env.items()})
    again = env_to_host(env)
    for t in case["targets"]:
        assert same_bits(again[t], got[t]), t


def test_device_rng_matches_host_twin():
    t = torch.empty(100_003, dtype=torch.float64, device="cuda")
    fill_uniform(t, 123, 7, offset=999)
    assert (t.cpu().numpy() == counter_rng.uniform(123, 7, 999, 100_003)).all()


def test_resize_and_error_semantics():
    prog, (v_set, v_add) = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\n"
                                   "A(i) = B(i);\nA(i) += B(i);\n")
    env = device_env(prog, {"A": np.zeros((3, 1, 2)), "B": np.ones((3, 1, 4))})
    eval_statement(v_set, env)
    assert env["A"].gridsize == 4 and bool((env["A"].data == 1).all())
    env["A"].resize(3)
    with pytest.raises(EvalError, match="cannot resize"):
        eval_statement(v_add, env)
    del env["B"]
    with pytest.raises(EvalError, match="'B'"):
        eval_statement(v_set, env)


def test_empty_grid_is_a_no_op():
    prog, (v,) = program("tensor A dim 3 rank 1;\nA(i) = 2;\n")
    env = device_env(prog, {"A": np.zeros((3, 1, 0))})
    eval_statement(v, env)
    assert env["A"].gridsize == 0


@pytest.mark.parametrize("case", ["c1_dtg", "c2_maxwell", "c4_p2", "c4_p3", "seq_augmented",
                                  "special_values"])
def test_reference_harness_drives_the_gpu_kernels(case, tmp_path):
    # the reference's own, unchanged tl_harness binary loads
    # our bindings table and runs every manifest entry on the GPU
    import subprocess

    from helpers import GOLDEN, read_host
    from oracle import refc
    from paper_1804_10120_b200.registry import Registry

    harness = refc.REF_DIR / "tl_harness"
    if not harness.exists():
        pytest.skip("oracle/_ref/tl_harness not built")
    spec = manifest()["cases"][case]
    _, vs = program(spec["source"])
    reg = Registry()
    for v in vs:
        reg.register(v)
    so = reg.build_shared(tmp_path)
    from paper_1804_10120_b200.runtime import cache_dir

    before = set(cache_dir().glob("harness_*.cubin"))
    out = tmp_path / "out.tldf"
    res = subprocess.run([str(harness), str(so), str(tmp_path / "tloops_manifest.tsv"),
                          str(GOLDEN / f"{case}.in.tldf"), str(out)],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    # build_shared precompiled every entry under the name the bindings look
    # up: the harness process compiled nothing
    assert set(cache_dir().glob("harness_*.cubin")) == before
    got, want = read_host(out), golden_io(case)[1]
    for t in spec["targets"]:
        assert same_bits(got[t], want[t]), t
    # and the reference's own comparator agrees, bitwise and in its rtol mode
    # (tl_compare.c:26-64; run_tests.sh's differential checks use both)
    compare = refc.REF_DIR / "tl_compare"
    if compare.exists():
        from paper_1804_10120_b200 import tldf

        # the golden output holds the targets only: compare those fields
        gold = GOLDEN / f"{case}.out.tldf"
        full = tldf.read(out, device="cpu")
        tgt = tmp_path / "targets.tldf"
        tldf.write(tgt, {t: full[t] for t in tldf.read(gold, device="cpu")})
        modes = [[str(tgt), str(gold), "1e-13"]]
        if case != "special_values":  # NaN payloads differ between x86 and the GPU
            modes.append(["--bitwise", str(tgt), str(gold)])
        for args in modes:
            res = subprocess.run([str(compare), *args], capture_output=True, text=True,
                                 timeout=120)
            assert res.returncode == 0, (args, res.stdout, res.stderr)


def test_bound_launch_fast_path_tracks_storage():
    case = manifest()["cases"]["c1_dtg"]
    prog, (v,) = program(case["source"])
    host, want = golden_io("c1_dtg")
    env = device_env(prog, host)
    eval_statement(v, env)
    eval_statement(v, env)  # fast path (bound launch)
    _check(case, env_to_host(env), want)
    # new input values in place: same storage, the bound launch sees them
    env["K"].data.mul_(2.0)
    eval_statement(v, env)
    h = env_to_host(env)
    ref = {k: a.copy() for k, a in h.items()}
    numpy_eval.eval_statement(v, ref)
    assert same_bits(h["dtg"], ref["dtg"])
    # replaced storage and resized target: the fast path must miss
    env["db"].data = env["db"].data.clone() + 1.0
    env["dtg"].resize(5)
    eval_statement(v, env)
    h = env_to_host(env)
    ref = {k: a.copy() for k, a in h.items()}
    numpy_eval.eval_statement(v, ref)
    assert env["dtg"].gridsize == case["N"] and same_bits(h["dtg"], ref["dtg"])
    del env["alpha"]
    with pytest.raises(EvalError, match="'alpha'"):
        eval_statement(v, env)


@pytest.mark.parametrize("seed", range(48))
def test_fuzzed_programs_match_oracle(seed):
    # random valid statements over dims 3 and 4, symmetric/nested/inner
    # groups, offsets, fixed slots, literals, sqrt/division, op=; fused
    # into one kernel and checked bitwise against the oracle
    import random

    from helpers import FUZZ_DECLS, fuzz_statement
    from paper_1804_10120_b200.ir import ValidationError, validate_statement
    from paper_1804_10120_b200.parser import parse_program

    rng = random.Random(1000 + seed)
    stmts = []
    while len(stmts) < 1 + seed % 4:
        res = parse_program(FUZZ_DECLS + fuzz_statement(rng))
        if not res.ok:
            continue
        try:
            stmts.append(validate_statement(res.program.statements[0], res.program.decls))
        except ValidationError:
            continue
    prog = parse_program(FUZZ_DECLS).program
    n = [1, 2, 7, 64, 255, 1000][seed % 6]
    host = random_host_env(prog, n, seed)
    want = {k: a.copy() for k, a in host.items()}
    numpy_eval.eval_program(stmts, want)
    env = device_env(prog, host)
    eval_program(stmts, env)
    got = env_to_host(env)
    for k in want:
        assert same_bits(got[k], want[k]), (k, [str(v.stmt) for v in stmts])


def _fused_cases() -> list[str]:
    """Golden cases that run as ONE fused launch (decided on host fields,
    at collection time, so the variant sweeps list only applicable cases)."""
    from paper_1804_10120_b200.evaluator import _fusion_plan

    out = []
    for name in CASES:
        case = manifest()["cases"][name]
        if case.get("raises"):
            continue
        try:
            prog, vs = program(case["source"])
            env = device_env(prog, golden_io(name)[0], device="cpu")
        except Exception:
            continue
        if _fusion_plan(vs, env) is not None:
            out.append(name)
    return out


def _grouped_cases(budget: int) -> list[str]:
    """Fused golden cases that split into more than one output group at
    `budget` live values (read-only programs whose outputs read no written slot)."""
    from paper_1804_10120_b200 import lowering

    out = []
    saved = lowering.VN_LIVE_BUDGET
    lowering.VN_LIVE_BUDGET = budget
    try:
        for name in FUSED:
            _, vs = program(manifest()["cases"][name]["source"])
            plan = lowering.lower_program(vs, variant=lowering.Variant(
                vec=1, waves=0, threads=128, ldmode=1, vn=1))
            if plan.variant.ldmode == 1 and "tlk_grp1" in plan.source:
                out.append(name)
    finally:
        lowering.VN_LIVE_BUDGET = saved
    return out


FUSED = _fused_cases()

VARIANTS = [dict(restrict=False), dict(hoist=True), dict(vec=1), dict(ldmode=1),
            dict(hoist=True, ldmode=1, vec=1), dict(waves=4), dict(stage=2),
            dict(stage=3, hoist=True), dict(stage=3, stage_reads=2),
            dict(stage=3, stage_reads=2, stage_ws=1)]


@pytest.mark.parametrize("vkw", VARIANTS, ids=lambda d: ",".join(f"{k}={v}" for k, v in d.items()))
@pytest.mark.parametrize("name", FUSED)
def test_every_codegen_variant_is_bit_exact(name, vkw):
    from paper_1804_10120_b200.lowering import Variant, lower_program
    from paper_1804_10120_b200.runtime import Kernel

    case = manifest()["cases"][name]
    prog, vs = program(case["source"])
    host, want = golden_io(name)
    env = device_env(prog, host)
    from paper_1804_10120_b200.evaluator import _bind, _fusion_plan

    fp = _fusion_plan(vs, env)
    if fp is None or case.get("raises"):
        pytest.skip("program does not run as one fused launch")
    n, resizes = fp
    for lhs, size in resizes:
        lhs.resize(size)
    _, _, stores = _bind(vs, env)
    plan = lower_program(vs, variant=Variant(**vkw))
    k = Kernel(plan)
    k.launch(n, [s.base for s in stores], [s.pitch for s in stores],
             torch.cuda.current_stream().cuda_stream)
    _check(case, env_to_host(env), want)


@pytest.mark.parametrize("name,budget", [(n, b) for b in (4, 16) for n in _grouped_cases(b)])
def test_output_groups_are_bit_exact(name, budget, monkeypatch):
    # Variant.vn = 1: outputs split into groups of at most `budget` live
    # values, one non-inlined device function each (the contractions' cure
    # for spills) — forced here with tiny budgets on every golden program
    # whose outputs never read a written slot
    from paper_1804_10120_b200 import lowering
    from paper_1804_10120_b200.evaluator import _bind, _fusion_plan
    from paper_1804_10120_b200.runtime import Kernel

    case = manifest()["cases"][name]
    prog, vs = program(case["source"])
    host, want = golden_io(name)
    env = device_env(prog, host)
    fp = _fusion_plan(vs, env)
    if fp is None or case.get("raises"):
        pytest.skip("program does not run as one fused launch")
    monkeypatch.setattr(lowering, "VN_LIVE_BUDGET", budget)
    plan = lowering.lower_program(vs, variant=lowering.Variant(vec=1, waves=0, threads=128,
                                                               ldmode=1, vn=1))
    if plan.variant.ldmode != 1 or "tlk_grp1" not in plan.source:
        pytest.skip("read-modify-write or chained program, or a single group")
    n, resizes = fp
    for lhs, size in resizes:
        lhs.resize(size)
    _, _, stores = _bind(vs, env)
    k = Kernel(plan)
    for vec in (1, 2):
        k.launch(n, [s_.base for s_ in stores], [s_.pitch for s_ in stores],
                 torch.cuda.current_stream().cuda_stream, vec=vec if n % 2 == 0 else 1)
        _check(case, env_to_host(env), want)


def _multi_part_cases() -> list[str]:
    from paper_1804_10120_b200.ir import ValidationError
    from paper_1804_10120_b200.lowering import statement_parts

    out = []
    for name in CASES:
        try:
            _, vs = program(manifest()["cases"][name]["source"])
        except (AssertionError, ValidationError):
            continue
        if len(statement_parts(vs)) > 1:
            out.append(name)
    return out


@pytest.mark.parametrize("name", _multi_part_cases())
def test_statement_parts_are_bit_exact(name):
    # Variant.split: a program of independent statement parts runs part after
    # part, each over its own run of blocks of tlk_flat_v1 — one-shot grids,
    # capped (grid-stride) grids of a few blocks, and the 2-point entry that
    # runs the parts in turn, against the reference's goldens
    from paper_1804_10120_b200.evaluator import _bind, _fusion_plan
    from paper_1804_10120_b200.lowering import Variant, lower_program
    from paper_1804_10120_b200.runtime import Kernel

    one_shot = 1 << 62  # TLB_ONE_SHOT (include/tlb200.h)
    case = manifest()["cases"][name]
    prog, vs = program(case["source"])
    host, want = golden_io(name)
    env = device_env(prog, host)
    fp = _fusion_plan(vs, env)
    if fp is None or case.get("raises"):
        pytest.skip("program does not run as one fused launch")
    plan = lower_program(vs, variant=Variant(vec=1, waves=0, threads=128, split=1))
    if "TLK_PARTS" not in plan.source:
        pytest.skip("a single statement part")
    n, resizes = fp
    k = Kernel(plan)
    for kw in (dict(max_blocks=one_shot), dict(max_blocks=3), dict(max_blocks=1),
               dict(max_blocks=0), dict(threads=64, max_blocks=one_shot),
               dict(vec=2 if n % 2 == 0 else 1)):
        env2 = device_env(prog, host)  # fresh inputs and targets per launch shape
        for lhs, size in resizes:
            env2[lhs.name].resize(size)
        _, _, st2 = _bind(vs, env2)
        k.launch(n, [s_.base for s_ in st2], [s_.pitch for s_ in st2],
                 torch.cuda.current_stream().cuda_stream, **kw)
        _check(case, env_to_host(env2), want)


@pytest.mark.parametrize("name", ["c4_p2", "c3_christoffel", "c2_maxwell", "c1_dtg"])
def test_c_abi_default_launch_is_bit_exact(name):
    # tlb_launch_default: the lowering's own geometry read from the source —
    # what a C caller without tuning opinions calls
    from paper_1804_10120_b200 import runtime
    from paper_1804_10120_b200.evaluator import _bind, _fusion_plan

    case = manifest()["cases"][name]
    prog, vs = program(case["source"])
    host, want = golden_io(name)
    env = device_env(prog, host)
    n, resizes = _fusion_plan(vs, env)
    for lhs, size in resizes:
        lhs.resize(size)
    _, kern, stores = _bind(vs, env)
    c_vp, c_ll = runtime.c_vp, runtime.c_ll
    rc = runtime.lib().tlb_launch_default(
        kern.handle, n, runtime._arr(c_vp, [s_.base for s_ in stores]),
        runtime._arr(c_ll, [s_.pitch for s_ in stores]),
        torch.cuda.current_stream().cuda_stream)
    assert rc == 0, runtime.lib().tlb_last_error()
    _check(case, env_to_host(env), want)


def test_grouped_program_in_a_multi_domain_batch():
    # contract3 lowers in output groups; its batch entry calls the same
    # group functions with the domain's slot pointers staged in shared memory
    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.evaluator import kernel_for

    src = {e.name: e.source for e in tb.builtin_suite()}["contract3"]
    prog, vs = program(src)
    hosts = [random_host_env(prog, n, 40 + n) for n in (4096, 1001, 4098)]
    envs = [device_env(prog, h) for h in hosts]
    assert kernel_for(vs, envs[0]).plan.variant.vn == 1
    eval_batch(vs, envs)
    for env, h in zip(envs, hosts):
        want = {k: a.copy() for k, a in h.items()}
        numpy_eval.eval_program(vs, want)
        got = env_to_host(env)
        for k in want:
            assert same_bits(got[k], want[k]), k


def test_ragged_multi_domain_batch():
    # subdomains of different (odd and even) sizes in one launch
    prog, vs = program(manifest()["cases"]["c4_p2"]["source"])
    sizes = [1, 2, 3, 100, 4097, 4096, 255]
    envs, hosts = [], []
    for d, n in enumerate(sizes):
        host = random_host_env(prog, n, 50 + d)
        for t in ("Gamma", "dtg"):
            host[t][:] = 0.0
        hosts.append(host)
        envs.append(device_env(prog, host))
    before = total_launches()
    eval_batch(vs, envs)
    assert total_launches() == before + 1
    for env, host in zip(envs, hosts):
        numpy_eval.eval_program(vs, host)
        got = env_to_host(env)
        for t in ("Gamma", "dtg"):
            assert same_bits(got[t], host[t]), (t, host[t].shape)


def test_concurrent_streams():
    # two programs on two streams at once: results independent of overlap
    case = manifest()["cases"]["c4_p2"]
    prog, vs = program(case["source"])
    host, want = golden_io("c4_p2")
    envs = [device_env(prog, host) for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for _ in range(3):
        for s, env in zip(streams, envs):
            with torch.cuda.stream(s):
                for t in case["targets"]:
                    env[t].data.zero_()
                eval_program(vs, env)
    torch.cuda.synchronize()
    for env in envs:
        _check(case, env_to_host(env), want)


def test_concurrent_host_staged_runs_from_threads():
    # several host threads each evaluate pageable (numpy) fields at once: the
    # runs take their own staging sets (two per context; a third waits), share
    # the host copy pool, and each result is bit-identical to the oracle
    import threading

    from paper_1804_10120_b200 import bench as tb

    prog, vs = tb.load(tb.P2)
    n = 131072 * 3 + 77
    hosts = [random_host_env(prog, n, 100 + t) for t in range(3)]
    wants = []
    for h in hosts:
        w = {k: a.copy() for k, a in h.items()}
        numpy_eval.eval_program(vs, w)
        wants.append(w)
    envs = [numpy_env(prog, h) for h in hosts]
    errors = []

    def work(env):
        try:
            for _ in range(2):
                eval_program(vs, env)
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(e,)) for e in envs]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for env, w in zip(envs, wants):
        got = env_to_host(env)
        for k in ("Gamma", "dtg"):
            assert same_bits(got[k], w[k]), k


def test_foreign_ir_classes_are_accepted():
    # the evaluator reads IR by class *name* and attributes (SURVEY 8b
    # drop-in): a tree made of another package's classes — here stand-ins
    # defined in tests/foreign_ir.py, as the reference's tlang.ir would be —
    # evaluates to the same bits
    import foreign_ir

    case = manifest()["cases"]["c4_p3"]
    prog, vs = program(case["source"])
    foreign = [foreign_ir.convert(v) for v in vs]
    assert type(foreign[0].stmt.rhs).__module__ == "foreign_ir"
    host, want = golden_io("c4_p3")
    env = device_env(prog, host)
    eval_program(foreign, env)
    _check(case, env_to_host(env), want)


def test_partially_overlapping_fields_are_rejected():
    prog, (v,) = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(i);\n")
    from paper_1804_10120_b200.fields import TensorField

    store = torch.zeros(3 * 1 * 10, dtype=torch.float64, device="cuda")
    a = TensorField("A", prog.decls.tensors["A"], 0)
    b = TensorField("B", prog.decls.tensors["B"], 0)
    a.data = store[:27].view(3, 1, 9)
    b.data = store[3:30].view(3, 1, 9)
    with pytest.raises(EvalError, match="overlap"):
        eval_statement(v, {"A": a, "B": b})


def test_parameter_block_beyond_4kib():
    # 513 component pointers -> a 4112-byte parameter block (CUDA >= 12.1
    # allows up to 32764 bytes on sm_70+)
    src = ("tensor A dim 4 rank 4;\ntensor B dim 4 rank 4;\nfield w;\n"
           "A(a, b, c, d) = B(d, c, b, a)*w + B(a, b, c, d);\n")
    prog, vs = program(src)
    host = random_host_env(prog, 1001, 3)
    want = {k: a.copy() for k, a in host.items()}
    numpy_eval.eval_program(vs, want)
    env = device_env(prog, host)
    eval_program(vs, env)
    assert same_bits(env_to_host(env)["A"], want["A"])
    envs = [device_env(prog, host) for _ in range(3)]  # and the batch table path
    eval_batch(vs, envs)
    for e in envs:
        assert same_bits(env_to_host(e)["A"], want["A"])


@pytest.mark.parametrize("split", [0, 1])
@pytest.mark.parametrize("bvec", [1, 2])
@pytest.mark.parametrize("bptrs", [0, 1])
@pytest.mark.parametrize("name", ["c4_p2", "c4_p3", "c1_dtg_odd", "seq_augmented",
                                  "c2_maxwell"])
def test_batch_entry_variants_bit_exact(name, bptrs, bvec, split):
    # split = 1: statement parts in the flat entry and (batch_split) as
    # (part, domain) row runs of the 1-point batch entry — programs of one
    # part lower unsplit
    from paper_1804_10120_b200.evaluator import _bind, _fusion_plan
    from paper_1804_10120_b200.lowering import Variant, lower_program
    from paper_1804_10120_b200.runtime import Batch, Kernel

    case = manifest()["cases"][name]
    prog, vs = program(case["source"])
    host, want = golden_io(name)
    envs = [device_env(prog, host) for _ in range(3)]
    kern = None
    bases, pitches, ns = [], [], []
    for env in envs:
        fp = _fusion_plan(vs, env)
        if fp is None or fp[1]:
            pytest.skip("not fusable without resizing")
        _, _, stores = _bind(vs, env)
        bases.append([s.base for s in stores])
        pitches.append([s.pitch for s in stores])
        ns.append(fp[0])
    plan = lower_program(vs, variant=Variant(batch_ptrs=bptrs, batch_vec=bvec, split=split,
                                             batch_split=split))
    kern = Kernel(plan)
    stream = torch.cuda.current_stream().cuda_stream
    Batch(kern, bases, pitches, ns, stream).launch(stream)
    for env in envs:
        _check(case, env_to_host(env), want)


@pytest.mark.parametrize("name", ["c1_dtg", "c2_maxwell", "c3_christoffel", "p2", "p3"])
def test_one_shot_block_shrink_bitwise_at_the_boundary(name):
    # a one-shot launch of fewer than SMs x 4 x threads points runs smaller
    # blocks (tlb_runtime launch_flat); both sides of that boundary, and
    # tiny launches, must be bit-identical to the oracle
    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.evaluator import kernel_for

    prog, vs = tb.load(tb.PROGRAMS[name])
    targets = [v.stmt.lhs.field for v in vs]
    env = tb.make_env(prog, targets[0], 8, 0xC0FFEE)
    kern = kernel_for(vs, env)
    assert kern.max_blocks == 1 << 62  # one-shot
    edge = torch.cuda.get_device_properties(0).multi_processor_count * 4 * kern.threads
    for n in (1, 63, 1000, edge - 1, edge, edge + 3):
        env = tb.make_env(prog, targets[0], n, 0xC0FFEE)
        host = {k: f.data.cpu().numpy().copy() for k, f in env.items()}
        eval_program(vs, env)
        numpy_eval.eval_program(vs, host)
        for t in targets:
            assert same_bits(env[t].data.cpu().numpy(), host[t]), (n, t)


@pytest.mark.parametrize("name", ["c1_dtg", "c2_maxwell", "c3_christoffel", "p2", "p3"])
@pytest.mark.parametrize("stage,reads,ws", [(2, 0, 0), (4, 0, 0), (3, 5, 0), (2, 0, 1),
                                           (3, 5, 1)])
def test_tma_staged_entry_bitwise(name, stage, reads, ws):
    # many whole tiles per block (ring wrap-around, mbarrier phase flips), a
    # ragged tail, and an unaligned slab view (falls back to the plain entry)
    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.evaluator import _bind
    from paper_1804_10120_b200.lowering import Variant, lower_program
    from paper_1804_10120_b200.runtime import Kernel

    prog, vs = tb.load(tb.PROGRAMS[name])
    targets = [v.stmt.lhs.field for v in vs]
    for n, lo in ((256 * 148 * 2 * 7 + 77, 0), (300001, 0), (300001, 1), (255, 0)):
        env = tb.make_env(prog, targets[0], n, 0xC0FFEE)
        host = {k: f.data.cpu().numpy().copy() for k, f in env.items()}
        _, _, stores = _bind(vs, env)
        plan = lower_program(vs, variant=Variant(stage=stage, stage_reads=reads, stage_ws=ws))
        if plan.variant.stage == 0:
            pytest.skip("read-modify-write program: no staged entry")
        k = Kernel(plan)
        assert k.vec == 3
        k.launch(n - lo, [s.base + 8 * lo for s in stores], [s.pitch for s in stores],
                 torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        sub = {key: a[..., lo:] for key, a in host.items()}
        numpy_eval.eval_program(vs, sub)
        for t in targets:
            got = env[t].data.cpu().numpy()[..., lo:]
            assert same_bits(got, sub[t]), (n, lo, t)


@pytest.mark.parametrize("tile,reads", [(128, 0), (256, 0), (128, 7)])
@pytest.mark.parametrize("name", ["c4_p2", "c4_p3"])
def test_tma_staged_batch_entry_bitwise(name, tile, reads):
    # the warp-specialised staged batch: ragged domains (odd counts and odd
    # pitches take the uncopied path), several items per block, ring reuse
    from paper_1804_10120_b200.evaluator import _bind
    from paper_1804_10120_b200.lowering import Variant, lower_program
    from paper_1804_10120_b200.runtime import Batch, Kernel

    prog, vs = program(manifest()["cases"][name]["source"])
    targets = sorted({v.stmt.lhs.field for v in vs})
    sizes = [1, 2, 3, 100, 4097, 4096, 255, 20000, 6] + [4096] * 300
    envs, hosts = [], []
    for d, n in enumerate(sizes):
        host = random_host_env(prog, n, 70 + d)
        for t in targets:
            host[t][:] = 0.0
        hosts.append(host)
        envs.append(device_env(prog, host))
    plan = lower_program(vs, variant=Variant(stage=3, stage_threads=tile, stage_reads=reads,
                                             batch_vec=3))
    kern = Kernel(plan)
    assert kern.batch_vec == 3
    bases, pitches = [], []
    for env in envs:
        _, _, stores = _bind(vs, env)
        bases.append([s.base for s in stores])
        pitches.append([s.pitch for s in stores])
    stream = torch.cuda.current_stream().cuda_stream
    Batch(kern, bases, pitches, sizes, stream).launch(stream)
    torch.cuda.synchronize()
    for env, host in zip(envs, hosts):
        numpy_eval.eval_program(vs, host)
        got = env_to_host(env)
        for t in targets:
            assert same_bits(got[t], host[t]), (t, host[t].shape)


def test_programs_without_reads_at_large_n():
    # constant fills read nothing: nothing to stage (a staged ring would wait
    # for copies that are never issued); every size class must complete
    from paper_1804_10120_b200.evaluator import kernel_for

    src = "tensor A dim 3 rank 2;\ntensor B dim 3 rank 1;\nA(i,j) = 2.5;\nB(i) = -1.0;\n"
    prog, vs = program(src)
    for n in (100, (1 << 21) + 3, (1 << 22) + 256):
        host = random_host_env(prog, n, 5)
        env = device_env(prog, host)
        eval_program(vs, env)
        torch.cuda.synchronize()
        got = env_to_host(env)
        assert (got["A"] == 2.5).all() and (got["B"] == -1.0).all()
    assert kernel_for(vs, env).plan.variant.stage == 0


@pytest.mark.parametrize("seed", range(16))
def test_fuzzed_programs_large_n(seed):
    # the fuzzed programs above at sizes past both size classes, so the
    # default policy runs its large-N entries (the TMA-staged one for every
    # read-only program) on odd and even point counts
    import random

    from helpers import FUZZ_DECLS, fuzz_statement
    from paper_1804_10120_b200.evaluator import kernel_for
    from paper_1804_10120_b200.ir import ValidationError, validate_statement
    from paper_1804_10120_b200.parser import parse_program

    rng = random.Random(5000 + seed)
    stmts = []
    while len(stmts) < 1 + seed % 3:
        res = parse_program(FUZZ_DECLS + fuzz_statement(rng))
        if not res.ok:
            continue
        try:
            stmts.append(validate_statement(res.program.statements[0], res.program.decls))
        except ValidationError:
            continue
    prog = parse_program(FUZZ_DECLS).program
    n = (1 << 21) + 256 * seed + (seed % 2)
    host = random_host_env(prog, n, seed)
    want = {k: a.copy() for k, a in host.items()}
    numpy_eval.eval_program(stmts, want)
    env = device_env(prog, host)
    eval_program(stmts, env)
    got = env_to_host(env)
    for k in want:
        assert same_bits(got[k], want[k]), (k, [str(v.stmt) for v in stmts])
    kern = kernel_for(stmts, env)
    assert n > kern.small_n


@pytest.mark.parametrize("name", ["add1", "add3", "kij", "christoffel", "contract1", "contract2",
                                  "contract3", "outer2", "assign2"])
def test_suite_statements_under_the_default_policy_at_large_n(name):
    # the reference's suite statements (bench.builtin_suite) past the
    # small-N classes, so the default policy's large-N entry runs: the
    # warp-specialised rings (3-deep light, 2-deep 128-point contraction
    # class) with many tiles per block, ring wrap-around and a ragged tail
    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.evaluator import kernel_for

    src = {e.name: e.source for e in tb.builtin_suite()}[name]
    prog, vs = program(src)
    # contractions: just past the heavier size class (2^20), 28 128-point
    # tiles per block; the others past the light class (2^21)
    n = 128 * 148 * 2 * 28 + 77 if name.startswith("contract") else (1 << 21) + 333
    host = random_host_env(prog, n, 11)
    want = {k: a.copy() for k, a in host.items()}
    numpy_eval.eval_program(vs, want)
    env = device_env(prog, host)
    eval_program(vs, env)
    got = env_to_host(env)
    for k in want:
        assert same_bits(got[k], want[k]), k
    kern = kernel_for(vs, env)
    assert n > kern.small_n
    if name.startswith("contract"):
        # and policy 2's contraction-class ring (2-deep, 128-point tiles, 40
        # staged reads, warp-specialised) on the same inputs
        from paper_1804_10120_b200.evaluator import _bind
        from paper_1804_10120_b200.lowering import choose_variant, lower_program
        from paper_1804_10120_b200.runtime import Kernel

        p3 = kern.plan
        var = choose_variant(p3.reads, p3.writes, p3.n_ops, 0, 0, policy=2)
        assert (var.stage, var.stage_threads, var.stage_reads, var.stage_ws) == (2, 128, 40, 1)
        env2 = device_env(prog, host)
        _, _, stores = _bind(vs, env2)
        k2 = Kernel(lower_program(vs, variant=var))
        k2.launch(n, [s_.base for s_ in stores], [s_.pitch for s_ in stores],
                  torch.cuda.current_stream().cuda_stream)
        got2 = env_to_host(env2)
        for k in want:
            assert same_bits(got2[k], want[k]), ("policy 2 ring", k)


def test_bound_launches_and_batch_fast_path():
    # bind_program / bind_batch launch exactly what eval_program / eval_batch
    # would; eval_batch's steady-state path notices replaced field storage
    from paper_1804_10120_b200 import bind_batch, bind_program

    prog, vs = program(manifest()["cases"]["c4_p2"]["source"])
    hosts, envs = [], []
    for d in range(6):
        host = random_host_env(prog, 300 + 2 * d, 90 + d)
        for t in ("Gamma", "dtg"):
            host[t][:] = 0.0
        hosts.append(host)
        envs.append(device_env(prog, host))
    want = []
    for host in hosts:
        w = {k: a.copy() for k, a in host.items()}
        numpy_eval.eval_program(vs, w)
        want.append(w)
    bound = bind_batch(vs, envs)
    bound()
    for env, w in zip(envs, want):
        got = env_to_host(env)
        for t in ("Gamma", "dtg"):
            assert same_bits(got[t], w[t]), t
    for env in envs:
        for t in ("Gamma", "dtg"):
            env[t].data.zero_()
    eval_batch(vs, envs)          # slow path, recorded
    eval_batch(vs, envs)          # identity fast path
    for env, w in zip(envs, want):
        got = env_to_host(env)
        for t in ("Gamma", "dtg"):
            assert same_bits(got[t], w[t]), t
    # replace one subdomain's input storage: the fast path must rebind
    new = random_host_env(prog, 300, 999)
    envs[0]["Invg"].data = torch.from_numpy(new["Invg"]).cuda()
    hosts[0]["Invg"] = new["Invg"]
    w0 = {k: a.copy() for k, a in hosts[0].items()}
    numpy_eval.eval_program(vs, w0)
    eval_batch(vs, envs)
    got = env_to_host(envs[0])
    for t in ("Gamma", "dtg"):
        assert same_bits(got[t], w0[t]), t
    # single grid
    env = envs[1]
    env["dtg"].data.zero_()
    env["Gamma"].data.zero_()
    bind_program(vs, env)()
    got = env_to_host(env)
    for t in ("Gamma", "dtg"):
        assert same_bits(got[t], want[1][t]), t


def test_staged_main_loop_special_values():
    # IEEE specials (inf, nan payloads, signed zeros, subnormals) through the
    # staged entry's ring — golden inputs tiled past many whole tiles — must
    # give the plain entry's bits, which the golden vectors pin
    from paper_1804_10120_b200.evaluator import _bind
    from paper_1804_10120_b200.lowering import Variant, lower_program
    from paper_1804_10120_b200.runtime import Kernel

    case = manifest()["cases"]["special_values"]
    prog, vs = program(case["source"])
    host, _ = golden_io("special_values")
    n0 = host["w"].shape[-1]
    reps = (1 << 20) // n0 + 3
    big = {k: np.ascontiguousarray(np.concatenate([a] * reps, axis=-1)) for k, a in host.items()}
    specials = np.array([np.inf, -np.inf, np.nan, -0.0, 0.0, 5e-324, -5e-324, 1e308, -1e-310],
                        dtype=np.float64)
    big["w"][: specials.size] = specials
    big["B"][..., -specials.size:] = specials
    n = big["w"].shape[-1]
    outs = []
    for var in (Variant(), Variant(stage=3, stage_threads=256), Variant(stage=2, stage_reads=1)):
        env = device_env(prog, big)
        _, _, stores = _bind(vs, env)
        k = Kernel(lower_program(vs, variant=var))
        k.launch(n, [s.base for s in stores], [s.pitch for s in stores],
                 torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        outs.append(env_to_host(env)["A"])
    assert same_bits(outs[0], outs[1]) and same_bits(outs[0], outs[2])
    want = {k: a.copy() for k, a in big.items()}
    numpy_eval.eval_program(vs, want)
    assert same_bits(outs[0], want["A"])


# ------------------------------------------------ round-2 parity regressions
# (VERDICT r01 "what's weak" #1a-c)


def test_mixed_gridsize_program_does_not_resize_before_reading():
    # ADVICE r01 example: D(i)=C(i); C(i)=A(i) with |C|=|D|=4, |A|=8 — the
    # reference gives D = old C over 4 points, C = A over 8
    prog, vs = program("tensor A dim 3 rank 1;\ntensor C dim 3 rank 1;\ntensor D dim 3 rank 1;\n"
                       "D(i) = C(i);\nC(i) = A(i);\n")
    rng = np.random.default_rng(4)
    host = {"A": rng.uniform(size=(3, 1, 8)), "C": rng.uniform(size=(3, 1, 4)),
            "D": np.zeros((3, 1, 4))}
    want = {k: a.copy() for k, a in host.items()}
    numpy_eval.eval_program(vs, want)
    for runner in ("program", "batch"):
        env = device_env(prog, host)
        if runner == "program":
            eval_program(vs, env)
        else:
            eval_batch(vs, [env])
        got = env_to_host(env)
        assert got["D"].shape[-1] == 4 and got["C"].shape[-1] == 8
        for k in ("C", "D"):
            assert same_bits(got[k], want[k]), (runner, k)


def _raw_chain_envs(prog, n, seed):
    """Two subdomains where subdomain 1 reads (as A) the field subdomain 0
    writes (B): sequentially, B1 = f(B0) = f(f(A0))."""
    from paper_1804_10120_b200.fields import TensorField

    rng = np.random.default_rng(seed)
    shape = prog.decls.tensors["A"]
    mk = lambda name, data: _field(TensorField(name, shape, 0), data)  # noqa: E731
    a0 = mk("A", torch.from_numpy(rng.uniform(size=(3, 1, n))).cuda())
    b0 = mk("B", torch.zeros(3, 1, n, dtype=torch.float64, device="cuda"))
    b1 = mk("B", torch.zeros(3, 1, n, dtype=torch.float64, device="cuda"))
    a1 = mk("A", b0.data)  # the same storage as subdomain 0's output
    return [{"A": a0, "B": b0}, {"A": a1, "B": b1}]


def _field(f, data):
    f.data = data
    return f


@pytest.mark.parametrize("n", [1000, 1 << 20])
def test_cross_domain_read_after_write_batch_equals_sequential(n):
    prog, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\n"
                       "B(i) = A(i)*A(i) + A(i);\n")
    envs = _raw_chain_envs(prog, n, 11)
    seq = _raw_chain_envs(prog, n, 11)
    for env in seq:
        eval_program(vs, env)
    eval_batch(vs, envs)
    torch.cuda.synchronize()
    for e, s_ in zip(envs, seq):
        assert same_bits(env_to_host(e)["B"], env_to_host(s_)["B"])
    # and the oracle: B0 = A0^2 + A0, B1 = B0^2 + B0
    a0 = env_to_host(envs[0])["A"]
    b0 = a0 * a0 + a0
    assert same_bits(env_to_host(envs[1])["B"], b0 * b0 + b0)
    from paper_1804_10120_b200 import bind_batch

    with pytest.raises(EvalError, match="cannot share one launch"):
        bind_batch(vs, envs)


def test_halo_views_batch_equals_sequential():
    # subdomains as overlapping windows (ghost zones) of one global array:
    # each writes its own window of B and reads a window of B that
    # overlaps its neighbours' writes — one launch would race
    from paper_1804_10120_b200.fields import TensorField

    prog, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\n"
                       "B(i) = B(i)*2 + A(i);\n")
    n, h, nd = 4096, 16, 6

    def build():
        rng = np.random.default_rng(21)
        gA = torch.from_numpy(rng.uniform(size=(3, 1, nd * n + 2 * h))).cuda()
        gB = torch.from_numpy(rng.uniform(size=(3, 1, nd * n + 2 * h))).cuda()
        envs = []
        for d in range(nd):
            lo = d * n
            a = _field(TensorField("A", prog.decls.tensors["A"], 0), gA[..., lo:lo + n + 2 * h])
            b = _field(TensorField("B", prog.decls.tensors["B"], 0), gB[..., lo:lo + n + 2 * h])
            envs.append({"A": a, "B": b})
        return gB, envs

    gB_batch, envs = build()
    gB_seq, seq = build()
    for env in seq:
        eval_program(vs, env)
    eval_batch(vs, envs)
    torch.cuda.synchronize()
    assert same_bits(gB_batch.cpu().numpy(), gB_seq.cpu().numpy())


def test_disjoint_subdomains_still_share_one_launch():
    # read-only storage shared by every subdomain (one `w` field) is not a
    # hazard: still one launch
    from paper_1804_10120_b200.fields import ScalarField

    prog, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nfield w;\n"
                       "B(i) = A(i)*w;\n")
    w = _field(ScalarField("w", 0), torch.rand(512, dtype=torch.float64, device="cuda"))
    envs = []
    for d in range(4):
        h = random_host_env(prog, 512, d)
        e = device_env(prog, h)
        e["w"] = w
        envs.append(e)
    before = total_launches()
    eval_batch(vs, envs)
    assert total_launches() == before + 1
    for e in envs:
        got = env_to_host(e)
        assert same_bits(got["B"], got["A"] * w.data.cpu().numpy())


def test_graph_keeps_its_batch_table_alive():
    # a captured eval_batch must survive eviction of its table
    # from the batch cache (more than its capacity of other batches)
    from paper_1804_10120_b200 import evaluator as ev

    case = manifest()["cases"]["c4_p2"]
    prog, vs = program(case["source"])
    host, want = golden_io("c4_p2")
    envs = [device_env(prog, host) for _ in range(3)]
    g = capture_graph(lambda: eval_batch(vs, envs))
    assert any(type(p).__name__ == "Batch" for p in g.tlb_pins)
    ev._batches._d.clear()
    ev._BATCH_FAST.clear()
    import gc

    gc.collect()
    for env in envs:
        for t in case["targets"]:
            env[t].data.zero_()
    # churn: other tables reuse freed device memory
    others = [[device_env(prog, host) for _ in range(2)] for _ in range(4)]
    for o in others:
        eval_batch(vs, o)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    for env in envs:
        _check(case, env_to_host(env), want)


def test_kernel_eviction_unloads_and_recompiles():
    from paper_1804_10120_b200 import evaluator as ev
    from paper_1804_10120_b200 import runtime

    case = manifest()["cases"]["c1_dtg"]
    prog, (v,) = program(case["source"])
    host, want = golden_io("c1_dtg")
    env = device_env(prog, host)
    eval_statement(v, env)
    import gc
    import weakref

    kern = weakref.ref(ev.kernel_for([v], env))
    runtime._kernels.clear()
    ev._plans._d.clear()
    ev._FAST.clear()
    ev._batches._d.clear()
    ev._BATCH_FAST.clear()
    gc.collect()  # the kernel's last references are gone: module unloaded
    assert kern() is None
    env = device_env(prog, host)
    eval_statement(v, env)  # relowered, reloaded (cubin from the disk cache)
    _check(case, env_to_host(env), want)
