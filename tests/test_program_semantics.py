"""Host-side program semantics (no GPU): when a program may run as one fused
launch, literal folding through the register shadow, cross-subdomain
hazards of one batched launch, and the bounded host caches.

Round-2 regressions of VERDICT r01 "what's weak" #1a-c and ADVICE r01; the
GPU side of the same cases is in test_gpu_parity.py, and the reference's
own outputs for them are golden cases (tests/golden/make_golden.py)."""

import math

import numpy as np
import pytest

from helpers import NumpyTensorField, numpy_env, program
from paper_1804_10120_b200 import evaluator as ev
from paper_1804_10120_b200.lowering import lower_program


def _env(prog, sizes, seed=0):
    rng = np.random.default_rng(seed)
    host = {}
    for name, shape in prog.decls.tensors.items():
        host[name] = rng.uniform(size=(shape.outer_count, shape.inner_count, sizes[name]))
    for name in prog.decls.scalar_fields:
        host[name] = rng.uniform(size=sizes[name])
    return numpy_env(prog, host)


# ------------------------------------------------------------ literal folding


def test_literal_through_a_field_write_folds_with_ieee_semantics():
    # A(i) = 1; A(i) /= 0 — the reference stores 1.0 into an array, then
    # divides the ARRAY by 0 under errstate(divide="ignore"): inf, no error
    _, vs = program("tensor A dim 3 rank 1;\nA(i) = 1;\nA(i) /= 0;\nA(i) *= -1;\n")
    plan = lower_program(vs)
    stores = [ln for ln in plan.source.splitlines() if "tl_st(" in ln and "+ x" in ln]
    ninf = np.float64(-np.inf).view(np.int64)
    assert len(stores) == 3 and all(f"{ninf}LL" in ln for ln in stores)


def test_read_of_a_zero_written_earlier_is_not_a_python_division():
    _, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\n"
                    "A(i) = 0;\nB(i) = B(i)*(1/A(0));\n")
    lower_program(vs)  # no ZeroDivisionError: A(0) is a float64 array element


def test_literal_only_subtree_still_raises_like_the_reference():
    _, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(i)*(1/0);\n")
    with pytest.raises(ZeroDivisionError):
        lower_program(vs)


def test_nan_and_inf_literals_are_emitted_as_bit_patterns():
    _, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\n"
                    "A(i) = 0;\nA(i) /= 0;\nB(i) = B(i)*A(0);\n")
    plan = lower_program(vs)
    # A = 0/0 is folded to NaN and emitted by bit pattern (no decimal text)
    nan_bits = np.array([np.float64(0.0)], dtype=np.float64)
    with np.errstate(all="ignore"):
        nan_bits = (nan_bits / nan_bits).view(np.int64)[0]
    assert f"__longlong_as_double({nan_bits}LL)" in plan.source
    assert math.isnan(np.int64(nan_bits).view(np.float64))


# ------------------------------------------------------ fusion decisions


MIXED = ("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\n"
         "B(i) = A(i);\nA(i) = C(i);\n")


def test_resize_of_a_field_read_earlier_is_not_fused_and_nothing_is_touched():
    prog, vs = program(MIXED)
    env = _env(prog, {"A": 4, "B": 4, "C": 8})
    before = {k: f.data.copy() for k, f in env.items()}
    assert ev._fusion_plan(vs, env) is None
    for k, f in env.items():
        assert f.data.shape == before[k].shape and (f.data == before[k]).all()


def test_resize_of_a_field_first_used_by_its_statement_is_hoisted():
    prog, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\n"
                       "A(2) = C(1);\nB(i) = A(i) + C(i);\n")
    env = _env(prog, {"A": 5, "B": 5, "C": 9})
    n, resizes = ev._fusion_plan(vs, env)
    assert n == 9 and [f.name for f, _ in resizes] == ["A", "B"]
    assert env["A"].gridsize == 5  # decided, not applied


@pytest.mark.parametrize("src,sizes", [
    # op= on a mismatched target (the reference raises at that statement)
    ("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) += B(i);\n", {"A": 3, "B": 4}),
    # disagreeing right-hand sides
    ("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\n"
     "A(i) = B(i) + C(i);\n", {"A": 4, "B": 4, "C": 5}),
    # two gridsizes in one program
    ("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\n"
     "tensor D dim 3 rank 1;\nA(i) = B(i);\nC(i) = D(i);\n", {"A": 4, "B": 4, "C": 6, "D": 6}),
])
def test_unfusable_programs_go_sequential(src, sizes):
    prog, vs = program(src)
    assert ev._fusion_plan(vs, _env(prog, sizes)) is None


def test_missing_field_goes_sequential():
    prog, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(i);\n")
    env = _env(prog, {"A": 4, "B": 4})
    del env["B"]
    assert ev._fusion_plan(vs, env) is None


def test_uniform_program_fuses_without_resizes():
    prog, vs = program(MIXED)
    env = _env(prog, {"A": 6, "B": 6, "C": 6})
    assert ev._fusion_plan(vs, env) == (6, [])


# ------------------------------------------------------- batch hazards


def _spans(*doms):
    out = []
    for d, ranges in enumerate(doms):
        for lo, hi, w in ranges:
            out.append((lo, hi, d, w))
    return out


def test_disjoint_subdomains_are_not_a_hazard():
    assert not ev._cross_domain_hazard(_spans([(0, 10, True), (10, 20, False)],
                                              [(20, 30, True), (30, 40, False)]))


def test_shared_read_only_storage_is_not_a_hazard():
    assert not ev._cross_domain_hazard(_spans([(0, 10, True), (100, 200, False)],
                                              [(20, 30, True), (100, 200, False)]))


@pytest.mark.parametrize("doms", [
    ([(0, 10, True)], [(0, 10, False)]),           # one reads what the other writes
    ([(0, 10, True)], [(5, 15, True)]),            # partially overlapping writes
    ([(0, 10, False)], [(20, 30, True), (9, 12, False)]),  # a halo read overlapping a write
])
def test_overlaps_involving_a_write(doms):
    got = ev._cross_domain_hazard(_spans(*doms))
    has_write_overlap = any(
        w1 or w2 for d1, r1 in enumerate(doms) for d2, r2 in enumerate(doms) if d1 < d2
        for lo1, hi1, w1 in r1 for lo2, hi2, w2 in r2 if lo1 < hi2 and lo2 < hi1)
    assert got == has_write_overlap


def test_hazard_agrees_with_brute_force():
    rng = np.random.default_rng(3)
    for _ in range(500):
        doms = []
        for d in range(rng.integers(2, 5)):
            cur = int(rng.integers(0, 40))
            ranges = []
            for _ in range(rng.integers(1, 4)):  # disjoint within a domain
                lo = cur + int(rng.integers(0, 10))
                hi = lo + int(rng.integers(1, 12))
                ranges.append((lo, hi, bool(rng.integers(0, 2))))
                cur = hi
            doms.append(ranges)
        want = any(
            w1 or w2 for d1, r1 in enumerate(doms) for d2, r2 in enumerate(doms) if d1 < d2
            for lo1, hi1, w1 in r1 for lo2, hi2, w2 in r2 if lo1 < hi2 and lo2 < hi1)
        assert ev._cross_domain_hazard(_spans(*doms)) == want, doms


# --------------------------------------------------------- bounded caches


def test_lru_evicts_least_recently_used():
    c = ev._LRU(3)
    for k in "abc":
        c.put(k, k.upper())
    assert c.get("a") == "A"  # refresh a
    c.put("d", "D")
    assert c.get("b") is None and c.get("a") == "A" and len(c) == 3


def test_host_caches_are_bounded():
    assert ev._NAMES.cap and ev._FAST.cap and ev._FAST_NAMES.cap and ev._BATCH_FAST.cap
    assert ev._plans._d.cap and ev._batches._d.cap
    from paper_1804_10120_b200 import runtime

    assert runtime.KERNEL_CACHE_SIZE > 0


def test_alias_detection_includes_strides():
    # a transposed view of the same buffer (same address, same
    # shape, other strides) is a different field — it must not be merged
    # into the other name as an alias (it then overlaps it: rejected)
    prog, vs = program("tensor A dim 3 rank 1 inner rank 1;\ntensor B dim 3 rank 1 inner rank 1;\n"
                       "A(i)(j) = B(j)(i);\n")
    buf = np.random.default_rng(0).uniform(size=(3, 3, 2))
    a = NumpyTensorField("A", prog.decls.tensors["A"], buf)
    b = NumpyTensorField("B", prog.decls.tensors["B"], buf.transpose(1, 0, 2))
    assert a.data.ctypes.data == b.data.ctypes.data and a.data.shape == b.data.shape
    with pytest.raises(ev.EvalError, match="overlap"):
        ev._bind(vs, {"A": a, "B": b})
    # an exact alias (same view) is still one field
    plan, _, stores = ev._bind(vs, {"A": a, "B": NumpyTensorField("B", a.shape, buf)})
    assert [f.name for f in plan.fields] == ["A"]
