"""Pin the CPU oracle (oracle/) to the reference's own outputs: the numpy
restatement must reproduce the reference evaluator bit for bit on every
golden case, the per-point restatement within tl_compare's 1e-13."""

import numpy as np
import pytest

from helpers import case_names, golden_io, manifest, program, run_case, same_bits
from oracle import numpy_eval, pointwise


@pytest.mark.parametrize("name", case_names())
def test_numpy_oracle_bitwise_equals_reference(name):
    case = manifest()["cases"][name]
    _, vs = program(case["source"])
    env, want = golden_io(name)
    run_case(case, lambda: numpy_eval.eval_program(vs, env), exact=False)
    for t in case["targets"]:
        assert same_bits(env[t], want[t]), t


@pytest.mark.parametrize("name", [n for n in case_names()
                                  if manifest()["cases"][n]["N"] <= 64])
def test_pointwise_oracle_within_tolerance(name):
    case = manifest()["cases"][name]
    _, vs = program(case["source"])
    env, want = golden_io(name)
    if case.get("raises") or case.get("sizes"):
        pytest.skip("the per-point oracle has no gridsize/error semantics")
    for v in vs:
        pointwise.run(v, env)
    for t in case["targets"]:
        a, b = env[t], want[t]
        assert (np.isnan(a) == np.isnan(b)).all()
        fin = np.isfinite(a) & np.isfinite(b)
        assert (a[~fin & ~np.isnan(a)] == b[~fin & ~np.isnan(b)]).all()
        assert numpy_eval.max_rel_error(a[fin], b[fin]) <= 1e-13, t


@pytest.mark.parametrize("name", case_names())
def test_oracle_counts_equal_reference(name):
    case = manifest()["cases"][name]
    _, vs = program(case["source"])
    for v, st in zip(vs, case["statements"]):
        assert list(numpy_eval.data_count(v)) == st["count_data"]


def test_counter_rng_matches_reference_formula():
    from oracle import counter_rng

    x = counter_rng.uniform(0xC0FFEE, 5, 1000, 64)
    y = counter_rng.uniform(0xC0FFEE, 5, 0, 1064)[1000:]
    assert (x == y).all()
    assert ((x >= 0) & (x < 1)).all()
    assert len(set(x.tolist())) == 64
