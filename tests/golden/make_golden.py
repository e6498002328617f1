"""Generate golden vectors by running the REFERENCE package (build container
only: it imports ``tlang`` read-only from /root/reference/pkg/src, which does
not exist on the GPU box).  The outputs are committed next to this script:

  <case>.in.tldf    inputs, seeded exactly like bench.make_env
                    (pkg/src/tlang/bench.py:72-87) plus per-case setup
  <case>.out.tldf   every statement target after the reference evaluator
                    (pkg/src/tlang/evaluator.py:204-236) ran the program
  manifest.json     per case: source, N, seed, and the reference's
                    signature / count_data / LHS component order /
                    component counts / alias tables; parser and validation
                    verdicts for malformed programs.

Run:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

from tlang import bench, tldf  # noqa: E402
from tlang.evaluator import eval_statement, eval_statement_per_component  # noqa: E402
from tlang.ir import ValidationError, count_data, signature, validate_statement  # noqa: E402
from tlang.parser import TensorDecl, parse_program, render  # noqa: E402
from tlang.registry import _combined_alias  # noqa: E402
from tlang.codegen_c import collect_args  # noqa: E402

OUT = Path(__file__).resolve().parent
SEED = 0xC0FFEE

SPECIALS = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 1e308, -1e308,
                     2.2250738585072014e-308, 1.0, -1.0, 0.5, 3.0, 1e-300, -7.5])

DTG = ("tensor dtg dim 3 rank 2 sym(0,1);\nfield alpha;\ntensor K dim 3 rank 2 sym(0,1);\n"
       "tensor db dim 3 rank 2;\n"
       "dtg(sym<0,1>, i, j) = -2*alpha*K(i,j) + db(i,j) + db(j,i);\n")
MAXWELL = """tensor dE dim 3 rank 1 inner rank 1;
tensor dB dim 3 rank 1 inner rank 1;
tensor dtE dim 3 rank 1;
tensor dtB dim 3 rank 1;
tensor divE dim 1 rank 1;
tensor divB dim 1 rank 1;
dtE(0) = dB(2)(1) - dB(1)(2);
dtE(1) = dB(0)(2) - dB(2)(0);
dtE(2) = dB(1)(0) - dB(0)(1);
dtB(0) = dE(1)(2) - dE(2)(1);
dtB(1) = dE(2)(0) - dE(0)(2);
dtB(2) = dE(0)(1) - dE(1)(0);
divE(0) = Sum(i, dE(i)(i));
divB(0) = Sum(i, dB(i)(i));
"""
CHRISTOFFEL = """tensor Gamma dim 3 rank 3 sym(1,2);
tensor Invg dim 3 rank 2 sym(0,1);
tensor dg dim 3 rank 2 sym(0,1) inner rank 1;
Gamma(sym<1,2>, i, j, k) = 0.5*Sum(l, Invg(i,l)*(dg(j,l)(k)+dg(l,k)(j)-dg(j,k)(l)));
"""
P2 = """tensor Gamma dim 3 rank 3 sym(1,2);
tensor Invg dim 3 rank 2 sym(0,1);
tensor dg dim 3 rank 2 sym(0,1) inner rank 1;
tensor dtg dim 3 rank 2 sym(0,1);
field alpha;
tensor K dim 3 rank 2 sym(0,1);
tensor db dim 3 rank 2;
Gamma(sym<1,2>, i, j, k) = 0.5*Sum(l, Invg(i,l)*(dg(j,l)(k)+dg(l,k)(j)-dg(j,k)(l)));
dtg(sym<0,1>, i, j) = -2*alpha*K(i,j) + db(i,j) + db(j,i);
"""
P3 = """tensor Gamma dim 3 rank 3 sym(1,2);
tensor Invg dim 3 rank 2 sym(0,1);
tensor dg dim 3 rank 2 sym(0,1) inner rank 1;
tensor beta dim 3 rank 1;
tensor dbeta dim 3 rank 1 inner rank 1;
tensor db dim 3 rank 2;
tensor dtg dim 3 rank 2 sym(0,1);
tensor K dim 3 rank 2 sym(0,1);
field alpha;
Gamma(sym<1,2>, i, j, k) = 0.5*Sum(l, Invg(i,l)*(dg(j,l)(k)+dg(l,k)(j)-dg(j,k)(l)));
db(i, j) = dbeta(j)(i) - Sum(k, Gamma(k, i, j)*beta(k));
dtg(sym<0,1>, i, j) = -2*alpha*K(i,j) + db(i,j) + db(j,i);
"""

# reference harness-differential edge programs (pkg/tests/test_harness_differential.py:78-148)
EDGE = {
    "seq_augmented": (
        "tensor h dim 3 rank 2 sym(0,1);\ntensor v dim 3 rank 1;\nfield lapse;\n"
        "h(sym<0,1>, i, j) = 0.25*lapse*v(i)*v(j);\n"
        "h(sym<0,1>, i, j) += v(i)*v(j);\n"
        "h(sym<0,1>, i, j) *= 2;\n"
        "v(i) = Sum(k, h(i,k)*v(k));\n", 33),
    "shadowed_sum": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\n"
        "A(i) = B(i)*Sum(i, C(i));\n", 16),
    "nested_shadowed_sums": (
        "tensor A dim 3 rank 1;\ntensor T dim 3 rank 1;\ntensor U dim 3 rank 2;\n"
        "A(i) = Sum(l, T(l)*Sum(l, U(i, l)));\n", 8),
    "generated_identifiers": (
        "index x: 3;\nindex s0: 3;\ntensor A dim 3 rank 2;\ntensor B dim 3 rank 2;\n"
        "A(x, s0) = B(s0, x);\n", 12),
    "offsets_fixed_division": (
        "tensor g dim 3 rank 2 sym(0,1);\ntensor psi dim 4 rank 2 sym(0,1);\nfield w;\n"
        "g(sym<0,1>, i, j) = psi(i+1, j+1)/w;\n", 21),
    "inner_group_contraction": (
        "tensor v dim 3 rank 1;\ntensor dh dim 3 rank 2 sym(0,1) inner rank 1;\n"
        "v(i) = Sum(k, dh(i,k)(k));\n", 10),
    "sqrt_negation": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nfield w;\n"
        "A(i) = -B(i)*sqrt(w) - B(i)/2;\n", 17),
    # evaluator unit cases (pkg/tests/test_evaluator.py)
    "scalar_rhs_zero": ("tensor A dim 3 rank 2;\nA(i, j) = 0;\n", 5),
    "all_fixed_target": ("tensor A dim 3 rank 2;\nA(2, 1) = 7;\n", 3),
    "augmented_ops": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nfield w;\n"
        "A(i) += B(i);\nA(i) -= 0.25*B(i);\nA(i) *= w;\nA(i) /= w + 1;\n", 16),
    "aliased_write_order": ("tensor A dim 3 rank 2;\nA(i, j) = A(j, i);\n", 1),
    "symmetric_alias_read": (
        "tensor S dim 3 rank 2 sym(0,1);\ntensor A dim 3 rank 2;\n"
        "A(i, j) = S(j, i) - S(i, j)*2;\nS(sym<0,1>, i, j) = A(i, j) + A(j, i);\n", 9),
    "constant_folding": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nconst c = 3;\n"
        "A(i) = B(i)*(2*c - -1)/sqrt(4*c) + B(i)*(1 - 1) + B(i)*sqrt(0 - 1)*0;\n", 9),
    "negative_zero_sum": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 2;\n"
        "A(i) = Sum(j, -B(i, j)*0);\n", 7),
    "special_values": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nfield w;\n"
        "A(i) = B(i)/w - B(i)*sqrt(w) + w*B(i) - B(i)/(w - w);\n", 40),
    "rank4_dim4_contraction": (
        "tensor R dim 4 rank 4 sym(0,1) sym(2,3);\ntensor G dim 4 rank 2 sym(0,1);\n"
        "tensor T dim 4 rank 2;\n"
        "T(a, b) = Sum(c, Sum(d, G(c, d)*R(a, c, b, d)));\n", 11),
    "three_slot_chain": (
        "tensor C dim 3 rank 3 sym(0,1) sym(1,2);\ntensor v dim 3 rank 1;\n"
        "C(sym<0,1> && sym<1,2>, i, j, k) = v(i)*v(j)*v(k) - v(k)*v(j)*v(i)/3;\n", 13),
}

# round-2 parity cases (VERDICT r01 "what's weak" #1a/#1b): literal values that
# reach a field through a write and are then read back, and a program whose
# later statement resizes a field an earlier one reads
EDGE.update({
    "fused_literal_div_zero": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\n"
        "A(i) = 0;\nB(i) = C(i)/A(1) + C(i)*(1/A(0)) - C(i)*(A(1)*0/A(2));\n", 7),
    "augmented_div_after_literal": (
        "tensor A dim 3 rank 1;\ntensor S dim 3 rank 2 sym(0,1);\n"
        "A(i) = 1;\nA(i) /= 0;\nA(i) *= -1;\nS(sym<0,1>, i, j) = A(i)*A(j) - A(j)/A(0)*A(i);\n", 5),
    "mixed_gridsize_read_before_resize": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\n"
        "B(i) = A(i);\nA(i) = C(i);\n", 4),
    "mixed_gridsize_resize_first_use": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\n"
        "A(2) = C(1);\nB(i) = A(i) + C(i);\n", 5),
})
# fields whose gridsize differs from the case's N: name -> N (fresh uniform
# data from default_rng(seed + 1), after the declaration-order fixture)
SIZES = {
    "mixed_gridsize_read_before_resize": {"C": 8},
    "mixed_gridsize_resize_first_use": {"C": 9},
}
# programs the reference stops part-way through: the error it raises and the
# targets as they are at that point (earlier statements ran)
RAISES = {
    "error_after_first_statement": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\n"
        "tensor D dim 3 rank 1;\nB(i) = A(i)*2;\nC(i) += D(i);\nA(i) = D(i);\n", 4,
        {"C": 3}),
    "error_literal_zero_division_second": (
        "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\n"
        "A(i) = B(i)*2;\nB(i) = A(i)*(1/0);\n", 6, {}),
}

SPECIAL_CASES = {"special_values"}
ARANGE_CASES = {"aliased_write_order", "augmented_ops"}

BAD_PROGRAMS = [
    "tensor A dim 3 rank 1;\nA(i) = B(i);\n",
    "tensor A dim 3 rank 1\ntensor B dim 3 rank 1;\n",
    "tensor A dim 3 rank 1;\ntensor A dim 3 rank 1;\n",
    "tensor sym dim 3 rank 1;\n",
    "tensor A dim 3 rank 2 sym(1,0);\n",
    "tensor A dim 3 rank 1;\nA(i) = 2 $ 3;\n",
    "tensor A dim 3 rank 1;\nA(z) = 1;\n",
    "field f;\nf = 1;\n",
    "tensor A dim 0 rank 1;\n",
    "tensor A dim 3 rank 1;\nA(i) = ;\n",
    "index p: 0;\n",
    "const c = x;\n",
    "tensor A dim 3 rank 2 sym(0,2);\n",
    "tensor A dim 3 rank 1;\nA(i) == 1;\nA(i) = 1;\n",
    "tensor A dim 3 rank 1;\nA(i) = Sum(i A(i));\n",
    "tensor A dim 3 rank 1;\nfield f;\nA(i) = f(i);\n",
    "tensor A dim 3 rank 1;\nA(i) = 1e5e + .5 + 2.;\n",
    "tensor A dim 3 rank 1;\nA(i) = A(i+x);\n",
]

INVALID_STATEMENTS = [
    "tensor A dim 3 rank 2;\nA(i, i) = 0;\n",
    "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(j);\n",
    "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\ntensor C dim 3 rank 1;\nA(i) = B(i) + C(0);\n",
    "tensor A dim 3 rank 2 sym(0,1);\ntensor B dim 3 rank 2;\nA(i, j) = B(i, j);\n",
    "tensor A dim 3 rank 2;\ntensor B dim 3 rank 2;\nA(sym<0,1>, i, j) = B(i, j);\n",
    "tensor A dim 3 rank 1;\ntensor B dim 4 rank 1;\nA(a) = B(a);\n",
    "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(i+1);\n",
    "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(i)/B(i);\n",
    "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = sqrt(B(i));\n",
    "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) *= B(i);\n",
    "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(i) + Sum(j, B(i));\n",
    "tensor A dim 3 rank 1;\ntensor B dim 3 rank 2;\nA(i) = B(i);\n",
    "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(3) = B(0);\n",
    "tensor dh dim 3 rank 1 inner rank 2 sym(0,1);\ntensor B dim 3 rank 1;\ndh(i)(j, k) = B(i);\n",
    "tensor g dim 3 rank 2 sym(0,1);\ntensor B dim 3 rank 1;\ng(sym<0,1>, i, 0) = B(i);\n",
    "tensor g dim 3 rank 2 sym(0,1);\ntensor B dim 3 rank 1;\ng(i, 0) = B(i);\n",
]


def seeded(program, targets, n, seed):
    env = bench.make_env(program, targets[0], n, seed)
    for t in targets:
        env[t].data[:] = 0.0
    return env


def describe(program, vs):
    tensors = {}
    for it in program.items:
        if isinstance(it, TensorDecl):
            shape = program.decls.tensors[it.name]
            from tlang.codegen_c import ArgDescriptor

            arg = ArgDescriptor("rhs", it.name, "R", shape.dim, shape.outer_rank,
                                shape.inner_rank, shape.outer_sym, shape.inner_sym)
            tensors[it.name] = {
                "outer_count": shape.outer_count,
                "inner_count": shape.inner_count,
                "alias": _combined_alias(arg),
            }
    stmts = []
    for v in vs:
        stmts.append({
            "signature": signature(v),
            "count_data": list(count_data(v)),
            "lhs_order": [[b[var] for var in v.lhs_vars] for b in v.lhs_assignments()],
            "loop_sym": [list(p) for p in v.loop_sym.inequalities],
            "args": [[a.role, a.name, a.param] for a in collect_args(v)],
        })
    return {"tensors": tensors, "statements": stmts, "render": render(program)}


def make_case(name, source, n, seed=SEED, per_component_check=True, sizes=None,
              expect_error=False):
    res = parse_program(source)
    assert res.ok, (name, res.diagnostics)
    program = res.program
    vs = [validate_statement(s, program.decls) for s in program.statements]
    targets = list(dict.fromkeys(v.stmt.lhs.field for v in vs))
    env = seeded(program, targets, n, seed)
    if sizes:
        rng = np.random.default_rng(seed + 1)
        for fname, m in sizes.items():
            f = env[fname]
            f.data = rng.uniform(0.0, 1.0, f.data.shape[:-1] + (m,))
    if name in SPECIAL_CASES:
        for fname, f in env.items():
            if fname in targets:
                continue
            flat = f.data.reshape(-1)
            flat[: len(SPECIALS)] = SPECIALS
            if fname == "w":
                f.data[: len(SPECIALS)] = SPECIALS[::-1]
    if name in ARANGE_CASES:
        for t in targets:
            env[t].data[:] = np.arange(env[t].data.size, dtype=float).reshape(env[t].data.shape)
    (OUT / f"{name}.in.tldf").write_bytes(tldf.dumps(env))
    if per_component_check and len(vs) == 1:
        env2 = tldf.loads(tldf.dumps(env))
        eval_statement_per_component(vs[0], env2)
    error = None
    try:
        for v in vs:
            eval_statement(v, env)
    except Exception as exc:  # noqa: BLE001 — recorded, the point of the case
        if not expect_error:
            raise
        error = {"type": type(exc).__name__, "message": str(exc)}
    assert (error is not None) == expect_error, name
    if per_component_check and len(vs) == 1:
        a, b = env2[targets[0]].data, env[targets[0]].data
        assert a.tobytes() == b.tobytes(), name
    (OUT / f"{name}.out.tldf").write_bytes(tldf.dumps({t: env[t] for t in targets}))
    out = {"source": source, "N": n, "seed": seed, "targets": targets,
           **describe(program, vs)}
    if sizes:
        out["sizes"] = sizes
    if error is not None:
        out["raises"] = error
    return out


def main() -> None:
    for old in OUT.glob("*.tldf"):
        old.unlink()
    manifest = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg",
                "cases": {}}
    cases = manifest["cases"]
    for entry in bench.builtin_suite():
        cases[f"suite_{entry.name}"] = make_case(f"suite_{entry.name}", entry.source, 64)
    for entry in bench.worked_examples() + bench.contraction_demos()[:1]:
        cases[f"demo_{entry.name}"] = make_case(f"demo_{entry.name}", entry.source, 16)
    cases["c1_dtg"] = make_case("c1_dtg", DTG, 64)
    cases["c1_dtg_odd"] = make_case("c1_dtg_odd", DTG, 37)
    cases["c2_maxwell"] = make_case("c2_maxwell", MAXWELL, 100)
    cases["c3_christoffel"] = make_case("c3_christoffel", CHRISTOFFEL, 64)
    cases["c4_p2"] = make_case("c4_p2", P2, 64)
    cases["c4_p3"] = make_case("c4_p3", P3, 48)
    for name, (src, n) in EDGE.items():
        cases[name] = make_case(name, src, n, sizes=SIZES.get(name))
    for name, (src, n, sizes) in RAISES.items():
        cases[name] = make_case(name, src, n, sizes=sizes, expect_error=True)
    bad = []
    for src in BAD_PROGRAMS:
        res = parse_program(src)
        bad.append({"source": src,
                    "diagnostics": [[d.line, d.col, d.message] for d in res.diagnostics]})
    manifest["bad_programs"] = bad
    invalid = []
    for src in INVALID_STATEMENTS:
        res = parse_program(src)
        assert res.ok, (src, res.diagnostics)
        codes = []
        for s in res.program.statements:
            try:
                validate_statement(s, res.program.decls)
                codes.append(None)
            except ValidationError as exc:
                codes.append(exc.code)
        invalid.append({"source": src, "codes": codes})
    manifest["invalid_statements"] = invalid
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")
    size = sum(p.stat().st_size for p in OUT.glob("*.tldf"))
    print(f"{len(cases)} cases, {size / 1e6:.2f} MB of TLDF")


if __name__ == "__main__":
    main()
