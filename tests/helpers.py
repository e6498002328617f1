"""Shared test helpers: golden cases, host/device environments, comparisons."""

from __future__ import annotations

import json
import random
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def manifest() -> dict:
    return json.loads((GOLDEN / "manifest.json").read_text())


def case_names() -> list[str]:
    return sorted(manifest()["cases"])


def run_case(case: dict, fn, exact: bool = True) -> None:
    """Run ``fn`` (a whole golden program); when the reference stopped
    part-way through (``case["raises"]``), expect that error — same type
    name and message when ``exact`` (the product), any error otherwise (the
    CPU oracle) — the targets are then compared as the reference left them."""
    import pytest

    want = case.get("raises")
    if not want:
        fn()
        return
    with pytest.raises(Exception) as ei:
        fn()
    if exact:
        assert type(ei.value).__name__ == want["type"], ei.value
        assert str(ei.value) == want["message"]


def program(source: str):
    from paper_1804_10120_b200.ir import validate_statement
    from paper_1804_10120_b200.parser import parse_program

    res = parse_program(source)
    assert res.ok, res.diagnostics
    prog = res.program
    return prog, [validate_statement(s, prog.decls) for s in prog.statements]


def read_host(path: Path) -> dict:
    """TLDF → dict name -> np.ndarray (host copies)."""
    from paper_1804_10120_b200 import tldf

    fields = tldf.read(path, device="cpu")
    return {k: f.data.numpy().copy() for k, f in fields.items() if hasattr(f, "data")}


def golden_io(name: str) -> tuple[dict, dict]:
    return read_host(GOLDEN / f"{name}.in.tldf"), read_host(GOLDEN / f"{name}.out.tldf")


def device_env(prog, host: dict, device="cuda") -> dict:
    """Fields of this package on `device` filled from host arrays."""
    import torch
    from paper_1804_10120_b200.fields import ScalarField, TensorField

    env = {}
    for name, shape in prog.decls.tensors.items():
        f = TensorField(name, shape, 0, device=device)
        f.data = torch.from_numpy(host[name].copy()).to(device)
        env[name] = f
    for name in prog.decls.scalar_fields:
        f = ScalarField(name, 0, device=device)
        f.data = torch.from_numpy(host[name].copy()).to(device)
        env[name] = f
    return env


def same_bits(a, b) -> bool:
    """Bitwise equality modulo NaN payloads."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    eq = a.view(np.uint64) == b.view(np.uint64)
    return bool((eq | (np.isnan(a) & np.isnan(b))).all())


class NumpyTensorField:
    """Stand-in with the reference TensorField's surface (numpy-backed
    ``data`` (outer, inner, N), ``shape``, ``gridsize``, ``resize``) — what a
    user of the reference package hands to the drop-in evaluator."""

    def __init__(self, name, shape, data):
        self.name, self.shape, self.data = name, shape, data

    @property
    def gridsize(self):
        return self.data.shape[2]

    def resize(self, n):
        if n != self.gridsize:
            self.data = np.zeros(self.data.shape[:2] + (n,))


class NumpyScalarField:
    def __init__(self, name, data):
        self.name, self.data = name, data

    @property
    def gridsize(self):
        return self.data.shape[0]

    def resize(self, n):
        if n != self.gridsize:
            self.data = np.zeros(n)


def numpy_env(prog, host: dict) -> dict:
    env = {}
    for name, shape in prog.decls.tensors.items():
        env[name] = NumpyTensorField(name, shape, host[name].copy())
    for name in prog.decls.scalar_fields:
        env[name] = NumpyScalarField(name, host[name].copy())
    return env


def env_to_host(env: dict) -> dict:
    out = {}
    for k, f in env.items():
        d = f.data
        out[k] = d.copy() if isinstance(d, np.ndarray) else d.detach().cpu().numpy().copy()
    return out


RANDOM_DECLS = """tensor A dim 3 rank 1;
tensor B dim 3 rank 2;
tensor S dim 3 rank 2 sym(0,1);
tensor D dim 3 rank 2 sym(0,1) inner rank 1;
tensor T dim 3 rank 2;
tensor U dim 3 rank 2 sym(0,1);
field w;
"""


def random_program(rng, n_statements: int = 2) -> str:
    """Random valid statements over RANDOM_DECLS (free indices i, j)."""

    def scal(depth):
        opts = ["w", "2.5", "sqrt(w)", "(w + 1)", "Sum(k, A(k))", "-w", "0.125"]
        if depth > 0:
            a, b = scal(depth - 1), scal(depth - 1)
            opts += [f"({a}*{b})", f"({a} - {b})", f"({a}/({b} + 3))"]
        return opts[rng.integers(len(opts))]

    def vec(depth, sym_ok=True):
        opts = ["B(i, j)", "B(j, i)", "S(i, j)", "S(j, i)", "A(i)*A(j)", "T(i, j)", "T(j, i)",
                "U(j, i)", "Sum(k, B(i, k)*B(k, j))", "Sum(k, D(i, j)(k))",
                "Sum(k, D(i, k)(j)*A(k))", "Sum(l, Sum(k, S(i, k)*B(k, l)*S(l, j)))"]
        if depth > 0:
            a, b = vec(depth - 1), vec(depth - 1)
            s = scal(depth - 1)
            opts += [f"({a} + {b})", f"({a} - {b})", f"{s}*{a}", f"{a}/({s} + 2)", f"-{a}",
                     f"{a}*{s}"]
        return opts[rng.integers(len(opts))]

    lines = []
    for _ in range(n_statements):
        target = ["T(i, j)", "U(sym<0,1>, i, j)"][rng.integers(2)]
        op = ["=", "=", "+=", "-=", "*=", "/="][rng.integers(6)]
        rhs = scal(2) if op in ("*=", "/=") else vec(2)
        if op in ("*=", "/="):
            rhs = f"({rhs} + 1.5)"
        lines.append(f"{target} {op} {rhs};")
    return RANDOM_DECLS + "\n".join(lines) + "\n"


def random_host_env(prog, n: int, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape in prog.decls.tensors.items():
        out[name] = rng.uniform(0.0, 1.0, (shape.outer_count, shape.inner_count, n))
    for name in prog.decls.scalar_fields:
        out[name] = rng.uniform(0.0, 1.0, n)
    return out


FUZZ_DECLS = ("tensor A dim 3 rank 1;\ntensor B dim 3 rank 2;\ntensor S dim 3 rank 2 sym(0,1);\n"
         "tensor D dim 3 rank 2 sym(0,1) inner rank 1;\ntensor Q dim 4 rank 2 sym(0,1);\n"
         "tensor R dim 4 rank 3 sym(1,2);\nfield w;\nconst cc = 1.5;\nindex p: 2;\n")

LEAVES = {
    "i": ["A(i)", "B(i, 1)", "S(0, i)", "D(i, i)(0)", "Sum(j, B(i, j)*A(j))",
          "Sum(k, D(i, k)(k))", "A(p+1)*0 + A(i)", "B(i, p)*0 + A(i)"],
    "ij": ["B(i, j)", "B(j, i)", "S(i, j)", "S(j, i)", "A(i)*A(j)", "Sum(k, B(i, k)*S(k, j))",
           "D(i, j)(0)", "Sum(k, D(j, i)(k)*A(k))", "B(i+0, j)"],
    "ijk": ["D(i, j)(k)", "D(j, k)(i)", "A(i)*B(j, k)", "Sum(l, D(i, l)(k)*B(l, j))"],
    "ab": ["Q(a, b)", "Q(b, a)", "Sum(c, Q(a, c)*Q(c, b))", "R(0, a, b)", "R(a, b, 3)"],
    "abc": ["R(a, b, c)", "R(a, c, b)", "Q(a, b)*Q(c, 0)", "Sum(d, R(a, d, b)*Q(d, c))"],
}
LHS = [("A(i)", "i"), ("B(i, j)", "ij"), ("S(sym<0,1>, i, j)", "ij"), ("B(i, 0)", "i"),
       ("D(i, j)(k)", "ijk"), ("Q(sym<0,1>, a, b)", "ab"), ("R(a, sym<1,2>, b, c)", "abc"),
       ("R(sym<1,2>, a, b, c)", "abc"), ("S(i, j)", "ij"), ("B(i, i)", "i")]
SCALARS = ["w", "cc", "2", "0.25", "sqrt(w)", "(w + 1)", "Sum(i, A(i))", "S(0, 1)", "Q(0, 3)",
           "-w", "(w*w - cc)"]


def fuzz_statement(rng: random.Random) -> str:
    """One random statement over FUZZ_DECLS (mostly valid, some not)."""
    def scal(d):
        if d == 0 or rng.random() < 0.5:
            return rng.choice(SCALARS)
        return f"({scal(d - 1)} {rng.choice('+-*/')} {scal(d - 1)})"

    def vec(free, d):
        if d == 0 or rng.random() < 0.35:
            return rng.choice(LEAVES[free])
        r = rng.random()
        if r < 0.3:
            return f"({vec(free, d - 1)} {rng.choice('+-')} {vec(free, d - 1)})"
        if r < 0.5:
            return f"{scal(1)}*{vec(free, d - 1)}"
        if r < 0.65:
            return f"{vec(free, d - 1)}/{scal(1)}"
        if r < 0.8:
            return f"-{vec(free, d - 1)}"
        return f"{vec(free, d - 1)}*{scal(1)}"

    lhs, free = rng.choice(LHS)
    op = rng.choice(["=", "=", "+=", "-=", "*=", "/="])
    rhs = scal(2) if op in ("*=", "/=") or rng.random() < 0.05 else vec(free, 3)
    if rng.random() < 0.05:  # an occasional invalid mutation
        rhs = rhs.replace("(i", "(z", 1).replace("(a", "(i", 1)
    return f"{lhs} {op} {rhs};\n"
