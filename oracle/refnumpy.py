"""Run the reference package's own numpy evaluator — TEST/BASELINE
INFRASTRUCTURE ONLY (bench.py's CPU legs; never the product path).

The paper's "NonAccel" CPU path is the reference's ``eval_statement``
(pkg/src/tlang/evaluator.py:204-236): per canonical LHS component one numpy
pass per expression node, optionally over grid chunks on a thread pool
(``chunk=..., threads=...``, :213-236).  This module imports that package
UNMODIFIED — from oracle/_ref/tlang (copied there by oracle/build_ref.py, so
it travels to the GPU box like the compiled oracle/_ref/*.so), or from
/root/reference/pkg/src in the build container — and drives it exactly as
the reference's CLI does (cli.py:93-99: statements in order over one env of
its own TensorField/ScalarField objects).
"""

from __future__ import annotations

import importlib
import math
import sys
from pathlib import Path

REF_COPY = Path(__file__).resolve().parent / "_ref"
REF_SRC = Path("/root/reference/pkg/src")


def available() -> bool:
    return (REF_COPY / "tlang" / "evaluator.py").exists() or (REF_SRC / "tlang").exists()


def _tlang():
    if "tlang" not in sys.modules:
        for root in (REF_COPY, REF_SRC):
            if (root / "tlang" / "evaluator.py").exists():
                sys.path.insert(0, str(root))
                break
        else:
            raise FileNotFoundError("reference package not found: run python oracle/build_ref.py")
    return importlib.import_module("tlang")


class RefNumpyProgram:
    """A program parsed and validated by the reference package itself."""

    def __init__(self, text: str):
        _tlang()
        from tlang.ir import validate_statement
        from tlang.parser import parse_program

        res = parse_program(text)
        if res.diagnostics:
            raise ValueError(res.diagnostics)
        self.program = res.program
        self.vs = [validate_statement(s, self.program.decls) for s in self.program.statements]

    def env(self, arrays: dict) -> dict:
        """Reference fields wrapping the given float64 arrays (no copy):
        tensors ``(outer, inner, N)``, scalar fields ``(N,)``."""
        from tlang.fields import ScalarField, TensorField

        env = {}
        for name, shape in self.program.decls.tensors.items():
            f = TensorField(name, shape, 0)
            f.data = arrays[name]
            env[name] = f
        for name in self.program.decls.scalar_fields:
            f = ScalarField(name, 0)
            f.data = arrays[name]
            env[name] = f
        return env

    def run(self, env: dict, threads: int = 1) -> None:
        """Every statement in order (cli.py:93-99); ``threads > 1`` uses the
        reference's own chunked thread pool with one chunk per thread."""
        from tlang.evaluator import eval_statement

        for v in self.vs:
            if threads > 1:
                n = env[v.stmt.lhs.field].gridsize or 1
                for name in env:
                    n = max(n, getattr(env[name], "gridsize", 0))
                eval_statement(v, env, chunk=max(1, math.ceil(n / threads)), threads=threads)
            else:
                eval_statement(v, env)
