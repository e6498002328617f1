"""Shared test helpers: golden cases, host/device environments, comparisons."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def manifest() -> dict:
    return json.loads((GOLDEN / "manifest.json").read_text())


def case_names() -> list[str]:
    return sorted(manifest()["cases"])


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
