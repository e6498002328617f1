"""Per-point pure-Python oracle — TEST INFRASTRUCTURE ONLY.

Restates the reference's independent naive oracle (pkg/tests/oracle.py:33-146):
for every canonical LHS assignment (filtered odometer, oracle.py:33-41) and
every grid point, the RHS is evaluated on Python floats; a Sum accumulates in
a plain loop starting from ``0.0`` (oracle.py:74-78 — note: NOT the
evaluator's "start from term 0" chain, so it agrees with the evaluator only
to ~1e-13 relative / up to the sign of a zero); ``touched`` collects the
(field, outer slot, inner slot) arrays used, which is the brute-force N_e.
Small sizes only (seconds at N <= 64).
"""

from __future__ import annotations

import math

import numpy as np

from .numpy_eval import _k, _leaf_slots, lhs_bindings, prepare


def _point(e, v, env, binding, x, touched):
    k = _k(e)
    if k == "Const":
        return float(e.value)
    if k == "FieldRef":
        if touched is not None:
            touched.add((e.name,))
        return float(env[e.name][x])
    if k == "Leaf":
        o, i = _leaf_slots(v, e.leaf, binding)
        if touched is not None:
            touched.add((e.leaf.field, o, i))
        return float(env[e.leaf.field][o, i, x])
    if k in ("Add", "Sub", "Mul", "Div"):
        a = _point(e.l, v, env, binding, x, touched)
        b = _point(e.r, v, env, binding, x, touched)
        if k == "Add":
            return a + b
        if k == "Sub":
            return a - b
        if k == "Mul":
            return a * b
        if b == 0.0:
            return float(np.float64(a) / np.float64(b))
        return a / b
    if k == "Neg":
        return -_point(e.e, v, env, binding, x, touched)
    if k == "Sqrt":
        a = _point(e.e, v, env, binding, x, touched)
        return math.sqrt(a) if a >= 0 else float("nan")
    if k == "Sum":
        total = 0.0
        for val in range(e.var.dim):
            total += _point(e.body, v, env, {**binding, e.var: val}, x, touched)
        return total
    raise TypeError(f"not an expression node: {e!r}")


def run(v, env, touched: set | None = None) -> dict:
    """Execute one statement point by point on a dict of numpy arrays;
    returns the number of writes per (outer, inner) target component."""
    with np.errstate(all="ignore"):
        n = prepare(v, env)
        lhs = v.stmt.lhs
        writes: dict = {}
        for binding in lhs_bindings(v):
            o, i = _leaf_slots(v, lhs, binding)
            writes[(o, i)] = writes.get((o, i), 0) + 1
            if touched is not None:
                touched.add((lhs.field, o, i))
            tgt = env[lhs.field]
            for x in range(n):
                val = _point(v.stmt.rhs, v, env, binding, x, touched)
                cur = float(tgt[o, i, x])
                op = v.stmt.op
                if op == "=":
                    new = val
                elif op == "+=":
                    new = cur + val
                elif op == "-=":
                    new = cur - val
                elif op == "*=":
                    new = cur * val
                else:
                    new = float(np.float64(cur) / np.float64(val))
                tgt[o, i, x] = new
    return writes
