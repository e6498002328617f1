"""Numpy restatement of the reference evaluator — TEST INFRASTRUCTURE ONLY.

Follows ``tlang.evaluator.eval_statement`` (pkg/src/tlang/evaluator.py):

* _prepare   (evaluator.py:180-201): RHS gridsize agreement, ``=`` resizes
  the target (zero-filled), ``op=`` on a mismatched target is an error;
* the LHS loop (evaluator.py:222-228) runs over canonical components in
  storage order (symmetry.py:122-145: slot 0 fastest, slot p bounded
  below by its paired higher slot);
* _eval       (evaluator.py:122-147): one float64 numpy op per node over
  the whole grid, literals as Python floats, ``sqrt`` as ``np.sqrt``, a
  Sum as ``acc = body[0]; acc = acc + body[k]`` (evaluator.py:142-146);
* _store      (evaluator.py:150-161): ``= += -= *= /=`` on the component.

It shares no code with the product package: component numbering is
recomputed here by filtering full odometer enumerations against the raw
inequality pairs (the technique of the reference's own independent oracle,
pkg/tests/oracle.py:33-41).  IR nodes are read by class name, so trees
from the reference package or from ``paper_1804_10120_b200`` both work.

An environment is a plain dict ``name -> np.ndarray`` (tensor fields
``(outer_count, inner_count, N)``, scalar fields ``(N,)``).
"""

from __future__ import annotations

from functools import lru_cache
from itertools import product

import numpy as np


class OracleError(RuntimeError):
    pass


def _pairs(sym) -> tuple:
    if sym is None:
        return ()
    return tuple(tuple(p) for p in sym.inequalities)


def odometer(dims, pairs):
    """Value tuples (slot 0 fastest) satisfying v[p] >= v[q] for each pair."""
    out = []
    for rev in product(*[range(d) for d in reversed(dims)]):
        vals = tuple(reversed(rev))
        if all(vals[p] >= vals[q] for p, q in pairs):
            out.append(vals)
    return out


def _linked(pairs, rank):
    """Slot classes under the pair relation (breadth-first search)."""
    adj = {s: set() for s in range(rank)}
    for p, q in pairs:
        adj[p].add(q)
        adj[q].add(p)
    seen, classes = set(), []
    for s in range(rank):
        if s in seen:
            continue
        todo, cls = [s], []
        seen.add(s)
        while todo:
            a = todo.pop(0)
            cls.append(a)
            for b in sorted(adj[a]):
                if b not in seen:
                    seen.add(b)
                    todo.append(b)
        classes.append(sorted(cls))
    return classes


@lru_cache(maxsize=None)
def _table(dim, rank, pairs):
    return {vals: n for n, vals in enumerate(odometer((dim,) * rank, pairs))}


def group_slot(dim, rank, pairs, idx) -> int:
    """Storage slot of a multi-index of one group (its representative's
    position in the filtered odometer)."""
    idx = list(idx)
    for cls in _linked(pairs, rank):
        vals = sorted((idx[s] for s in cls), reverse=True)
        for s, v in zip(cls, vals):
            idx[s] = v
    return _table(dim, rank, pairs)[tuple(idx)]


def group_count(dim, rank, pairs) -> int:
    return len(_table(dim, rank, pairs))


class Shape:
    """Plain-data copy of a tensor shape."""

    def __init__(self, shape):
        self.dim = shape.dim
        self.outer_rank = shape.outer_rank
        self.inner_rank = shape.inner_rank
        self.outer_pairs = _pairs(shape.outer_sym)
        self.inner_pairs = _pairs(shape.inner_sym)
        self.outer_count = group_count(self.dim, self.outer_rank, self.outer_pairs)
        self.inner_count = group_count(self.dim, self.inner_rank, self.inner_pairs)

    def slots(self, outer, inner):
        return (group_slot(self.dim, self.outer_rank, self.outer_pairs, outer),
                group_slot(self.dim, self.inner_rank, self.inner_pairs, inner))


def _k(node) -> str:
    return type(node).__name__


def _val(term, binding) -> int:
    return term.value if _k(term) == "Fixed" else binding[term.var] + term.offset


def _leaf_slots(v, leaf, binding):
    shape = Shape(v.decls.tensors[leaf.field])
    return shape.slots([_val(t, binding) for t in leaf.outer],
                       [_val(t, binding) for t in leaf.inner])


def lhs_bindings(v):
    """Canonical LHS assignments in storage order (ir.py:237-241)."""
    dims = tuple(var.dim for var in v.lhs_vars)
    for vals in odometer(dims, _pairs(v.loop_sym)):
        yield dict(zip(v.lhs_vars, vals))


def _field_names(e, out):
    k = _k(e)
    if k == "Leaf":
        name = e.leaf.field
    elif k == "FieldRef":
        name = e.name
    else:
        name = None
    if name is not None and name not in out:
        out.append(name)
    if k in ("Add", "Sub", "Mul", "Div"):
        _field_names(e.l, out)
        _field_names(e.r, out)
    elif k in ("Neg", "Sqrt"):
        _field_names(e.e, out)
    elif k == "Sum":
        _field_names(e.body, out)
    return out


def _get(env, name):
    if name not in env:
        raise OracleError(f"{name!r} is not present in the data environment")
    return env[name]


def prepare(v, env) -> int:
    """evaluator.py:180-201 on a dict of arrays (resizes in the dict)."""
    target = v.stmt.lhs.field
    lhs = _get(env, target)
    sizes = [(_get(env, n).shape[-1]) for n in _field_names(v.stmt.rhs, [])]
    if len(set(sizes)) > 1:
        raise OracleError("right-hand-side fields disagree on gridsize")
    n = sizes[0] if sizes else lhs.shape[-1]
    if sizes and n == 0:
        raise OracleError("field used in arithmetic before it holds data")
    if lhs.shape[-1] != n:
        if v.stmt.op != "=":
            raise OracleError("cannot resize")
        env[target] = np.zeros(lhs.shape[:-1] + (n,))
    return n


def _eval(e, v, env, binding, lo, hi):
    k = _k(e)
    if k == "Const":
        return e.value
    if k == "FieldRef":
        return env[e.name][lo:hi]
    if k == "Leaf":
        o, i = _leaf_slots(v, e.leaf, binding)
        return env[e.leaf.field][o, i, lo:hi]
    if k == "Add":
        return _eval(e.l, v, env, binding, lo, hi) + _eval(e.r, v, env, binding, lo, hi)
    if k == "Sub":
        return _eval(e.l, v, env, binding, lo, hi) - _eval(e.r, v, env, binding, lo, hi)
    if k == "Mul":
        return _eval(e.l, v, env, binding, lo, hi) * _eval(e.r, v, env, binding, lo, hi)
    if k == "Div":
        return _eval(e.l, v, env, binding, lo, hi) / _eval(e.r, v, env, binding, lo, hi)
    if k == "Neg":
        return -_eval(e.e, v, env, binding, lo, hi)
    if k == "Sqrt":
        return np.sqrt(_eval(e.e, v, env, binding, lo, hi))
    if k == "Sum":
        acc = _eval(e.body, v, env, {**binding, e.var: 0}, lo, hi)
        for val in range(1, e.var.dim):
            acc = acc + _eval(e.body, v, env, {**binding, e.var: val}, lo, hi)
        return acc
    raise OracleError(f"not an expression node: {e!r}")


def eval_statement(v, env, lo: int = 0, hi: int | None = None) -> None:
    """Execute one statement on a dict of numpy arrays, in place.  With
    ``lo/hi`` only grid points [lo, hi) are computed (slab checks)."""
    n = prepare(v, env)
    hi = n if hi is None else hi
    lhs = v.stmt.lhs
    op = v.stmt.op
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        for binding in lhs_bindings(v):
            o, i = _leaf_slots(v, lhs, binding)
            values = _eval(v.stmt.rhs, v, env, binding, lo, hi)
            tgt = env[lhs.field]
            if op == "=":
                tgt[o, i, lo:hi] = values
            elif op == "+=":
                tgt[o, i, lo:hi] += values
            elif op == "-=":
                tgt[o, i, lo:hi] -= values
            elif op == "*=":
                tgt[o, i, lo:hi] *= values
            else:
                tgt[o, i, lo:hi] /= values


def eval_program(vs, env, lo: int = 0, hi: int | None = None) -> None:
    for v in vs:
        eval_statement(v, env, lo, hi)


def data_count(v) -> tuple[int, int]:
    """(N_e, N_d) by brute-force enumeration (ir.py:453-482 restated)."""
    touched = set()

    def visit(e, binding):
        k = _k(e)
        if k == "Leaf":
            touched.add((e.leaf.field, *_leaf_slots(v, e.leaf, binding)))
        elif k == "FieldRef":
            touched.add((e.name,))
        elif k in ("Add", "Sub", "Mul", "Div"):
            visit(e.l, binding)
            visit(e.r, binding)
        elif k in ("Neg", "Sqrt"):
            visit(e.e, binding)
        elif k == "Sum":
            for val in range(e.var.dim):
                visit(e.body, {**binding, e.var: val})

    def consts(e) -> int:
        k = _k(e)
        if k in ("Add", "Sub", "Mul", "Div"):
            return consts(e.l) + consts(e.r)
        if k in ("Neg", "Sqrt"):
            return consts(e.e)
        if k == "Sum":
            return consts(e.body)
        return int(k == "Const")

    for b in lhs_bindings(v):
        touched.add((v.stmt.lhs.field, *_leaf_slots(v, v.stmt.lhs, b)))
        visit(v.stmt.rhs, b)
    return len(touched), consts(v.stmt.rhs)


def max_rel_error(a, b) -> float:
    """tl_compare's measure (pkg/harness/tl_compare.c:86-101,
    pkg/tests/oracle.py:138-146): max |a-b| / max(|a|,|b|), 0 where both 0."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    scale = np.maximum(np.abs(a), np.abs(b))
    with np.errstate(invalid="ignore", divide="ignore"):
        rel = np.where(scale > 0, np.abs(a - b) / np.where(scale > 0, scale, 1.0), 0.0)
    return float(np.nanmax(rel)) if rel.size else 0.0


def same_bits(a, b, nan_payload: bool = False) -> bool:
    """Bitwise equality of two float64 arrays; NaNs compare equal to NaNs
    (any payload) unless ``nan_payload``."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    ia, ib = a.view(np.uint64), b.view(np.uint64)
    if nan_payload:
        return bool((ia == ib).all())
    both_nan = np.isnan(a) & np.isnan(b)
    return bool(((ia == ib) | both_nan).all())
