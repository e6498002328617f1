"""Stand-in IR classes with the reference's class and attribute names but
no relation to this package's classes — used to show the evaluator accepts
trees built by another implementation of the IR (the reference's own
tlang.ir in a real drop-in)."""

from dataclasses import dataclass
from typing import Any


@dataclass(frozen=True)
class Fixed:
    value: int


@dataclass(frozen=True)
class VarTerm:
    var: Any
    offset: int = 0


@dataclass(frozen=True)
class TensorLeaf:
    field: str
    outer: tuple
    inner: tuple = ()
    declared_sym: Any = None


@dataclass(frozen=True)
class Leaf:
    leaf: TensorLeaf


@dataclass(frozen=True)
class Const:
    value: float


@dataclass(frozen=True)
class FieldRef:
    name: str


@dataclass(frozen=True)
class Add:
    l: Any
    r: Any


@dataclass(frozen=True)
class Sub:
    l: Any
    r: Any


@dataclass(frozen=True)
class Mul:
    l: Any
    r: Any


@dataclass(frozen=True)
class Div:
    l: Any
    r: Any


@dataclass(frozen=True)
class Neg:
    e: Any


@dataclass(frozen=True)
class Sqrt:
    e: Any


@dataclass(frozen=True)
class Sum:
    var: Any
    body: Any


@dataclass(frozen=True)
class Statement:
    lhs: TensorLeaf
    op: str
    rhs: Any


class Decls:
    def __init__(self, tensors, scalars):
        self.tensors, self.scalar_fields = tensors, scalars

    def tensor(self, name):
        return self.tensors[name]


class Validated:
    def __init__(self, stmt, decls, lhs_shape, lhs_vars, loop_sym, assignments):
        self.stmt, self.decls, self.lhs_shape = stmt, decls, lhs_shape
        self.lhs_vars, self.loop_sym, self._assign = lhs_vars, loop_sym, assignments

    def lhs_assignments(self):
        return iter(self._assign)


def _terms(ts):
    return tuple(Fixed(t.value) if type(t).__name__ == "Fixed" else VarTerm(t.var, t.offset)
                 for t in ts)


def _leaf(lf):
    return TensorLeaf(lf.field, _terms(lf.outer), _terms(lf.inner), lf.declared_sym)


def _expr(e):
    k = type(e).__name__
    if k == "Leaf":
        return Leaf(_leaf(e.leaf))
    if k == "Const":
        return Const(e.value)
    if k == "FieldRef":
        return FieldRef(e.name)
    if k in ("Add", "Sub", "Mul", "Div"):
        return globals()[k](_expr(e.l), _expr(e.r))
    if k in ("Neg", "Sqrt"):
        return globals()[k](_expr(e.e))
    return Sum(e.var, _expr(e.body))


def convert(v):
    stmt = Statement(_leaf(v.stmt.lhs), v.stmt.op, _expr(v.stmt.rhs))
    decls = Decls(dict(v.decls.tensors), set(v.decls.scalar_fields))
    return Validated(stmt, decls, v.lhs_shape, v.lhs_vars, v.loop_sym, list(v.lhs_assignments()))
