"""Lowering: validated tensor statements → one fused sm_100a kernel.

This is the step the reference performs as text emission
(``codegen_cuda.emit_cuda``, pkg/src/tlang/codegen_cuda.py:135-204, whose
kernels are never launched) re-designed around what a B200 wants:

* **one thread step = one grid point (or two, with 128-bit accesses)**, not
  one thread per (point, LHS component): all canonical LHS components of a
  point are produced by the same thread, so every input component is
  loaded from HBM exactly once per point and the reference's sequential
  component-loop semantics (reads of the target see components written
  earlier in the loop) hold per point for free;
* **compile-time index resolution**: LHS bindings are enumerated in
  ``lhs_assignments`` (iter_canonical) order, Sum indices are substituted
  while walking (an inner Sum over a bound index shadows it,
  evaluator.py:83-85), every leaf is resolved to its canonical component
  ``o*inner_count + i`` (ir.leaf_component) — the kernel holds no index
  arithmetic and no pointer arrays;
* **exact arithmetic order**: the RHS is emitted in parse-tree order and a
  ``Sum`` as the left-associated chain ``body[0] + body[1] + ...``
  starting from term 0 (evaluator.py:142-146), each operation one IEEE
  fp64 op; NVRTC runs with ``--fmad=false`` so no DFMA contraction can
  change a rounding.  Constant-only subtrees are folded *with the very
  Python/numpy scalar semantics the reference evaluator applies to them*
  (Python floats, ``np.sqrt`` → ``np.float64``), so even their corner
  cases (ZeroDivisionError on a literal ``1/0``) match;
* **register shadow**: within a point, the current value of every
  (field, component) the program touched lives in an SSA register; later
  reads (same statement through permuted/symmetric indices, or later
  statements of a program, S10/S11) read the register, and each written
  component is stored once, after its last write.  This makes a whole
  *program* of statements one kernel with the same
  bits as running the statements one by one;
* value numbering removes repeated identical operations (bitwise safe: no
  reassociation, no commutation).

The lowering reads IR nodes by class name and attribute names only, so a
statement built by the reference ``tlang`` package lowers as well.
"""

from __future__ import annotations

import hashlib
import math
import os
import struct
from dataclasses import dataclass, field as dc_field
from pathlib import Path
from typing import Any, Mapping, Sequence

import numpy as np

from .symmetry import SymmetrySpec, iter_canonical, slot_index

TEMPLATE_PATH = Path(__file__).with_name("csrc") / "tlk_template.cuh"
LOWERING_VERSION = "tlk-1"
MAX_PARAM_SLOTS = 4000  # 8 + 8*4000 bytes <= 32764-byte parameter block (CUDA >= 12.1, sm_70+)

SLOT_READ = 1
SLOT_WRITE = 2


class LoweringError(ValueError):
    pass


# ------------------------------------------------------------ duck typing --


def kind(node: Any) -> str:
    return type(node).__name__


def as_sym(sym: Any) -> SymmetrySpec:
    if sym is None:
        return SymmetrySpec()
    if isinstance(sym, SymmetrySpec):
        return sym
    return SymmetrySpec(tuple(tuple(p) for p in sym.inequalities))


@dataclass(frozen=True)
class FieldInfo:
    """A field the kernel touches (program-wide numbering)."""

    name: str
    is_tensor: bool
    dim: int = 0
    outer_rank: int = 0
    inner_rank: int = 0
    outer_sym: SymmetrySpec = SymmetrySpec()
    inner_sym: SymmetrySpec = SymmetrySpec()
    outer_count: int = 1
    inner_count: int = 1

    @property
    def n_components(self) -> int:
        return self.outer_count * self.inner_count

    def component(self, outer: Sequence[int], inner: Sequence[int]) -> int:
        o = slot_index(self.dim, self.outer_rank, self.outer_sym, outer)
        i = slot_index(self.dim, self.inner_rank, self.inner_sym, inner)
        return o * self.inner_count + i


def tensor_info(name: str, shape: Any) -> FieldInfo:
    from .symmetry import component_count

    osym, isym = as_sym(shape.outer_sym), as_sym(shape.inner_sym)
    return FieldInfo(
        name, True, shape.dim, shape.outer_rank, shape.inner_rank, osym, isym,
        component_count(shape.dim, shape.outer_rank, osym),
        component_count(shape.dim, shape.inner_rank, isym),
    )


# ---------------------------------------------------------------- SSA IR --


@dataclass
class Instr:
    op: str  # "ld" | "add" | "sub" | "mul" | "div" | "neg" | "sqrt" | "st"
    dst: int = -1  # register (not for "st")
    a: Any = None  # operand: int register or _Lit
    b: Any = None
    slot: int = -1  # "ld" / "st"


@dataclass(frozen=True)
class _Lit:
    """A folded constant, kept as the exact Python object the reference's
    evaluator would hold (float or np.float64)."""

    value: Any

    def c_text(self) -> str:
        x = float(self.value)
        if math.isfinite(x):
            return f"({x.hex()})"
        bits = struct.unpack("<q", struct.pack("<d", x))[0]
        return f"(__longlong_as_double({bits}LL))"


@dataclass
class KernelPlan:
    """Everything a launch needs besides the field addresses."""

    source: str
    fields: list[FieldInfo]
    slot_field: list[int]
    slot_comp: list[int]
    slot_flags: list[int]
    flops_per_point: int  # algorithmic: binary ops (+ sqrt) after Sum expansion
    n_ops: int  # emitted arithmetic instructions after value numbering
    statements: int
    key: str = ""
    lhs_fields: list[int] = dc_field(default_factory=list)
    variant: "Variant | None" = None
    phases: int = 1
    # launches of at most variant.small_n points use small_variant (and, when
    # its code generation differs, small_plan's kernel): see Variant.small_class
    small_variant: "Variant | None" = None
    small_plan: "KernelPlan | None" = None

    @property
    def n_slots(self) -> int:
        return len(self.slot_field)

    @property
    def reads(self) -> int:
        return sum(1 for f in self.slot_flags if f & SLOT_READ)

    @property
    def writes(self) -> int:
        return sum(1 for f in self.slot_flags if f & SLOT_WRITE)

    @property
    def bytes_per_point(self) -> int:
        """Algorithmic HBM bytes per grid point: each read component once,
        each written component once (read-modify-write counts twice)."""
        return 8 * (self.reads + self.writes)


# --------------------------------------------------------------- builder --


class _Builder:
    def __init__(self) -> None:
        self.instrs: list[Instr] = []
        self.nreg = 0
        self.vn: dict[tuple, int] = {}
        self.slots: dict[tuple[int, int], int] = {}
        self.slot_flags: list[int] = []
        self.shadow: dict[int, Any] = {}  # slot -> current operand
        self.flops = 0
        self.chained = 0  # reads served by the register shadow of a written slot
        self.groups = 1  # output groups (Variant.vn = 1: one device function each)

    def slot(self, f: int, c: int) -> int:
        key = (f, c)
        if key not in self.slots:
            self.slots[key] = len(self.slots)
            self.slot_flags.append(0)
        return self.slots[key]

    def reg(self) -> int:
        self.nreg += 1
        return self.nreg - 1

    def read(self, f: int, c: int):
        s = self.slot(f, c)
        if self.slot_flags[s] & SLOT_WRITE:
            self.chained += 1
        if s not in self.shadow:
            r = self.reg()
            self.instrs.append(Instr("ld", r, slot=s))
            self.slot_flags[s] |= SLOT_READ
            self.shadow[s] = r
        return self.shadow[s]

    def begin_group(self) -> None:
        """Start a new output group (Variant.vn = 1): its instructions become
        a separate non-inlined device function, so nothing — loaded inputs,
        shared subexpressions — stays live from one group into the next, and
        the compiler cannot merge a group's recomputed subexpressions with an
        earlier group's.  Only for programs whose outputs never read a
        written slot (the register shadow then holds loads only)."""
        self.instrs.append(Instr("grp"))
        self.groups += 1
        self.vn.clear()
        self.shadow.clear()

    def snapshot(self):
        return len(self.instrs), dict(self.vn), dict(self.shadow), self.flops

    def rollback(self, snap) -> None:
        n, vn, shadow, flops = snap
        del self.instrs[n:]
        self.vn, self.shadow, self.flops = vn, shadow, flops

    def write(self, f: int, c: int, val) -> None:
        s = self.slot(f, c)
        self.slot_flags[s] |= SLOT_WRITE
        if isinstance(val, _Lit):
            # a literal stored into a field becomes a float64 array element in
            # the reference (evaluator.py:150-161); later reads of it take part
            # in numpy array arithmetic under errstate(divide/invalid="ignore")
            # (evaluator.py:224) — IEEE inf/nan, never a Python
            # ZeroDivisionError — so the shadow keeps np.float64 semantics
            val = _Lit(np.float64(val.value))
        self.shadow[s] = val
        self.instrs.append(Instr("st", a=val, slot=s))

    def binary(self, op: str, a, b):
        if isinstance(a, _Lit) and isinstance(b, _Lit):
            return _Lit(_fold_binary(op, a.value, b.value))
        self.flops += 1
        key = (op, _vn_key(a), _vn_key(b))
        r = self.vn.get(key)
        if r is None:
            r = self.reg()
            self.instrs.append(Instr(op, r, a, b))
            self.vn[key] = r
        return r

    def unary(self, op: str, a):
        if isinstance(a, _Lit):
            if op == "neg":
                return _Lit(-a.value)
            with np.errstate(all="ignore"):
                return _Lit(np.sqrt(a.value))
        if op == "sqrt":
            self.flops += 1
        key = (op, _vn_key(a))
        r = self.vn.get(key)
        if r is None:
            r = self.reg()
            self.instrs.append(Instr(op, r, a))
            self.vn[key] = r
        return r


def _vn_key(x):
    # literals by bit pattern: 0.0 and -0.0 must not be merged
    if isinstance(x, _Lit):
        return ("c", struct.pack("<d", float(x.value)))
    return x


def _fold_binary(op: str, x, y):
    # the reference evaluates literal-only subtrees on Python scalars
    # (evaluator.py:124-141); reproduce that exactly, exceptions included
    with np.errstate(all="ignore"):
        if op == "add":
            return x + y
        if op == "sub":
            return x - y
        if op == "mul":
            return x * y
        return x / y  # ZeroDivisionError for Python-float operands, as in the reference


_BIN = {"Add": "add", "Sub": "sub", "Mul": "mul", "Div": "div"}


class _Lowerer:
    def __init__(self, alias: Mapping[str, str] | None):
        self.b = _Builder()
        self.fields: list[FieldInfo] = []
        self.index: dict[str, int] = {}
        self.alias = dict(alias or {})

    def field(self, name: str, info_fn) -> int:
        rep = self.alias.get(name, name)
        k = self.index.get(rep)
        if k is None:
            k = len(self.fields)
            self.index[rep] = k
            self.fields.append(info_fn(rep))
        return k

    def tensor(self, v, name: str) -> int:
        k = self.field(name, lambda n: tensor_info(n, v.decls.tensor(name)))
        if not self.fields[k].is_tensor:
            raise LoweringError(f"{name!r} is used as a tensor and as a scalar field")
        return k

    def scalar(self, name: str) -> int:
        k = self.field(name, lambda n: FieldInfo(n, False))
        if self.fields[k].is_tensor:
            raise LoweringError(f"{name!r} is used as a tensor and as a scalar field")
        return k

    @staticmethod
    def term_value(t, binding) -> int:
        return t.value if kind(t) == "Fixed" else binding[t.var] + t.offset

    def leaf_slot(self, v, leaf, binding) -> tuple[int, int]:
        f = self.tensor(v, leaf.field)
        info = self.fields[f]
        outer = [self.term_value(t, binding) for t in leaf.outer]
        inner = [self.term_value(t, binding) for t in leaf.inner]
        return f, info.component(outer, inner)

    def expr(self, v, e, binding):
        k = kind(e)
        if k == "Const":
            return _Lit(e.value)
        if k == "Leaf":
            return self.b.read(*self.leaf_slot(v, e.leaf, binding))
        if k == "FieldRef":
            return self.b.read(self.scalar(e.name), 0)
        op = _BIN.get(k)
        if op is not None:
            a = self.expr(v, e.l, binding)
            return self.b.binary(op, a, self.expr(v, e.r, binding))
        if k == "Neg":
            return self.b.unary("neg", self.expr(v, e.e, binding))
        if k == "Sqrt":
            return self.b.unary("sqrt", self.expr(v, e.e, binding))
        if k == "Sum":
            acc = self.expr(v, e.body, {**binding, e.var: 0})
            for val in range(1, e.var.dim):
                acc = self.b.binary("add", acc, self.expr(v, e.body, {**binding, e.var: val}))
            return acc
        raise LoweringError(f"not an expression node: {e!r}")

    def statement(self, v, only: set[int] | None = None, budget: int = 0) -> None:
        """Lower one statement, its canonical LHS components in storage order.
        ``budget`` > 0 splits the outputs into groups (Builder.begin_group)
        whose bodies keep at most ~budget values live (_max_live): an output
        that would push the current group past it starts the next group."""
        stmt = v.stmt
        dims = tuple(var.dim for var in v.lhs_vars)
        for n, values in enumerate(iter_canonical(dims, as_sym(v.loop_sym))):
            if only is not None and n not in only:
                continue
            binding = dict(zip(v.lhs_vars, values))
            snap = self.b.snapshot() if budget else None
            self.component(v, binding)
            if budget:
                start = max((k for k, i in enumerate(self.b.instrs[:snap[0]]) if i.op == "grp"),
                            default=-1) + 1
                had_output = any(i.op == "st" for i in self.b.instrs[start:snap[0]])
                if had_output and _max_live(self.b.instrs[start:]) > budget:
                    self.b.rollback(snap)
                    self.b.begin_group()
                    self.component(v, binding)

    def component(self, v, binding) -> None:
        stmt = v.stmt
        f, c = self.leaf_slot(v, stmt.lhs, binding)
        rhs = self.expr(v, stmt.rhs, binding)
        if stmt.op == "=":
            val = rhs
        else:
            cur = self.b.read(f, c)
            val = self.b.binary(_AUG[stmt.op], cur, rhs)
        self.b.write(f, c, val)


_AUG = {"+=": "add", "-=": "sub", "*=": "mul", "/=": "div"}
_CSYM = {"add": "+", "sub": "-", "mul": "*", "div": "/"}


def _operand(x) -> str:
    return x.c_text() if isinstance(x, _Lit) else f"v{x}"


def _emit_body(instrs: list[Instr], slot_flags: list[int], hoist_loads: bool = False,
               restrict: bool = True, direct: set[int] | frozenset = frozenset()) -> list[str]:
    """C++ text of the per-point body.

    With ``restrict`` (default) the body is a function of one
    ``__restrict__`` pointer per slot: distinct (field, component) slots
    never overlap (components of a field are ``pitch >= n`` apart, fields
    are distinct allocations, aliased names were merged into one field), so
    the compiler may issue every load as early as register pressure allows
    instead of keeping each load behind the preceding stores.  Loads of a
    slot only ever precede its stores (the register shadow serves reads
    after writes), so no load may legally move *after* a store of its own
    slot, and none is asked to.  ``hoist_loads`` additionally places all
    loads first in the source.
    """
    if any(ins.op == "grp" for ins in instrs):
        return _emit_groups(instrs, slot_flags, hoist_loads, restrict, direct)
    # keep only the final store of every slot; earlier values were consumed
    # through the register shadow
    last = {}
    for k, ins in enumerate(instrs):
        if ins.op == "st":
            last[ins.slot] = k
    nslots = len(slot_flags)
    if restrict:
        params = ", ".join(
            ("double* __restrict__" if slot_flags[j] & SLOT_WRITE else
             "const double* __restrict__") + f" p{j}" for j in range(nslots))
        out = ["template <typename T, int LD = TLK_LDMODE>",
               f"__device__ __forceinline__ void tlk_body(const long long x, {params}) {{"]
        ptr = "p{}".format
    else:
        out = ["template <typename T, int LD = TLK_LDMODE, typename P>",
               "__device__ __forceinline__ void tlk_point(const P& P_, const long long x) {"]
        ptr = "P_.p[{}]".format
    if hoist_loads:
        # SSA + one load per slot before any store of that slot: loads may
        # all be issued first (maximum memory-level parallelism)
        instrs = [i for i in instrs if i.op == "ld"] + [i for i in instrs if i.op != "ld"]
        last = {ins.slot: k for k, ins in enumerate(instrs) if ins.op == "st"}
    for k, ins in enumerate(instrs):
        if ins.op == "ld":
            # `direct` slots bypass the staged entry's ring: under LD 3 they
            # still load from global memory
            ld = "(LD == 3 ? 1 : LD)" if ins.slot in direct else "LD"
            out.append(f"  const T v{ins.dst} = tl_ld<T, {ld}>({ptr(ins.slot)} + x);")
        elif ins.op == "st":
            if last[ins.slot] != k:
                continue
            val = ins.a
            src = f"tl_splat<T>{val.c_text()}" if isinstance(val, _Lit) else f"v{val}"
            out.append(f"  tl_st({ptr(ins.slot)} + x, {src});")
        elif ins.op in _CSYM:
            out.append(f"  const T v{ins.dst} = {_operand(ins.a)} {_CSYM[ins.op]} "
                       f"{_operand(ins.b)};")
        elif ins.op == "neg":
            out.append(f"  const T v{ins.dst} = -{_operand(ins.a)};")
        elif ins.op == "sqrt":
            out.append(f"  const T v{ins.dst} = tl_sqrt({_operand(ins.a)});")
        else:  # pragma: no cover
            raise LoweringError(f"bad instruction {ins}")
    out.append("}")
    if restrict:
        args = ", ".join(f"P_.p[{j}]" for j in range(nslots))
        out += ["template <typename T, int LD = TLK_LDMODE, typename P>",
                "__device__ __forceinline__ void tlk_point(const P& P_, const long long x) {",
                f"  tlk_body<T, LD>(x, {args});", "}"]
    return out


def _emit_instr(ins: Instr, ptr, direct, keep_store: bool) -> str | None:
    if ins.op == "ld":
        ld = "(LD == 3 ? 1 : LD)" if ins.slot in direct else "LD"
        return f"  const T v{ins.dst} = tl_ld<T, {ld}>({ptr(ins.slot)} + x);"
    if ins.op == "st":
        if not keep_store:
            return None
        val = ins.a
        src = f"tl_splat<T>{val.c_text()}" if isinstance(val, _Lit) else f"v{val}"
        return f"  tl_st({ptr(ins.slot)} + x, {src});"
    if ins.op in _CSYM:
        return f"  const T v{ins.dst} = {_operand(ins.a)} {_CSYM[ins.op]} {_operand(ins.b)};"
    if ins.op == "neg":
        return f"  const T v{ins.dst} = -{_operand(ins.a)};"
    if ins.op == "sqrt":
        return f"  const T v{ins.dst} = tl_sqrt({_operand(ins.a)});"
    raise LoweringError(f"bad instruction {ins}")  # pragma: no cover


def _emit_groups(instrs: list[Instr], slot_flags: list[int], hoist_loads: bool,
                 restrict: bool, direct, inline: bool = False, point: bool = True) -> list[str]:
    """Body of a program lowered in output groups (Variant.vn = 1): one
    ``__noinline__`` device function per group, each loading what it reads
    (through the kernel's parameter block, passed by reference:
    ``__grid_constant__`` in the flat entries, so no copy), computing with its
    own value numbering and storing its outputs; ``tlk_point`` calls them in
    order.  Separate functions are what keeps ptxas from re-merging the
    subexpressions groups recompute (its CSE sees through any inline asm).

    ``inline`` (statement parts, Variant.split): the groups are independent
    statement parts with no field in common — ``__forceinline__`` functions,
    and ``tlk_part(part, P_, x)`` runs one of them (tlk_flat_v1 under
    TLK_PARTS); ``point=False`` leaves ``tlk_point`` to the fused body."""
    last = {ins.slot: k for k, ins in enumerate(instrs) if ins.op == "st"}
    groups: list[list[tuple[int, Instr]]] = [[]]
    for k, ins in enumerate(instrs):
        if ins.op == "grp":
            groups.append([])
        else:
            groups[-1].append((k, ins))
    out: list[str] = []
    for g, items in enumerate(groups):
        used = sorted({ins.slot for _, ins in items if ins.op in ("ld", "st")})
        attr = "__forceinline__" if inline else "__noinline__"
        out += ["template <typename T, int LD, typename P>",
                f"__device__ {attr} void tlk_grp{g}(const P& P_, const long long x) {{"]
        if restrict:
            for j in used:
                q = "double* __restrict__" if slot_flags[j] & SLOT_WRITE else \
                    "const double* __restrict__"
                out.append(f"  {q} p{j} = P_.p[{j}];")
            ptr = "p{}".format
        else:
            ptr = "P_.p[{}]".format
        if hoist_loads:
            items = [t for t in items if t[1].op == "ld"] + [t for t in items if t[1].op != "ld"]
        for k, ins in items:
            line = _emit_instr(ins, ptr, direct, last.get(ins.slot) == k)
            if line is not None:
                out.append(line)
        out.append("}")
    if point:
        out += ["template <typename T, int LD = TLK_LDMODE, typename P>",
                "__device__ __forceinline__ void tlk_point(const P& P_, const long long x) {"]
        out += [f"  tlk_grp{g}<T, LD>(P_, x);" for g in range(len(groups))]
        out.append("}")
    if inline:
        out += ["template <typename T, int LD = TLK_LDMODE, typename P>",
                "__device__ __forceinline__ void tlk_part(const unsigned part, const P& P_, "
                "const long long x) {",
                "  switch (part) {"]
        out += [f"    case {g}: tlk_grp{g}<T, LD>(P_, x); break;" for g in range(len(groups))]
        out += ["  }", "}"]
    return out


_TEMPLATE_CACHE: list[str] = []


def template_text() -> str:
    if not _TEMPLATE_CACHE:
        _TEMPLATE_CACHE.append(TEMPLATE_PATH.read_text())
    return _TEMPLATE_CACHE[0]


@dataclass(frozen=True)
class Variant:
    """Code-generation and launch choices of one fused kernel.

    restrict  per-slot ``__restrict__`` body parameters (always legal: slots
              never overlap)
    hoist     every load first in the body source
    ldmode    0 ``ld.global.cs``; 1 ``ld.global.nc.L1::no_allocate`` as a
              side-effect-free asm the compiler may move freely — only legal
              when no slot is both read and written (a load could otherwise
              sink below a later store of its own slot), enforced here
    vec       2 = two points per thread step (128-bit accesses), 1 = one
    waves     grid = waves x SMs x resident blocks (grid-stride loop); 0 = a
              one-shot grid: one block per `threads` points (pairs), every
              thread one loop trip (lowering policy 3)
    """

    restrict: bool = True
    hoist: bool = False
    ldmode: int = 0
    vec: int = 2
    waves: int = 1
    batch_vec: int = 1  # batch entry: points per thread (1, 2), or 3 = the staged batch entry
    batch_ptrs: int = 0  # TLK_BATCH_PTRS: 0 shared-memory staging, 1 direct table reads
    batch_threads: int = 0  # block size of the plain batch entries (0 = threads)
    small_n: int = 0  # launches of <= small_n points run small_class() (0: never)
    stage: int = 0  # >0: TMA-staged entry tlk_stage_v1 with a `stage`-deep tile ring
    threads: int = 256  # TLK_THREADS: block size of the flat and batch entries
    stage_threads: int = 128  # TLK_STAGE_THREADS: the staged entry's block = tile (points)
    stage_reads: int = 0  # read slots copied through the ring (0 = all; the rest load directly)
    minb: int = 0  # TLK_MINB: min resident blocks/SM of the flat entries (0 = unconstrained)
    stage_ws: int = 0  # TLK_STAGE_WS: staged entry with a dedicated producer warp (1) or not (0)
    batch_bound: int = 0  # TLK_BATCH_BOUND: the batch entries' __launch_bounds__ (0 = threads)
    vn: int = 0  # 1: outputs split into groups, one non-inlined device function each
    chunk: int = 1  # TLK_CHUNK: block-sized runs of points per block (tlk_flat_v1; tuning)
    split: int = 0  # 1: independent statement parts run one after another (TLK_PARTS)
    batch_split: int = 0  # 1: the 1-point batch entry runs the parts as row runs too

    def tag(self) -> str:
        t = (f"r{int(self.restrict)}h{int(self.hoist)}l{self.ldmode}"
             f"v{self.vec}w{self.waves}b{self.batch_vec}{self.batch_ptrs}")
        t += f"s{self.small_n.bit_length() - 1}" if self.small_n else ""
        t += f"k{self.batch_threads}" if self.batch_threads else ""
        t += f"g{self.stage}x{self.stage_threads}" if self.stage else ""
        t += f"r{self.stage_reads}" if self.stage and self.stage_reads else ""
        t += f"m{self.minb}" if self.minb else ""
        t += "p" if self.stage and self.stage_ws else ""
        t += f"q{self.batch_bound}" if self.batch_bound else ""
        t += "u" if self.vn else ""
        t += f"c{self.chunk}" if self.chunk > 1 else ""
        t += "y" if self.split else ""
        t += "z" if self.split and self.batch_split else ""
        return t + (f"n{self.threads}" if self.threads != 256 else "")

    def small_class(self) -> "Variant":
        """Choices for launches of at most ``small_n`` points, where a
        thread's dependent memory round trips, not bandwidth, set the time
        (profiles/r01/tune_smalln.jsonl, tune_cross.jsonl):

        * light kernels hoist every load to the top of the body — one
          round trip per point instead of one per statement: Maxwell at
          10^3-10^5 points 2.3-2.5x faster back to back, C1 at 64^3 1.1x,
          both 1-4 % faster at 2^20;
        * heavier kernels run one point per thread over 4 waves (a launch-
          time choice, same cubin): twice the threads in flight — C3 at
          64^3 16.4 vs 18.4 us for the staged entry; from 2^21 points the
          staged entry is ahead (profiles/r01/r01t/tune_smalln.jsonl)."""
        if self.vec == 1 and not self.stage:
            return Variant(**{**self.__dict__, "hoist": True, "small_n": 0})
        if self.waves == 0 and not self.stage:  # one-shot grids are already one wave here
            return Variant(**{**self.__dict__, "vec": 1, "small_n": 0})
        return Variant(**{**self.__dict__, "vec": 1, "waves": 4, "small_n": 0})

    def same_code(self, other: "Variant") -> bool:
        """Whether two variants compile to the same cubin (vec/waves are
        launch-time choices; both entry points are in every module)."""
        return ((self.restrict, self.hoist, self.ldmode, self.batch_ptrs, self.stage,
                 self.threads, self.stage_threads, self.stage_reads, self.minb, self.stage_ws,
                 self.batch_bound, self.vn, self.chunk, self.split, self.batch_split)
                == (other.restrict, other.hoist, other.ldmode, other.batch_ptrs, other.stage,
                    other.threads, other.stage_threads, other.stage_reads, other.minb,
                    other.stage_ws, other.batch_bound, other.vn, other.chunk, other.split,
                    other.batch_split))


def choose_variant(reads: int, writes: int, n_ops: int, rw_slots: int,
                   chained: int, statements: int = 1,
                   policy: int | None = None) -> Variant:
    """Default per-kernel choice — a policy fitted to measurements on B200
    (profiles/r01/tune_*.jsonl: 12 variants x 8 programs at 2^24-2^26 points).

    * light kernels (at most ~1.5 arithmetic ops per streamed array: C1,
      Maxwell, K_ij) are pure streams: one point per thread (8-byte
      accesses, twice the threads in flight) over 4 waves of blocks —
      +5-7 % over the 2-point variant;
    * heavier kernels keep 2 points per thread (128-bit accesses).  When no
      slot is both read and written, loads are made freely movable (the
      compiler schedules them against register pressure instead of behind
      earlier stores: +2 % on P2, +8 % on the write-heavy outer products);
      when statements also chain through registers (P3: Γ → ∇β → ∂t g)
      every load is hoisted to the top, otherwise each statement's loads
      wait for the previous statement's stores (2.1x on P3);
    * with read-modify-write slots the restrict-free 2-point body over 4
      waves is used;
    * the multi-domain batch entry always runs one point per thread with the
      domain's slot pointers staged in shared memory (small 16^3 domains:
      twice the blocks in flight hide the per-domain pointer fetch; C4 P2
      5.64 -> 6.10 TB/s, P3 chain 5.10 -> 5.87 TB/s, profiles/r01/tune_batch.jsonl),
      in 128-thread blocks for the heavier kernels (C4 P2 163.8 -> 159.7 us,
      P3 200.7 -> 196.6 us, profiles/r01/tune_batch_threads.jsonl);
    * above the small-N class, read-only-input programs run the TMA-staged
      entry (tlk_stage_v1): a 3-deep shared-memory ring fed by one bulk copy
      per staged read slot per tile, the remaining read slots loaded
      directly — both in flight together.  256-point tiles; light kernels
      stage half their reads, heavier ones three quarters (0.85 for
      non-chained programs of 32+ reads, whose ring then takes a whole SM).
      Measured against the plain entries at 2^24-2^26
      (profiles/r01/tune_stage_frac.jsonl, back to back): C1 +2-3 %,
      Maxwell +5-6 %, C3 +6-7 %, P2 +5-9 %, P3 0-3 %; P2 at 2^28 102.3 %
      of measured copy bandwidth (34 of 40 reads staged) vs 101.1 % (30 of
      40, 128-point tiles) and 99.1 % plain (profiles/r01/bench_stage_*).
      Staging every read caps P2 below the plain kernel.

    Round 2 (policy 2, the default; ``policy=1`` or TLK_POLICY=1 gives the
    round-1 choices above): the staged entry runs warp-specialised
    (``stage_ws``: a producer warp issues the bulk copies, consumer warps
    release a stage through an mbarrier instead of a block-wide barrier per
    tile).  Interleaved A/B on B200 (profiles/r02/tune_ab_*.jsonl, medians
    of 7 rounds x 10 launches, 2^24-2^28 points), against policy 1:

    * light single-statement kernels: 3-deep ring, warp-specialised —
      C1 +2.0 %, add1-3 +2.5-4.4 %, K_ij +2.0 %; multi-statement light
      programs keep the block-barrier ring (Maxwell, 8 statements: -1.6 to
      -2.0 % warp-specialised, and no staged share or ring depth recovers it);
    * heavier kernels of < 32 reads (C3): 3-deep ring of 256-point tiles,
      three quarters of the reads staged, warp-specialised: +1.3-2.8 %;
    * 32-48 reads (P2, P3): a 2-deep ring of 256-point tiles (0.85 / 0.75 of
      the reads), warp-specialised: P2 +1.9-2.6 % (2^24-2^28), P3 +1.0 %;
      the 3-deep warp-specialised ring is 2-4 % SLOWER than policy 1 on
      these, the 2-deep one faster;
    * more reads than that (the contractions: 90-108 reads, 81 writes) were
      left unstaged by policy 1 (a 3-deep ring of three quarters of their
      reads leaves 4 warps per SM); now 40 of them are staged through a
      2-deep ring of 128-point tiles (80 KB: 2 blocks per SM):
      contract1 +7.7 %, contract2 +32 %.
    """
    if policy is None:
        policy = int(os.environ.get("TLK_POLICY", "3"))
    arrays = reads + writes
    if policy >= 3:
        return _policy3(reads, writes, n_ops, rw_slots, chained)
    # the staged entries unroll per-slot loops: beyond a few hundred slots
    # (unmeasured territory, slow NVRTC compiles) the plain entries are used
    # write-dominated programs stream better through the plain entries
    # (outer products, copies: -3..-13 % staged, profiles/r01/tune_suite.jsonl)
    stageable = rw_slots == 0 and arrays <= STAGE_MAX_SLOTS and reads > writes
    if n_ops <= 1.5 * arrays:
        if not stageable:
            return Variant(restrict=True, hoist=False, ldmode=0, vec=1, waves=4,
                           small_n=SMALL_N_LIGHT)
        return Variant(restrict=True, hoist=True, ldmode=0, vec=1, waves=4,
                       small_n=SMALL_N_LIGHT, stage=3, stage_threads=256,
                       stage_reads=max(1, (reads + 1) // 2),
                       stage_ws=int(policy >= 2 and statements < 4))
    if rw_slots == 0:
        share = 0.85 if reads >= 32 and not chained else 0.75
        staged = max(1, round(share * reads))
        depth, tile = 3, 256
        if policy >= 2 and reads >= 32:
            depth = 2
            if staged > 40:  # contraction-class: 40 staged reads, 128-point tiles
                staged, tile = 40, 128
        return Variant(restrict=True, hoist=chained > 0, ldmode=1, vec=2, waves=4 if chained else 1,
                       small_n=SMALL_N_HEAVY, stage=depth if stageable else 0, stage_threads=tile,
                       stage_reads=staged, batch_threads=128, stage_ws=int(policy >= 2))
    return Variant(restrict=False, hoist=False, ldmode=0, vec=2, waves=4)


def _policy3(reads: int, writes: int, n_ops: int, rw_slots: int, chained: int) -> Variant:
    """Lowering policy 3 (round 2, the default): every kernel is the plain
    per-point entry over a ONE-SHOT grid (``waves=0``: one block per
    `threads` points, no grid-stride loop).  Persistent grid-stride grids —
    the plain entries' 1-4 waves and the TMA-staged entry's persistent ring
    alike — lose 2-36 % to it on this part: in interleaved A/B runs
    (profiles/r02/tuning/tune_ab_oneshot_*.jsonl, 2^21 and 2^26 points) the
    one-shot flat entry beats policy 2 (warp-specialised TMA rings) on C1
    +2.4 %, Maxwell +2.9 %, C3 +3-4 %, P2 +1.4-3.5 %, P3 +4-5 %, K_ij
    +6.5 %, contract1 +5 %, and the write-dominated programs the most
    (outer3 +36 %, assign3 +21 % at 2^26).  The device's own streaming probes
    agree (scripts/stream_probe.cu): pure writes 7.61 TB/s one-shot vs
    5.9-6.3 TB/s persistent with every store flavour, 256-bit stores and TMA
    bulk stores; copies 6.97 vs 6.08 TB/s.

    * light (<= 1.5 ops per streamed array, copies and the write-dominated
      outer products included): 1 point per thread, 512-thread blocks, every
      load hoisted to the top of the body — at 2^21-2^26 points the best of
      8 launch shapes on every write-dominated program
      (profiles/r02/tuning/tune_ab_write_dominated.jsonl: outer3 +66 %,
      assign1 +23 %, assign3 +21 %, outer1 +10 %, outer2 +8 % over policy
      2), and no size class: below ~300K points the runtime shrinks a
      one-shot grid's blocks so every SM gets ~4 (tlb_runtime launch_flat);
    * heavier: 1 point per thread, 128-thread blocks (register-heavy
      bodies: finer block granularity — P2 +0.3-4 %, P3 +17-23 %, contract1
      +3-4 % over 256 threads);
    * read-modify-write slots (`op=` statements, or a program that writes a
      field it also reads): 1 point per thread, 128-thread blocks, every
      load hoisted, no restrict.
    Loads stay as fitted in round 1 (hoisted for light and chained programs,
    movable ld.global.nc for heavier read-only ones).  The TMA-staged entry
    remains available as a variant (``stage``), bit-exact and tested."""
    arrays = reads + writes
    if rw_slots:
        # every load hoisted (the loads are not movable: ld.global.cs beside
        # stores of the same slots), one point per thread, 128-thread blocks:
        # +7-40 % over policy 2's 2-point 4-wave grid at 2^26
        # (profiles/r02/tuning/tune_ab_read_modify_write.jsonl: A+=B +9 %,
        # A*=2 +9 %, Gamma+= +40 %, dtg+= +7 %)
        return Variant(restrict=False, hoist=True, ldmode=0, vec=1, waves=0, threads=128,
                       batch_threads=256, batch_bound=256)
    # the multi-domain batch entries are unchanged from policy 2 (256-thread
    # launch bounds; 256- / 128-thread blocks): the flat entries' block size
    # must not change their code (P2's batch entry compiled for 128-thread
    # bounds took 88 instead of 106 registers and ran C4 in 173 vs 160 us)
    if n_ops <= 1.5 * arrays:
        return Variant(restrict=True, hoist=True, ldmode=0, vec=1, waves=0, threads=512,
                       batch_threads=256, batch_bound=256)
    # (no size class: a one-shot grid of 1-point threads is already the
    # round-1 small-N choice for heavier kernels)
    return Variant(restrict=True, hoist=chained > 0, ldmode=1, vec=1, waves=0, threads=128,
                   batch_threads=128, batch_bound=256)


# dynamic shared memory budget of the staged entry's tile ring (bytes; the
# 227 KB per-block maximum less room for the static mbarriers)
STAGE_SMEM_MAX = 224 * 1024

# largest program (read + written component arrays) the policy stages
STAGE_MAX_SLOTS = 256
# fewest resident warps per SM the policy accepts for a staged ring
STAGE_MIN_WARPS = 8


def _stage_warps(variant: "Variant", staged: int) -> int:
    """Warps per SM the staged entry can keep resident: blocks limited by the
    ring's shared memory (228 KB per SM, ~1 KB reserved per block) and by
    2048 threads per SM."""
    ring = variant.stage * max(staged, 1) * variant.stage_threads * 8
    blocks = min(228 * 1024 // (ring + 1024), 2048 // variant.stage_threads)
    return blocks * variant.stage_threads // 32

# size classes (Variant.small_class): largest launch, in points, that still
# runs the small-N choices — the crossovers in profiles/r01/tune_cross.jsonl
SMALL_N_LIGHT = 1 << 21
SMALL_N_HEAVY = 1 << 20  # the staged entry already wins at 2^21 (r01t/tune_smalln.jsonl)


def _env_variant(v: Variant) -> Variant:
    """TLK_* environment overrides (tuning experiments, scripts/tune_kernel.py)."""
    env = os.environ
    kw = {}
    if "TLK_RESTRICT" in env:
        kw["restrict"] = env["TLK_RESTRICT"] == "1"
    if "TLK_HOIST" in env:
        kw["hoist"] = env["TLK_HOIST"] == "1"
    if "TLK_LDMODE" in env:
        kw["ldmode"] = int(env["TLK_LDMODE"])
    if "TLK_VEC" in env:
        kw["vec"] = int(env["TLK_VEC"])
    if "TLK_WAVES" in env:
        kw["waves"] = int(env["TLK_WAVES"])
    if "TLK_BATCH_VEC" in env:
        kw["batch_vec"] = int(env["TLK_BATCH_VEC"])
    if "TLK_BATCH_PTRS" in env:
        kw["batch_ptrs"] = int(env["TLK_BATCH_PTRS"])
    if "TLK_BATCH_THREADS" in env:
        kw["batch_threads"] = int(env["TLK_BATCH_THREADS"])
    if "TLK_STAGE" in env:
        kw["stage"] = int(env["TLK_STAGE"])
    if "TLK_THREADS" in env:
        kw["threads"] = int(env["TLK_THREADS"])
    if "TLK_STAGE_THREADS" in env:
        kw["stage_threads"] = int(env["TLK_STAGE_THREADS"])
    if "TLK_STAGE_READS" in env:
        kw["stage_reads"] = int(env["TLK_STAGE_READS"])
    if "TLK_MINB" in env:
        kw["minb"] = int(env["TLK_MINB"])
    if "TLK_STAGE_WS" in env:
        kw["stage_ws"] = int(env["TLK_STAGE_WS"])
    if "TLK_SPLIT" in env:
        kw["split"] = int(env["TLK_SPLIT"])
    if "TLK_BATCH_SPLIT" in env:
        kw["batch_split"] = int(env["TLK_BATCH_SPLIT"])
    if kw:
        kw["small_n"] = 0  # a forced variant applies at every size ...
    if "TLK_SMALL_N" in env:
        kw["small_n"] = int(env["TLK_SMALL_N"])  # ... unless asked otherwise
    return Variant(**{**v.__dict__, **kw}) if kw else v


def lower_program(statements: Sequence[Any], alias: Mapping[str, str] | None = None,
                  components: Sequence[set[int] | None] | None = None,
                  hoist_loads: bool | None = None, variant: Variant | None = None) -> KernelPlan:
    """Lower validated statements, executed in order per grid point, to one
    fused kernel.  ``alias`` maps field names to a representative name when
    several names address the same storage.  ``components`` optionally
    restricts statement k to the given LHS component ordinals (the paper's
    per-component "Arrays" pathway, evaluator.py:239-257).  ``variant``
    fixes the code-generation/launch choices (default: ``choose_variant``,
    then TLK_* environment overrides)."""
    if not statements:
        raise LoweringError("nothing to lower: no statements")

    def lower(budget: int, parts: list[list[int]] | None = None, layout_of=None):
        low = _Lowerer(alias)
        if layout_of is not None:
            # keep another lowering's field order (the callers' layout) and slot
            # numbering (one parameter block serves both lowerings' bodies)
            low.fields, low.index = list(layout_of.fields), dict(layout_of.index)
            low.b.slots = dict(layout_of.b.slots)
            low.b.slot_flags = [0] * len(layout_of.b.slots)
        lhs = []
        order = [list(range(len(statements)))] if parts is None else parts
        for p, ks in enumerate(order):
            if p:
                low.b.begin_group()
            for k in ks:
                v = statements[k]
                lhs.append(low.tensor(v, v.stmt.lhs.field))
                low.statement(v, None if components is None else components[k], budget)
        return low, lhs

    low, lhs_fields = lower(0)
    if variant is not None and variant.vn and not low.b.chained and not any(
            f == SLOT_READ | SLOT_WRITE for f in low.b.slot_flags):
        low, lhs_fields = lower(VN_LIVE_BUDGET)
    b = low.b
    n_slots = len(b.slots)
    if n_slots > MAX_PARAM_SLOTS:
        raise LoweringError(f"program touches {n_slots} component arrays; at most "
                            f"{MAX_PARAM_SLOTS} fit one kernel parameter block")
    if n_slots == 0:
        raise LoweringError("statement writes no component")
    slot_field = [0] * n_slots
    slot_comp = [0] * n_slots
    for (f, c), s in b.slots.items():
        slot_field[s], slot_comp[s] = f, c
    n_ops = sum(1 for i in b.instrs if i.op not in ("ld", "st", "grp"))
    reads = sum(1 for f in b.slot_flags if f & SLOT_READ)
    writes = sum(1 for f in b.slot_flags if f & SLOT_WRITE)
    rw = sum(1 for f in b.slot_flags if f == SLOT_READ | SLOT_WRITE)
    phases = _phases(b.instrs)
    policy = variant is None
    if variant is None:
        chosen = choose_variant(reads, writes, n_ops, rw, b.chained, len(statements))
        if (int(os.environ.get("TLK_POLICY", "3")) >= 3 and len(statements) > 1
                and len(statement_parts(statements, alias)) > 1):
            # independent statement parts stream one after another (Variant.split):
            # +0.4-1.1 % on P2 and Maxwell at 2^21-2^28, -0.7 % at 2^18
            # (profiles/r02/tuning/tune_ab_split.jsonl)
            chosen = Variant(**{**chosen.__dict__, "split": 1})
        variant = _env_variant(chosen)
        if "TLK_STAGE_FRAC" in os.environ:  # tuning: staged share of the read slots
            frac = float(os.environ["TLK_STAGE_FRAC"])
            variant = Variant(**{**variant.__dict__,
                                 "stage_reads": max(1, round(frac * reads))})
        if _max_live(b.instrs) > VN_LIVE_TRIGGER and not rw and not b.chained:
            # program-wide value numbering keeps more values live than the
            # register file holds (contract3: 761 doubles — 729 products
            # shared across outputs — 5.7 KB of spills per thread): split the
            # outputs into groups of at most ~VN_LIVE_BUDGET live values, one
            # non-inlined device function each, recomputing what groups share
            # (every output's own operation sequence is unchanged: same bits)
            low2, lhs2 = lower(VN_LIVE_BUDGET)
            if low2.b.groups > 1:
                low, lhs_fields, b = low2, lhs2, low2.b
                variant = Variant(**{**variant.__dict__, "vn": 1})
                n_ops = sum(1 for i in b.instrs if i.op not in ("ld", "st", "grp"))
    parts = statement_parts(statements, alias) if variant.split else []
    if variant.split and (len(parts) < 2 or variant.vn or variant.chunk > 1 or variant.stage):
        # one part (or output groups / chunks / the staged ring already shape
        # the entry): no split
        variant = Variant(**{**variant.__dict__, "split": 0})
    if variant.split:
        # independent statement parts (no field in common): each part becomes
        # its own inlined body; tlk_flat_v1 gives every part its own run of
        # blocks, in order, so the parts stream one after another with fewer
        # concurrent DRAM streams each (the other entries run the parts in turn)
        fused = b  # the whole program's body: tlk_point, for every other entry
        low2, lhs2 = lower(0, parts, layout_of=low)
        if low2.b.slots != fused.slots or low2.b.slot_flags != fused.slot_flags:
            # one parameter block must serve both bodies; never expected
            variant = Variant(**{**variant.__dict__, "split": 0})
        elif policy and (min(_group_arrays(low2.b.instrs)) * variant.threads * 8
                         < SPLIT_MIN_BLOCK_BYTES):
            # a part that streams only a few arrays would run a full grid of
            # blocks with little work each: keep such programs fused
            variant = Variant(**{**variant.__dict__, "split": 0})
        else:
            low, lhs_fields, b = low2, lhs2, low2.b
    if hoist_loads is not None:
        variant = Variant(**{**variant.__dict__, "hoist": hoist_loads})
    if variant.ldmode == 1 and rw:
        variant = Variant(**{**variant.__dict__, "ldmode": 0})  # see Variant docstring
    if variant.stage and (rw or reads == 0):
        # a staged read-modify-write slot would be stored into its own tile;
        # a program that reads nothing has nothing to stage
        variant = Variant(**{**variant.__dict__, "stage": 0})
    if variant.stage:
        # the tile ring must fit the 227 KB a block can hold: shallower ring,
        # then smaller tiles; below two stages nothing overlaps, so the plain
        # entries are used instead
        tile = variant.stage_threads
        staged = min(reads, variant.stage_reads) if variant.stage_reads else reads
        depth = min(variant.stage, STAGE_SMEM_MAX // (8 * tile * max(staged, 1)))
        while depth < 2 and tile > 32:
            tile //= 2
            depth = min(variant.stage, STAGE_SMEM_MAX // (8 * tile * max(staged, 1)))
        if (depth, tile) != (variant.stage, variant.stage_threads):
            variant = Variant(**{**variant.__dict__, "stage": depth if depth >= 2 else 0,
                                 "stage_threads": tile})
        if policy and variant.stage and _stage_warps(variant, staged) < STAGE_MIN_WARPS:
            # a ring this large leaves too few warps per SM to consume it
            # (contract1, 90 reads: 4 warps, -13 %, profiles/r01/tune_suite.jsonl)
            variant = Variant(**{**variant.__dict__, "stage": 0})
    rord: list[int] = []
    if variant.stage:
        # TMA-staged entry: the first `stage_reads` read slots (all by
        # default) come through the shared-memory ring (tlk_point<double, 3>:
        # plain dereferences, LDS); the others load straight from global
        # memory (ld.global.nc: staged variants have no read-write slot)
        cap = variant.stage_reads or n_slots
        r = 0
        for fl in b.slot_flags:
            take = bool(fl & SLOT_READ) and r < cap
            rord.append(r if take else -1)
            r += 1 if take else 0
    direct = {j for j, o in enumerate(rord) if o < 0 and b.slot_flags[j] & SLOT_READ}
    if variant.split:
        # tlk_part (the parts: tlk_flat_v1's split runs) beside the fused
        # tlk_point that the 2-point, batch and staged entries keep: run per
        # point in turn, the parts cost C4's batch entry 23 % (160 -> 199 us)
        body = "\n".join(_emit_groups(b.instrs, b.slot_flags, variant.hoist, variant.restrict,
                                      direct, inline=True, point=False)
                         + _emit_body(fused.instrs, fused.slot_flags, variant.hoist,
                                      variant.restrict, direct))
    else:
        body = "\n".join(_emit_body(b.instrs, b.slot_flags, variant.hoist, variant.restrict,
                                    direct))
    header = [f"// generated by paper_1804_10120_b200.lowering ({LOWERING_VERSION})",
              f"// variant {variant.tag()}"]
    for v in statements:
        header.append("// " + _statement_comment(v))
    header.append(f"#define TLK_NSLOTS {n_slots}")
    header.append(f"#define TLK_THREADS {variant.threads}")
    # default flat-entry launch geometry for C-ABI callers that pass none
    # (tlb_exec_host: the host-staged path and the harness bindings)
    header.append(f"#define TLK_GRID_WAVES {variant.waves}")
    header.append(f"#define TLK_VEC {variant.vec}")
    if variant.minb:
        header.append(f"#define TLK_MINB {variant.minb}")
    if variant.batch_bound:
        header.append(f"#define TLK_BATCH_BOUND {variant.batch_bound}")
    if variant.chunk > 1:
        header.append(f"#define TLK_CHUNK {variant.chunk}")
    if variant.split:
        header.append(f"#define TLK_PARTS {b.groups}")
        if variant.batch_split:
            header.append("#define TLK_BATCH_SPLIT 1")
    if variant.stage:
        header.append(f"#define TLK_NSTAGE {variant.stage}")
        header.append(f"#define TLK_NREAD {len(rord) - rord.count(-1)}")
        header.append(f"#define TLK_STAGE_THREADS {variant.stage_threads}")
        header.append("#define TLK_RORD {" + ",".join(map(str, rord)) + "}")
        if variant.stage_ws:
            header.append("#define TLK_STAGE_WS 1")
        if variant.batch_vec == 3:
            header.append("#define TLK_STAGE_BATCH 1")
    header.append(f"#define TLK_LDMODE {variant.ldmode}")
    header.append(f"#define TLK_BATCH_PTRS {variant.batch_ptrs}")
    src = "\n".join(header) + "\n" + template_text().replace("// @@TLK_BODY@@", body)
    plan = KernelPlan(src, low.fields, slot_field, slot_comp, list(b.slot_flags), b.flops, n_ops,
                      len(statements), lhs_fields=lhs_fields, variant=variant, phases=phases)
    if variant.small_n:
        sv = variant.small_class()
        if sv.ldmode == 1 and rw:
            sv = Variant(**{**sv.__dict__, "ldmode": 0})
        plan.small_variant = sv
        if not variant.same_code(sv):
            plan.small_plan = lower_program(statements, alias, components, variant=sv)
    # identical source text can serve different slot maps (e.g. the
    # per-component kernels of one statement): the plan identity covers both
    ident = f"{src}\0{slot_field}\0{slot_comp}\0{plan.slot_flags}\0{variant.tag()}"
    plan.key = hashlib.sha256(ident.encode()).hexdigest()
    return plan


# largest number of simultaneously live values (doubles) program-wide value
# numbering may leave in a kernel before the lowering splits the outputs into
# groups (Variant.vn): 64 doubles = 128 registers leaves ptxas room for
# addresses and the call ABI (48 / 64: no spills in contract2/3; 96: 56 / 248
# bytes of spill stores; TLK_VN_BUDGET overrides, for tuning)
VN_LIVE_BUDGET = int(os.environ.get("TLK_VN_BUDGET", "64"))
# ... applied only when program-wide value numbering would keep more than this
# many values live: grouping costs recomputation, which pays where the
# ungrouped kernel spills heavily (contract3, 761 live: 58.4 -> 8.9 ms at
# 2^24) but not where it barely spills (contract2, 94 live, 56 B of stack:
# 5.08 -> 6.37 ms grouped; profiles/r02/tuning/tune_ab_output_groups.jsonl)
VN_LIVE_TRIGGER = 128


def _max_live(instrs: list[Instr]) -> int:
    """Peak number of simultaneously live SSA values when the body runs in
    source order (a value lives from its definition to its last use) — the
    register pressure the source order implies."""
    last: dict[int, int] = {}
    for k, ins in enumerate(instrs):
        for o in (ins.a, ins.b):
            if isinstance(o, int):
                last[o] = k
    live = peak = 0
    for k, ins in enumerate(instrs):
        for o in {ins.a, ins.b}:  # operands read at their last use die first
            if isinstance(o, int) and last.get(o) == k:
                live -= 1
        if ins.op not in ("st", "grp") and ins.dst >= 0:
            live += 1
            peak = max(peak, live)
            if ins.dst not in last:  # never used
                live -= 1
    return peak


# policy 3 splits a program into statement parts only when every part moves
# at least this many bytes per block (arrays x threads x 8 B, one point per
# thread).  Measured (profiles/r02/tuning/tune_ab_split*.jsonl, split vs
# fused at 2^24 / 2^26): Gamma + a 1-component copy (2 KB per 128-thread
# block) -13 %, + a vector copy (6 KB) -10 %, + a 3x3 copy (18 KB) -1 to -2 %;
# P2 (its smaller part: 22 arrays, 22.5 KB) +0.4-1.6 %, Maxwell (13 arrays in
# 512-thread blocks, 53 KB) +0.2-1.5 %
SPLIT_MIN_BLOCK_BYTES = 20480


def _group_arrays(instrs: list[Instr]) -> list[int]:
    """Distinct slots loaded or stored per 'grp'-separated group."""
    out, cur = [], set()
    for ins in instrs:
        if ins.op == "grp":
            out.append(len(cur))
            cur = set()
        elif ins.op in ("ld", "st"):
            cur.add(ins.slot)
    out.append(len(cur))
    return out


def statement_parts(statements: Sequence[Any], alias: Mapping[str, str] | None = None
                    ) -> list[list[int]]:
    """Statements grouped into independent parts: two statements are in one
    part when they touch (read or write) a common field, transitively.  Parts
    share no storage, so running part after part over the whole grid gives
    the bits of the sequential program (every statement of a part keeps its
    order).  Ordered by first statement."""
    alias = dict(alias or {})
    parent = list(range(len(statements)))

    def find(i: int) -> int:
        while parent[i] != i:
            parent[i] = parent[parent[i]]
            i = parent[i]
        return i

    owner: dict[str, int] = {}
    for k, v in enumerate(statements):
        for name in [v.stmt.lhs.field] + _field_names(v.stmt.rhs):
            r = alias.get(name, name)
            if r in owner:
                parent[find(k)] = find(owner[r])
            else:
                owner[r] = k
    parts: dict[int, list[int]] = {}
    for k in range(len(statements)):
        parts.setdefault(find(k), []).append(k)
    return sorted(parts.values(), key=lambda ks: ks[0])


def _field_names(e) -> list[str]:
    out, stack = [], [e]
    while stack:
        x = stack.pop()
        k = kind(x)
        if k == "Leaf":
            out.append(x.leaf.field)
        elif k == "FieldRef":
            out.append(x.name)
        elif k in ("Add", "Sub", "Mul", "Div"):
            stack += [x.l, x.r]
        elif k in ("Neg", "Sqrt"):
            stack.append(x.e)
        elif k == "Sum":
            stack.append(x.body)
    return out


def _phases(instrs: list[Instr]) -> int:
    """Number of load groups separated by stores in program order (1 = all
    loads precede all stores)."""
    n, seen_store = 0, True
    for ins in instrs:
        if ins.op == "st":
            seen_store = True
        elif ins.op == "ld" and seen_store:
            n += 1
            seen_store = False
    return n


def _statement_comment(v) -> str:
    try:
        from .ir import signature

        return signature(v).replace("\n", " ")
    except Exception:  # reference-built trees: the comment is informational
        return repr(v.stmt)[:200]
