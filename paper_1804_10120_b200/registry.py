"""Statement registry, manifest, and reference-harness bindings for the GPU.

Mirror of the reference's ``tlang.registry`` (pkg/src/tlang/registry.py):
statements register under their canonical signature, the first
registration takes the next 1-based ordinal, repeats return it
(registry.py:46-55), and ``manifest_text`` is the same
``ordinal<TAB>signature<TAB>N_e<TAB>N_d`` table (:57-60).

``write_all(out_dir, backend="b200")`` replaces the reference's
C/CUDA text emission with the B200 path: it writes

  tloops_manifest.tsv       the manifest, byte-identical to the reference's
  tloops_bindings_b200.c    the reference bindings ABI — ``tl_arg_desc``,
                            ``tl_entry``, ``tloops_entries[]``,
                            ``tloops_entry_count`` with the same descriptor
                            order, alias tables and field checks
                            (registry.py:134-270) — whose ``call`` hands the
                            harness's host pointer arrays to
                            ``tlb_harness_call`` (libtlb200): H2D, the fused
                            sm_100a kernel of that statement, D2H.

``build_shared`` compiles the bindings into a shared object the unchanged
``tl_harness`` (pkg/harness/tl_harness.c) can dlopen.
"""

from __future__ import annotations

import subprocess
from dataclasses import dataclass
from pathlib import Path

from .ir import count_data, signature
from .lowering import kind, lower_program
from .runtime import LIB_PATH, compile_options
from .symmetry import SymmetrySpec, alias_table, component_count

MANIFEST_NAME = "tloops_manifest.tsv"
BINDINGS_NAME = "tloops_bindings_b200.c"
# "cuda" is accepted as the reference's name for the GPU backend; the
# reference's CPU C emission ("c") is not part of this package (the
# reference's own emitted C is the CPU baseline, oracle/build_ref.py)
BACKENDS = ("b200", "cuda")
INCLUDE_DIR = Path(__file__).resolve().parent.parent / "include"


@dataclass
class RegistryEntry:
    ordinal: int
    signature: str
    stmt: object
    n_e: int
    n_d: int


@dataclass(frozen=True)
class ArgDescriptor:
    """One argument of an entry, in the reference's order (codegen_c.py:97-135):
    the target, then RHS tensors and scalar fields by first depth-first
    occurrence, then one number per literal occurrence."""

    role: str  # "lhs" | "rhs" | "scalar" | "const"
    name: str
    dim: int = 0
    outer_rank: int = 0
    inner_rank: int = 0
    outer_sym: SymmetrySpec = SymmetrySpec()
    inner_sym: SymmetrySpec = SymmetrySpec()
    value: float = 0.0

    @property
    def is_tensor(self) -> bool:
        return self.role in ("lhs", "rhs")

    @property
    def n_flat(self) -> int:
        return self.dim ** (self.outer_rank + self.inner_rank)

    @property
    def n_components(self) -> int:
        return (component_count(self.dim, self.outer_rank, self.outer_sym)
                * component_count(self.dim, self.inner_rank, self.inner_sym))

    def combined_alias(self) -> list[int]:
        """Flat index (outer group fastest, then inner) -> component
        (reference registry.py:170-180)."""
        outer = alias_table(self.dim, self.outer_rank, self.outer_sym)
        inner = alias_table(self.dim, self.inner_rank, self.inner_sym)
        ic = component_count(self.dim, self.inner_rank, self.inner_sym)
        nof = self.dim ** self.outer_rank
        return [outer[f % nof] * ic + inner[f // nof] for f in range(self.n_flat)]


def _sym(s) -> SymmetrySpec:
    return SymmetrySpec(tuple(tuple(p) for p in s.inequalities)) if s is not None else SymmetrySpec()


def collect_args(v) -> list[ArgDescriptor]:
    def tensor(name: str, role: str) -> ArgDescriptor:
        sh = v.decls.tensor(name)
        return ArgDescriptor(role, name, sh.dim, sh.outer_rank, sh.inner_rank, _sym(sh.outer_sym),
                             _sym(sh.inner_sym))

    args = [tensor(v.stmt.lhs.field, "lhs")]
    seen = {v.stmt.lhs.field}
    n_const = 0
    stack = [v.stmt.rhs]
    while stack:  # preorder, left to right
        e = stack.pop()
        k = kind(e)
        if k == "Leaf" and e.leaf.field not in seen:
            seen.add(e.leaf.field)
            args.append(tensor(e.leaf.field, "rhs"))
        elif k == "FieldRef" and e.name not in seen:
            seen.add(e.name)
            args.append(ArgDescriptor("scalar", e.name))
        elif k == "Const":
            args.append(ArgDescriptor("const", f"d{n_const}", value=e.value))
            n_const += 1
        if k in ("Add", "Sub", "Mul", "Div"):
            stack += [e.r, e.l]
        elif k in ("Neg", "Sqrt"):
            stack.append(e.e)
        elif k == "Sum":
            stack.append(e.body)
    return args


class Registry:
    """Deduplicating statement collection with stable 1-based ordinals."""

    def __init__(self) -> None:
        self._by_signature: dict[str, int] = {}
        self.entries: list[RegistryEntry] = []

    def __len__(self) -> int:
        return len(self.entries)

    def register(self, v) -> int:
        sig = signature(v)
        hit = self._by_signature.get(sig)
        if hit is not None:
            return hit
        n_e, n_d = count_data(v)
        self.entries.append(RegistryEntry(len(self.entries) + 1, sig, v, n_e, n_d))
        self._by_signature[sig] = len(self.entries)
        return len(self.entries)

    def manifest_text(self) -> str:
        return "".join(f"{e.ordinal}\t{e.signature}\t{e.n_e}\t{e.n_d}\n" for e in self.entries)

    def write_all(self, out_dir, backend: str = "b200") -> list[Path]:
        if backend not in BACKENDS:
            raise ValueError(f"backend must be one of {BACKENDS}, got {backend!r} (the CPU "
                             "C backend of the reference is not provided: this package runs "
                             "statements on the GPU)")
        if not self.entries:
            raise ValueError("registry is empty: nothing to generate")
        out = Path(out_dir)
        try:
            out.mkdir(parents=True, exist_ok=True)
            (out / MANIFEST_NAME).write_text(self.manifest_text())
            (out / BINDINGS_NAME).write_text(render_bindings(self.entries))
        except OSError as exc:
            raise RuntimeError(f"cannot write generated sources under {out}: {exc}") from exc
        return sorted([out / MANIFEST_NAME, out / BINDINGS_NAME])

    def build_shared(self, out_dir, so_name: str = "tloops_b200.so") -> Path:
        """write_all + compile the bindings into a harness-loadable .so."""
        self.write_all(out_dir)
        out = Path(out_dir)
        so = out / so_name
        cmd = ["cc", "-shared", "-fPIC", "-O2", "-std=c99", "-Wall", f"-I{INCLUDE_DIR}",
               str(out / BINDINGS_NAME), "-o", str(so), f"-L{LIB_PATH.parent}", "-ltlb200",
               f"-Wl,-rpath,{LIB_PATH.parent}"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"{' '.join(cmd)}\n{res.stderr}")
        precompile_harness(self.entries)
        return so


def harness_source(v) -> str:
    """The kernel source exactly as the bindings embed it (tl_src_NNNN:
    every line newline-terminated, see _c_string)."""
    return "".join(line + "\n" for line in lower_program([v]).source.split("\n"))


def harness_cubin_name(source: str, opts) -> str:
    """tlb_harness_call's cache file name: FNV-1a 64 over the source and each
    option, each followed by a 0xff separator (tlb_runtime.cpp)."""
    h = 1469598103934665603
    for text in [source, *opts]:
        for byte in text.encode():
            h = ((h ^ byte) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        h = ((h ^ 0xFF) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"harness_{h:016x}.cubin"


def precompile_harness(entries) -> list[Path]:
    """NVRTC-compile every entry's kernel into the cache the harness bindings
    read ($TLB_CACHE_DIR, else the package's _kcache next to libtlb200.so),
    so a harness process loads cubins instead of compiling (no GPU needed)."""
    import ctypes

    from .runtime import cache_dir, check, lib

    opts = compile_options()
    copts = (ctypes.c_char_p * len(opts))(*[o.encode() for o in opts])
    out = []
    for e in entries:
        src = harness_source(e.stmt)
        path = cache_dir() / harness_cubin_name(src, opts)
        if not path.exists():
            handle = ctypes.c_void_p()
            check(lib().tlb_compile(src.encode(), copts, len(opts), str(path).encode(),
                                    ctypes.byref(handle)), "tlb_compile")
            lib().tlb_kernel_destroy(handle)
        out.append(path)
    return out


# ------------------------------------------------------------ C rendering --

_TYPES = """\
/* Argument descriptors and entry table: the reference bindings ABI
 * (pkg/src/tlang/registry.py:134-167, mirrored by pkg/harness/tl_harness.c:24-48). */
typedef struct tl_arg_desc {
    const char* name;
    int kind;                /* 0 target tensor, 1 input tensor, 2 scalar field, 3 number */
    int dim;
    int outer_rank;
    int inner_rank;
    int n_outer_pairs;
    const unsigned char* outer_pairs;
    int n_inner_pairs;
    const unsigned char* inner_pairs;
    long n_components;
    long n_flat;
    const long* alias;
    double value;
} tl_arg_desc;

typedef struct tl_entry {
    int ordinal;
    const char* signature;
    int n_args;
    const tl_arg_desc* args;
    void (*call)(const long N, double** const* tensors,
                 const double* const* scalars, const double* numbers);
} tl_entry;
"""


def _c_string(text: str) -> str:
    out = []
    for line in text.split("\n"):
        esc = line.replace("\\", "\\\\").replace('"', '\\"')
        out.append(f'  "{esc}\\n"')
    return "\n".join(out)


def _c_list(values) -> str:
    return ",".join(str(v) for v in values)


def render_bindings(entries: list[RegistryEntry]) -> str:
    opts = compile_options()
    lines = ["/* generated by paper_1804_10120_b200.registry: reference bindings ABI,",
             " * calls forwarded to the fused sm_100a kernels of libtlb200 */",
             "#include <stdio.h>", "#include <stdlib.h>", "#include <stddef.h>",
             '#include "tlb200.h"', "", _TYPES,
             "static const char* const tl_opts[] = {" + ", ".join(f'"{o}"' for o in opts) + "};",
             ""]
    kinds = {"lhs": 0, "rhs": 1, "scalar": 2, "const": 3}
    for e in entries:
        tag = f"{e.ordinal:04d}"
        v = e.stmt
        args = collect_args(v)
        plan = lower_program([v])
        # descriptors (same text content as the reference's)
        for k, a in enumerate(args):
            if not a.is_tensor:
                continue
            if a.outer_sym.inequalities:
                flat = _c_list(x for p in a.outer_sym.inequalities for x in p)
                lines.append(f"static const unsigned char tl_osym_{tag}_a{k}[] = {{{flat}}};")
            if a.inner_sym.inequalities:
                flat = _c_list(x for p in a.inner_sym.inequalities for x in p)
                lines.append(f"static const unsigned char tl_isym_{tag}_a{k}[] = {{{flat}}};")
            lines.append(f"static const long tl_alias_{tag}_a{k}[] = "
                         f"{{{_c_list(a.combined_alias())}}};")
        lines.append(f"static const tl_arg_desc tl_args_{tag}[] = {{")
        for k, a in enumerate(args):
            if a.is_tensor:
                osym = f"tl_osym_{tag}_a{k}" if a.outer_sym.inequalities else "NULL"
                isym = f"tl_isym_{tag}_a{k}" if a.inner_sym.inequalities else "NULL"
                lines.append(
                    f'  {{"{a.name}", {kinds[a.role]}, {a.dim}, {a.outer_rank}, {a.inner_rank}, '
                    f"{len(a.outer_sym.inequalities)}, {osym}, {len(a.inner_sym.inequalities)}, "
                    f"{isym}, {a.n_components}, {a.n_flat}, tl_alias_{tag}_a{k}, 0.0}},")
            elif a.role == "scalar":
                lines.append(f'  {{"{a.name}", 2, 0, 0, 0, 0, NULL, 0, NULL, 1, 1, NULL, 0.0}},')
            else:
                lines.append(f'  {{"{a.name}", 3, 0, 0, 0, 0, NULL, 0, NULL, 0, 0, NULL, '
                             f"{float(a.value)!r}}},")
        lines.append("};")
        # kernel fields -> harness arguments
        tensors = [a.name for a in args if a.is_tensor]
        scalars = [a.name for a in args if a.role == "scalar"]
        fkind, farg, fncomp, fflat = [], [], [], []
        for fi, info in enumerate(plan.fields):
            if info.is_tensor:
                k = tensors.index(info.name)
                arg = next(a for a in args if a.is_tensor and a.name == info.name)
                alias = arg.combined_alias()
                first = [alias.index(c) for c in range(info.n_components)]
                lines.append(f"static const long tl_flat_{tag}_f{fi}[] = {{{_c_list(first)}}};")
                fkind.append(0)
                farg.append(k)
                fflat.append(f"tl_flat_{tag}_f{fi}")
            else:
                fkind.append(1)
                farg.append(scalars.index(info.name))
                fflat.append("NULL")
            fncomp.append(info.n_components)
        lines += [
            f"static const char tl_src_{tag}[] =",
            _c_string(plan.source) + ";",
            f"static const int tl_fkind_{tag}[] = {{{_c_list(fkind)}}};",
            f"static const int tl_farg_{tag}[] = {{{_c_list(farg)}}};",
            f"static const int tl_fncomp_{tag}[] = {{{_c_list(fncomp)}}};",
            f"static const long* const tl_fflat_{tag}[] = {{{', '.join(fflat)}}};",
            f"static const int tl_sfield_{tag}[] = {{{_c_list(plan.slot_field)}}};",
            f"static const long long tl_scomp_{tag}[] = {{{_c_list(plan.slot_comp)}}};",
            f"static const int tl_sflags_{tag}[] = {{{_c_list(plan.slot_flags)}}};",
            f"static tlb_harness_kernel tl_hk_{tag} = {{tl_src_{tag}, {len(opts)}, tl_opts, "
            f"{len(plan.fields)}, tl_fkind_{tag}, tl_farg_{tag}, tl_fncomp_{tag}, tl_fflat_{tag}, "
            f"{plan.n_slots}, tl_sfield_{tag}, tl_scomp_{tag}, tl_sflags_{tag}, NULL}};",
            f"static void tl_call_{tag}(const long N, double** const* T,",
            "                          const double* const* S, const double* D)",
            "{",
            "  (void)D; /* literals are folded into the fused kernel */",
            f"  if (tlb_harness_call(&tl_hk_{tag}, N, T, S) != 0) {{",
            "    /* the reference `call` has no error channel (void): report and",
            "       exit with TLB_HARNESS_EXIT_GPU, past the harness's own 2-6 */",
            f'    fprintf(stderr, "tl_harness: GPU kernel tl_{tag} (ordinal {e.ordinal}) '
            f'failed: %s\\n", tlb_last_error());',
            "    fflush(stderr);",
            "    exit(TLB_HARNESS_EXIT_GPU);",
            "  }",
            "}",
            "",
        ]
    lines.append("const tl_entry tloops_entries[] = {")
    for e in entries:
        tag = f"{e.ordinal:04d}"
        sig = e.signature.replace("\\", "\\\\").replace('"', '\\"')
        n_args = len(collect_args(e.stmt))
        lines.append(f'  {{{e.ordinal}, "{sig}", {n_args}, tl_args_{tag}, tl_call_{tag}}},')
    lines.append("};")
    lines.append(f"const int tloops_entry_count = {len(entries)};")
    lines.append("")
    return "\n".join(lines)
