"""Benchmark programs, fixtures and the bandwidth metric.

Mirror of the reference's ``tlang.bench`` (pkg/src/tlang/bench.py): the same
fourteen-statement suite, worked examples and contraction demos, the same
``bw_eff`` formula (8 bytes x (N_e*N + N_d) / t, :46-48), the same seeded
fixtures (``default_rng(0xC0FFEE)``, uniform(0,1) per field in declaration
order, target zeroed, :72-87) and the same timing protocol (reps runs, the
first discarded, median of the rest, :252-271) — plus the BASELINE.json
programs and device-side fixtures.

Timing here is device time: ``time_statement`` synchronises the GPU around
every run (CUDA events when no clock is injected).
"""

from __future__ import annotations

import csv
import json
import time
from dataclasses import dataclass
from pathlib import Path
from statistics import median
from typing import Callable, Iterable, Sequence

import numpy as np

from .evaluator import eval_program, eval_statement, eval_statement_per_component
from .fields import ScalarField, TensorField
from .ir import count_data, validate_statement
from .parser import FieldDecl, TensorDecl, parse_program

DEFAULT_SEED = 0xC0FFEE
DEFAULT_GRIDS = (32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536)
MODES = ("whole-tensor", "per-component")
CSV_COLUMNS = ("name", "mode", "N", "t_median_s", "bw_eff_gbps", "N_e", "N_d")
# --extended (SURVEY.md §5 metrics row): the device-side columns appended
EXT_COLUMNS = ("gpus", "points_per_s", "hbm_gbps", "roofline_frac", "fp64_frac")

# ------------------------------------------------- BASELINE.json programs --

DTG = """tensor dtg dim 3 rank 2 sym(0,1);
field alpha;
tensor K dim 3 rank 2 sym(0,1);
tensor db dim 3 rank 2;
dtg(sym<0,1>, i, j) = -2*alpha*K(i,j) + db(i,j) + db(j,i);
"""

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

PROGRAMS = {"c1_dtg": DTG, "c2_maxwell": MAXWELL, "c3_christoffel": CHRISTOFFEL, "p2": P2,
            "p3": P3}


def load(text: str):
    """(program, validated statements) of a source text."""
    res = parse_program(text)
    if res.diagnostics:
        raise ValueError(f"program failed to parse: {res.diagnostics}")
    prog = res.program
    return prog, [validate_statement(s, prog.decls) for s in prog.statements]


# ------------------------------------------------------------- the suite --


@dataclass(frozen=True)
class BenchResult:
    name: str
    mode: str
    gridsize: int
    t: float  # median seconds
    bw_eff: float  # GB/s
    n_e: int
    n_d: int
    bytes_per_point: int = 0  # algorithmic roofline bytes (read-modify-write twice)
    flops_per_point: int = 0

    def row(self) -> tuple:
        return (self.name, self.mode, self.gridsize, self.t, self.bw_eff, self.n_e, self.n_d)

    def extended_row(self, hbm_peak_gbs: float, fp64_peak_gflops: float) -> tuple:
        """EXT_COLUMNS: one GPU; points/s; algorithmic HBM GB/s and its
        fraction of the copy peak; achieved fp64 GFLOP/s over the fp64 peak."""
        hbm = self.bytes_per_point * self.gridsize / self.t / 1e9
        fl = self.flops_per_point * self.gridsize / self.t / 1e9
        return (1, self.gridsize / self.t, hbm, hbm / hbm_peak_gbs, fl / fp64_peak_gflops)


def bw_eff(n_e: int, n_d: int, gridsize: int, t: float) -> float:
    """Effective bandwidth in GB/s (reference bench.py:46-48)."""
    return 8.0 * (n_e * gridsize + n_d) / t / 1e9


@dataclass(frozen=True)
class SuiteEntry:
    name: str
    source: str

    def parse(self):
        prog, vs = load(self.source)
        (v,) = vs
        return prog, v

    def build_env(self, gridsize: int, seed: int = DEFAULT_SEED, device=None):
        prog, v = self.parse()
        return v, make_env(prog, v.stmt.lhs.field, gridsize, seed, device=device)


def make_env(program, target: str, gridsize: int, seed: int = DEFAULT_SEED, device=None) -> dict:
    """Fields for one run: uniform(0,1) inputs from default_rng(seed) in
    declaration order, zeroed target — the reference's exact numbers
    (bench.py:72-87), uploaded to `device`."""
    import torch

    rng = np.random.default_rng(seed)
    env: dict = {}
    for item in program.items:
        if isinstance(item, TensorDecl):
            f = TensorField(item.name, program.decls.tensors[item.name], gridsize, device=device)
            if item.name != target:
                f.data.copy_(torch.from_numpy(rng.uniform(0.0, 1.0, tuple(f.data.shape))))
            env[item.name] = f
        elif isinstance(item, FieldDecl):
            f = ScalarField(item.name, gridsize, device=device)
            if item.name != target:
                f.data.copy_(torch.from_numpy(rng.uniform(0.0, 1.0, gridsize)))
            env[item.name] = f
    return env


def _entry(name: str, decls: Sequence[str], stmt: str) -> SuiteEntry:
    return SuiteEntry(name, "\n".join([*decls, stmt]) + "\n")


def _vectors(prefix: str, names: str) -> list[str]:
    return [f"tensor {prefix}_{n} dim 3 rank 1;" for n in names.split()]


def _square(prefix: str, names: str, rank: int) -> list[str]:
    return [f"tensor {prefix}_{n} dim 3 rank {rank};" for n in names.split()]


def builtin_suite() -> list[SuiteEntry]:
    """The fourteen dimension-3 statements of reference bench.py:98-199."""
    return [
        _entry("assign1", _vectors("assign1", "A B"), "assign1_A(i) = assign1_B(i);"),
        _entry("assign2", _square("assign2", "A B", 2), "assign2_A(i, j) = assign2_B(i, j);"),
        _entry("assign3", _square("assign3", "A B", 3),
               "assign3_A(i, j, k) = assign3_B(i, j, k);"),
        _entry("add1", _vectors("add1", "A B C"), "add1_A(i) = add1_B(i) + add1_C(i);"),
        _entry("add2", _vectors("add2", "A B C D"),
               "add2_A(i) = add2_B(i) + add2_C(i) + add2_D(i);"),
        _entry("add3", _vectors("add3", "A B C D E"),
               "add3_A(i) = add3_B(i) + add3_C(i) + add3_D(i) + add3_E(i);"),
        _entry("outer1", ["tensor outer1_A dim 3 rank 2;", *_vectors("outer1", "B C")],
               "outer1_A(i, j) = outer1_B(i)*outer1_C(j);"),
        _entry("outer2", ["tensor outer2_A dim 3 rank 3;", *_vectors("outer2", "B C D")],
               "outer2_A(i, j, k) = outer2_B(i)*outer2_C(j)*outer2_D(k);"),
        _entry("outer3", ["tensor outer3_A dim 3 rank 4;", *_vectors("outer3", "B C D E")],
               "outer3_A(i, j, k, l) = outer3_B(i)*outer3_C(j)*outer3_D(k)*outer3_E(l);"),
        _entry("contract1",
               ["tensor contract1_A dim 3 rank 4;", "tensor contract1_B dim 3 rank 2;",
                "tensor contract1_E dim 3 rank 4;"],
               "contract1_A(i, j, k, l) = Sum(m, contract1_B(i, m)*contract1_E(m, j, k, l));"),
        _entry("contract2",
               ["tensor contract2_A dim 3 rank 4;", "tensor contract2_B dim 3 rank 2;",
                "tensor contract2_C dim 3 rank 2;", "tensor contract2_E dim 3 rank 4;"],
               "contract2_A(i, j, k, l) = "
               "Sum(m, Sum(n, contract2_C(j, n)*contract2_B(i, m)*contract2_E(m, n, k, l)));"),
        _entry("contract3",
               ["tensor contract3_A dim 3 rank 4;", "tensor contract3_B dim 3 rank 2;",
                "tensor contract3_C dim 3 rank 2;", "tensor contract3_D dim 3 rank 2;",
                "tensor contract3_E dim 3 rank 4;"],
               "contract3_A(i, j, k, l) = Sum(m, Sum(n, Sum(o, "
               "contract3_D(k, o)*contract3_C(j, n)*contract3_B(i, m)*contract3_E(m, n, o, l))));"),
        _entry("kij",
               ["tensor kij_K dim 3 rank 2 sym(0,1);", "field kij_alpha;",
                "tensor kij_g dim 3 rank 2 sym(0,1);", "tensor kij_beta dim 3 rank 1;"],
               "kij_K(sym<0,1>, i, j) = 2*kij_alpha*kij_g(i, j) + kij_beta(i)*kij_beta(j);"),
        _entry("christoffel",
               ["tensor christoffel_Gamma dim 3 rank 3 sym(1,2);",
                "tensor christoffel_Invg dim 3 rank 2 sym(0,1);",
                "tensor christoffel_dg dim 3 rank 2 sym(0,1) inner rank 1;"],
               "christoffel_Gamma(sym<1,2>, i, j, k) = 0.5*Sum(l, christoffel_Invg(i, l)"
               "*(christoffel_dg(j, l)(k) + christoffel_dg(l, k)(j) - christoffel_dg(j, k)(l)));"),
    ]


def worked_examples() -> list[SuiteEntry]:
    """Dimension-4 fixtures with pinned counts 42 and 19 (bench.py:202-223)."""
    return [
        _entry("sym42", ["tensor w42_C dim 4 rank 2 sym(0,1);", "tensor w42_A dim 4 rank 2;",
                         "tensor w42_B dim 4 rank 2;"],
               "w42_C(sym<0,1>, a, b) = Sum(c, w42_A(a, c)*w42_B(c, b));"),
        _entry("fix19", ["tensor w19_D dim 4 rank 2 sym(0,1);", "tensor w19_E dim 4 rank 2;",
                         "tensor w19_F dim 4 rank 2;"],
               "w19_D(sym<0,1>, i, 0) = Sum(c, w19_E(i+1, c)*w19_F(c, 0));"),
    ]


def contraction_demos() -> list[SuiteEntry]:
    return [
        _entry("demo_plain", ["tensor demo_C dim 4 rank 2;", "tensor demo_A dim 4 rank 2;",
                              "tensor demo_B dim 4 rank 2;"],
               "demo_C(a, b) = Sum(c, demo_A(a, c)*demo_B(c, b));"),
        worked_examples()[0],
        worked_examples()[1],
    ]


def suite_program_text(entries: Iterable[SuiteEntry] | None = None) -> str:
    entries = list(entries) if entries is not None else builtin_suite()
    return "\n".join(e.source for e in entries)


# ----------------------------------------------------------------- timing --


def _device_clock() -> float:
    import torch

    if torch.cuda.is_available():
        torch.cuda.synchronize()
    return time.perf_counter()


def time_statement(vstmt, env, *, reps: int = 21, mode: str = "whole-tensor",
                   clock: Callable[[], float] | None = None) -> float:
    """Median duration over `reps` runs, the first discarded (reference
    bench.py:252-271).  The default clock synchronises the GPU first, so a
    sample is the device execution time of the run."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    if reps < 2:
        raise ValueError("need at least 2 repetitions: the first is discarded")
    clock = clock or _device_clock
    run = eval_statement if mode == "whole-tensor" else eval_statement_per_component
    samples = []
    for _ in range(reps):
        t0 = clock()
        run(vstmt, env)
        samples.append(clock() - t0)
    return median(samples[1:])


def time_program(vs, env, *, reps: int = 21) -> float:
    """Median device time of ``eval_program`` (CUDA events), first run dropped."""
    import torch

    samples = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eval_program(vs, env)
        b.record()
        b.synchronize()
        samples.append(a.elapsed_time(b) / 1e3)
    return median(samples[1:])


def run(entry: SuiteEntry, gridsize: int, *, reps: int = 21, mode: str = "whole-tensor",
        seed: int = DEFAULT_SEED, clock=None) -> BenchResult:
    if gridsize < 1:
        raise ValueError("gridsize must be positive")
    vstmt, env = entry.build_env(gridsize, seed)
    n_e, n_d = count_data(vstmt)
    t = time_statement(vstmt, env, reps=reps, mode=mode, clock=clock)
    from .evaluator import plan_for

    plan = plan_for(vstmt, env)
    return BenchResult(entry.name, mode, gridsize, t, bw_eff(n_e, n_d, gridsize, t), n_e, n_d,
                       plan.bytes_per_point, plan.flops_per_point)


def sweep(entries: Sequence[SuiteEntry], gridsizes: Sequence[int] = DEFAULT_GRIDS, *,
          modes: Sequence[str] = ("whole-tensor",), reps: int = 21,
          seed: int = DEFAULT_SEED) -> list[BenchResult]:
    return [run(e, n, reps=reps, mode=m, seed=seed)
            for e in entries for m in modes for n in gridsizes]


def write_csv(results: Iterable[BenchResult], out, peaks: tuple[float, float] | None = None
              ) -> None:
    """CSV with the reference's columns (bench.py:307-312); with `peaks`
    (HBM GB/s, fp64 GFLOP/s) the EXT_COLUMNS appended."""
    w = csv.writer(out)
    w.writerow(CSV_COLUMNS + (EXT_COLUMNS if peaks else ()))
    for r in results:
        row = [r.name, r.mode, r.gridsize, repr(r.t), repr(r.bw_eff), r.n_e, r.n_d]
        if peaks:
            row += [repr(x) for x in r.extended_row(*peaks)]
        w.writerow(row)


def write_json(results: Iterable[BenchResult], out, peaks: tuple[float, float] | None = None
               ) -> None:
    rows = []
    for r in results:
        d = dict(zip(CSV_COLUMNS, r.row()))
        if peaks:
            d.update(zip(EXT_COLUMNS, r.extended_row(*peaks)))
        rows.append(d)
    json.dump(rows, out, indent=2)
    out.write("\n")


def device_peaks() -> tuple[float, float]:
    """(HBM GB/s, fp64 GFLOP/s) for the extended columns: MEASURED_PEAKS.json
    hbm_gbs when present (next to the package), else this box's device copy
    rate measured now; the fp64 side from tlb_fp64_probe (uncontracted
    DMUL + DADD, the kernels' instruction mix)."""
    import torch

    from .runtime import fp64_peak_gflops

    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    try:
        hbm = float(json.loads(p.read_text())["hbm_gbs"])
    except Exception:
        a = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        b.copy_(a)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            b.copy_(a)
        e.record()
        e.synchronize()
        hbm = 5 * 2 * a.numel() * 8 / (s.elapsed_time(e) / 1e3) / 1e9
        del a, b
    return hbm, fp64_peak_gflops()
