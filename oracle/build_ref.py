"""Build oracle/_ref from the reference checkout — TEST/BASELINE INFRASTRUCTURE.

Runs only where /root/reference exists (the build container); the outputs
are git-ignored but travel to the GPU box with the repo snapshot.

  1. The reference's C conformance harness, compiled directly from its
     sources with gcc (its own Makefile is not run; recipe restated from
     pkg/harness/Makefile:4-11):
       _ref/tl_harness  <- pkg/harness/tl_harness.c + tldf_io.c  (-ldl)
       _ref/tl_compare  <- pkg/harness/tl_compare.c + tldf_io.c  (-lm)
  2. The reference's CPU kernel path ("AccelCPU") for
     every benchmark program: the reference package itself
     (pkg/src/tlang, imported read-only) emits the C kernels and bindings
     (registry.py:62-94, codegen_c.py:224-254), which are compiled exactly
     as its harness does (`cc -shared -fPIC -O2 -std=c99`, tl_harness.c:77):
       _ref/<program>.so            exports tloops_entries / tloops_entry_count
       _ref/<program>.manifest.tsv  ordinal, signature, N_e, N_d
  3. The reference's CUDA emission for the same programs (the paper's GPU
     design: one thread per (point, LHS component), device pointer arrays),
     compiled as-is with nvcc for sm_100a into _ref/<program>_cuda.so — the
     comparator of SURVEY.md 8f #3 (driven by oracle/refcuda.py).
  4. The reference package itself (pkg/src/tlang, unmodified) as a build
     artefact under _ref/tlang, so that its numpy evaluator — the paper's
     "NonAccel" CPU path (evaluator.py:204-236, chunk + ThreadPoolExecutor)
     — can be timed on the GPU box's host cores beside the device numbers
     (bench.py, oracle/refnumpy.py).  Like the .so files it is git-ignored
     and travels with the repo snapshot; nothing under the product package
     imports it.

Usage: python oracle/build_ref.py [--force]
"""

from __future__ import annotations

import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref"
REF = Path("/root/reference/pkg")
ROOT = HERE.parent


def programs() -> dict[str, str]:
    sys.path.insert(0, str(ROOT))
    from paper_1804_10120_b200.bench import PROGRAMS, builtin_suite, suite_program_text

    progs = dict(PROGRAMS)
    progs["suite"] = suite_program_text(builtin_suite())
    return progs


def _run(cmd, **kw):
    res = subprocess.run(cmd, capture_output=True, text=True, **kw)
    if res.returncode != 0:
        raise RuntimeError(f"{' '.join(map(str, cmd))}\n{res.stdout}\n{res.stderr}")
    return res


def build(force: bool = False) -> Path:
    if not REF.exists():
        if OUT.exists():
            return OUT  # GPU box: use the prebuilt files
        raise FileNotFoundError("reference checkout not present and no prebuilt oracle/_ref")
    OUT.mkdir(exist_ok=True)
    cc = shutil.which("cc") or shutil.which("gcc")
    harness = REF / "harness"
    flags = ["-O2", "-std=c99", "-Wall", "-Wextra"]
    targets = {
        "tl_harness": ([harness / "tl_harness.c", harness / "tldf_io.c"], ["-ldl"]),
        "tl_compare": ([harness / "tl_compare.c", harness / "tldf_io.c"], ["-lm"]),
    }
    for name, (srcs, libs) in targets.items():
        exe = OUT / name
        if force or not exe.exists():
            _run([cc, *flags, *map(str, srcs), "-o", str(exe), *libs])

    pkg = OUT / "tlang"
    src_pkg = REF / "src" / "tlang"
    stamp = "".join(f"{p.name}:{p.stat().st_size}:{p.stat().st_mtime_ns};"
                    for p in sorted(src_pkg.glob("*.py")))
    if force or not (pkg / ".stamp").exists() or (pkg / ".stamp").read_text() != stamp:
        if pkg.exists():
            shutil.rmtree(pkg)
        shutil.copytree(src_pkg, pkg, ignore=shutil.ignore_patterns("__pycache__"))
        (pkg / ".stamp").write_text(stamp)

    sys.path.insert(0, str(REF / "src"))
    from tlang.ir import validate_statement
    from tlang.parser import parse_program
    from tlang.registry import Registry

    for name, text in programs().items():
        so = OUT / f"{name}.so"
        src_file = OUT / f"{name}.tl"
        fresh = so.exists() and (OUT / f"{name}_cuda.so").exists() and src_file.exists()
        if not force and fresh and src_file.read_text() == text:
            continue
        res = parse_program(text)
        assert res.ok, res.diagnostics
        reg = Registry()
        for s in res.program.statements:
            reg.register(validate_statement(s, res.program.decls))
        gen = OUT / f"{name}_gen"
        if gen.exists():
            shutil.rmtree(gen)
        reg.write_all(gen, "c")
        _run([cc, "-shared", "-fPIC", "-O2", "-std=c99", str(gen / "tloops_kernels.c"),
              str(gen / "tloops_bindings.c"), "-o", str(so), "-lm"])
        shutil.copy(gen / "tloops_manifest.tsv", OUT / f"{name}.manifest.tsv")
        cuda = OUT / f"{name}_cuda"
        if cuda.exists():
            shutil.rmtree(cuda)
        reg.write_all(cuda, "cuda")
        # the paper's GPU design as emitted (comparator):
        # default nvcc flags, as the reference's own syntax test compiles it
        # (test_acceptance.py:238-242), for sm_100a
        nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
        _run([nvcc, "-shared", "-Xcompiler", "-fPIC", "-O3",
              "-gencode", "arch=compute_100a,code=sm_100a",
              str(cuda / "tloops_kernels.cu"), str(cuda / "tloops_bindings.cu"),
              "-o", str(OUT / f"{name}_cuda.so")])
        src_file.write_text(text)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
