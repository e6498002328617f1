"""The C-ABI library: loads without a GPU, exports every symbol the header
declares, compiles with NVRTC host-only, and fails loudly (no fallback)
where a GPU is required."""

import re
from pathlib import Path

import pytest
import torch

from paper_1804_10120_b200 import runtime

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "tlb200.h").read_text()
    return sorted(set(re.findall(r"\b(tlb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert set(declared_symbols()) == set(runtime.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = runtime.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.tlb_abi_version() == 1


def test_library_exports_only_the_c_abi():
    # the dynamic symbol table holds exactly the header's functions: internal
    # helpers (launch geometry, source parsing, error plumbing) stay hidden
    import shutil
    import subprocess

    if not shutil.which("nm"):
        pytest.skip("no nm")
    out = subprocess.run(["nm", "-D", "--defined-only", str(runtime.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    funcs = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert funcs == set(declared_symbols())


def test_nvrtc_available_without_gpu():
    major, minor = runtime.nvrtc_version()
    assert (major, minor) >= (12, 8)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU error path")
def test_launch_without_driver_fails_loudly():
    lib = runtime.lib()
    rc = lib.tlb_init(1)
    assert rc != 0
    assert b"driver" in lib.tlb_last_error() or b"libcuda" in lib.tlb_last_error()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU error path")
def test_eval_without_gpu_raises_not_falls_back():
    from helpers import program
    from paper_1804_10120_b200 import EvalError, TensorField, eval_statement
    from paper_1804_10120_b200.runtime import TlbError

    prog, (v,) = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(i);\n")
    env = {n: TensorField(n, s, 4, device="cpu") for n, s in prog.decls.tensors.items()}
    with pytest.raises((EvalError, TlbError)):
        eval_statement(v, env)
    assert (env["A"].data == 0).all()


def test_compile_error_is_reported():
    from paper_1804_10120_b200.lowering import KernelPlan

    bad = KernelPlan("this is not CUDA", [], [0], [0], [1], 0, 0, 1, key="bad")
    with pytest.raises(runtime.TlbError, match="NVRTC"):
        runtime.Kernel(bad)
