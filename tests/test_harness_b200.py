"""The reference's unchanged conformance harness (oracle/_ref/tl_harness,
built from pkg/harness by oracle/build_ref.py) loading OUR bindings table:
its negative paths (reference pkg/harness/run_tests.sh:48-63) and the
b200 `call`'s own failure path.  None of these reach a kernel launch, so
they run without a GPU; the positive runs are GPU tests
(test_gpu_parity.py::test_reference_harness_drives_the_gpu_kernels)."""

import subprocess

import pytest

from helpers import GOLDEN, manifest, program

try:
    from oracle import refc

    HARNESS = refc.REF_DIR / "tl_harness"
except Exception:  # pragma: no cover
    HARNESS = None

pytestmark = pytest.mark.skipif(HARNESS is None or not HARNESS.exists(),
                                reason="oracle/_ref/tl_harness not built")


def _bindings(case, tmp_path):
    from paper_1804_10120_b200.registry import Registry

    _, vs = program(manifest()["cases"][case]["source"])
    reg = Registry()
    for v in vs:
        reg.register(v)
    return reg.build_shared(tmp_path), tmp_path / "tloops_manifest.tsv"


def _harness(*args):
    return subprocess.run([str(HARNESS), *map(str, args)], capture_output=True, text=True,
                          timeout=300)


def test_manifest_naming_a_missing_kernel_fails_with_the_symbol(tmp_path):
    # run_tests.sh:48-55: exit 4, the missing tl_0099 named on stderr
    so, _ = _bindings("c1_dtg", tmp_path)
    bad = tmp_path / "bad_manifest.tsv"
    bad.write_text("99\tbogus\t1\t0\n")
    out = tmp_path / "should_not_exist.tldf"
    res = _harness(so, bad, GOLDEN / "c1_dtg.in.tldf", out)
    assert res.returncode == 4, res.stderr
    assert "tl_0099" in res.stderr
    assert not out.exists()


def test_fixture_shape_mismatch_is_rejected(tmp_path):
    # run_tests.sh:57-63: exit 5, "fixture lacks field"
    so, man = _bindings("c4_p2", tmp_path)
    res = _harness(so, man, GOLDEN / "c1_dtg.in.tldf", tmp_path / "x.tldf")
    assert res.returncode == 5, res.stderr
    assert "fixture lacks field" in res.stderr


def test_kernel_failure_is_reported_not_aborted(tmp_path):
    # the b200 `call` cannot return an error (the reference's call is void):
    # it names the kernel and the cause, and exits TLB_HARNESS_EXIT_GPU (7)
    # instead of abort()ing — here the cause is that this host has no GPU
    import torch

    if torch.cuda.is_available():
        pytest.skip("needs a host without a CUDA device to make the call fail")
    so, man = _bindings("c1_dtg", tmp_path)
    out = tmp_path / "out.tldf"
    res = _harness(so, man, GOLDEN / "c1_dtg.in.tldf", out)
    assert res.returncode == 7, (res.returncode, res.stderr)
    assert "GPU kernel tl_0001 (ordinal 1) failed" in res.stderr
    assert "CUDA" in res.stderr or "cuda" in res.stderr
    assert not out.exists()
