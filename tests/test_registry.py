"""Registry mirror and the reference-harness bindings of the GPU path:
manifest byte-identical to the reference's, and a bindings table whose
descriptors equal the reference's emitted ones entry by entry."""

import ctypes

import pytest

from helpers import program
from oracle import refc
from paper_1804_10120_b200 import bench as tb
from paper_1804_10120_b200.registry import Registry


def _registry(text):
    _, vs = program(text)
    reg = Registry()
    for v in vs:
        reg.register(v)
    return reg


def _descs(lib_path):
    lib = ctypes.CDLL(str(lib_path))
    count = ctypes.c_int.in_dll(lib, "tloops_entry_count").value
    entries = (refc.TlEntry * count).in_dll(lib, "tloops_entries")
    out = []
    for e in entries:
        args = []
        for a in range(e.n_args):
            d = e.args[a]
            pairs = [d.outer_pairs[i] for i in range(2 * d.n_outer_pairs)]
            ipairs = [d.inner_pairs[i] for i in range(2 * d.n_inner_pairs)]
            alias = [d.alias[i] for i in range(d.n_flat)] if d.alias else []
            args.append((d.name, d.kind, d.dim, d.outer_rank, d.inner_rank, pairs, ipairs,
                         d.n_components, d.n_flat, alias, d.value))
        out.append((e.ordinal, e.signature, e.n_args, args))
    return out, lib


@pytest.mark.parametrize("name", ["suite", "p3", "c2_maxwell"])
def test_manifest_identical_to_reference(name, tmp_path):
    if not refc.available(name):
        pytest.skip("oracle/_ref not built")
    text = (refc.REF_DIR / f"{name}.tl").read_text()
    reg = _registry(text)
    assert reg.manifest_text() == (refc.REF_DIR / f"{name}.manifest.tsv").read_text()


@pytest.mark.parametrize("name", ["suite", "p3", "c2_maxwell"])
def test_bindings_descriptors_equal_reference(name, tmp_path):
    if not refc.available(name):
        pytest.skip("oracle/_ref not built")
    text = (refc.REF_DIR / f"{name}.tl").read_text()
    so = _registry(text).build_shared(tmp_path)
    ours, _l1 = _descs(so)
    ref, _l2 = _descs(refc.REF_DIR / f"{name}.so")
    assert ours == ref


def test_dedup_and_ordinals():
    prog_text = tb.DTG + "dtg(sym<0,1>, i, j) = -2*alpha*K(i,j) + db(i,j) + db(j,i);\n"
    reg = _registry(prog_text)
    assert len(reg) == 1 and reg.entries[0].ordinal == 1


def test_build_shared_precompiles_the_harness_cubins(tmp_path, monkeypatch):
    # the bindings' tlb_harness_call looks its cubin up by FNV-1a of the
    # embedded source + options; build_shared puts it there (no GPU needed)
    import shutil

    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.registry import Registry, harness_cubin_name, harness_source
    from paper_1804_10120_b200.runtime import compile_options

    if not shutil.which("cc"):
        pytest.skip("no C compiler")
    monkeypatch.setenv("TLB_CACHE_DIR", str(tmp_path / "cache"))
    (tmp_path / "cache").mkdir()
    _, vs = tb.load(tb.P2)
    reg = Registry()
    for v in vs:
        reg.register(v)
    reg.build_shared(tmp_path / "gen")
    names = {harness_cubin_name(harness_source(v), compile_options()) for v in vs}
    assert {p.name for p in (tmp_path / "cache").glob("harness_*.cubin")} == names
    # the bindings embed exactly that source text
    text = (tmp_path / "gen" / "tloops_bindings_b200.c").read_text()
    assert text.count("static const char tl_src_") == len(vs)
