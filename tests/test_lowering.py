"""Lowering (expression tree → fused kernel source): structure, NVRTC
compile for sm_100a, and static SASS checks — all without a GPU."""

import shutil
import subprocess

import pytest

from helpers import case_names, manifest, program
from paper_1804_10120_b200.lowering import SLOT_READ, SLOT_WRITE, lower_program
from paper_1804_10120_b200.runtime import get_kernel


def _sass(kernel) -> str:
    path = kernel.cubin_path
    if not path.exists():
        path.write_bytes(kernel.cubin())
    return subprocess.run(["cuobjdump", "-sass", str(path)], capture_output=True, text=True,
                          check=True).stdout


@pytest.mark.parametrize("name", case_names())
def test_every_golden_program_compiles_for_sm100a(name):
    case = manifest()["cases"][name]
    _, vs = program(case["source"])
    if case.get("raises", {}).get("type") == "ZeroDivisionError":
        # a literal `1/0`: the reference raises when the statement runs, and
        # so does lowering (Python-scalar folding); the statements before it lower
        with pytest.raises(ZeroDivisionError):
            lower_program(vs)
        vs = vs[:-1]
    plan = lower_program(vs)
    k = get_kernel(plan)
    assert len(k.cubin()) > 0


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="no cuobjdump")
@pytest.mark.parametrize("name", ["c3_christoffel", "c4_p2", "suite_kij", "c1_dtg"])
def test_no_fma_contraction_no_spills(name):
    # --fmad=false is a parity requirement: no DFMA may appear
    _, vs = program(manifest()["cases"][name]["source"])
    k = get_kernel(lower_program(vs))
    sass = _sass(k)
    assert "DFMA" not in sass
    assert "LDL" not in sass and "STL" not in sass
    assert any("LDG" in ln and ".128" in ln for ln in sass.splitlines())  # 128-bit loads
    assert "STG.E.EF.128" in sass  # streaming 128-bit stores


def test_algorithmic_bytes_equal_reference_counts():
    # single '=' statements that do not read their target: slots == N_e
    for name in ("c1_dtg", "c3_christoffel", "suite_contract3", "suite_kij"):
        case = manifest()["cases"][name]
        _, (v,) = program(case["source"])
        plan = lower_program([v])
        n_e = case["statements"][0]["count_data"][0]
        assert plan.n_slots == n_e
        assert plan.bytes_per_point == 8 * n_e


def test_program_fusion_counts():
    # C4 P2: 40 reads + 24 writes = 512 B/pt; P3: intermediates stay in
    # registers, 76 arrays
    _, vs = program(manifest()["cases"]["c4_p2"]["source"])
    p2 = lower_program(vs)
    assert (p2.reads, p2.writes, p2.bytes_per_point) == (40, 24, 512)
    assert p2.flops_per_point == 216 + 24
    _, vs = program(manifest()["cases"]["c4_p3"]["source"])
    p3 = lower_program(vs)
    assert p3.n_slots == 76


def test_register_shadow_reads_after_writes():
    _, vs = program("tensor A dim 3 rank 2;\nA(i, j) = A(j, i);\n")
    plan = lower_program(vs)
    # every component is written; only components not yet written when read
    # are loaded from memory: A(0,1),(0,2),(1,2) are read before written... and
    # the diagonal reads itself before its own write
    reads = [c for c, f in zip(plan.slot_comp, plan.slot_flags) if f & SLOT_READ]
    writes = [c for c, f in zip(plan.slot_comp, plan.slot_flags) if f & SLOT_WRITE]
    assert sorted(writes) == list(range(9))
    assert sorted(reads) == [0, 3, 4, 6, 7, 8]


def test_literal_division_by_zero_raises_like_reference():
    _, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(i)*(1/0);\n")
    with pytest.raises(ZeroDivisionError):
        lower_program(vs)


def test_signed_zero_literals_not_merged():
    _, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nfield w;\n"
                    "A(i) = B(i)*(w + 0)*(w + -0);\n")
    src = lower_program(vs).source
    assert "(0x0.0p+0)" in src and "(-0x0.0p+0)" in src


def test_reference_built_trees_lower_identically():
    ref = pytest.importorskip("tlang.parser", reason="reference package not importable")
    del ref
    import sys

    from tlang.ir import validate_statement as ref_validate
    from tlang.parser import parse_program as ref_parse

    src = manifest()["cases"]["c4_p3"]["source"]
    r = ref_parse(src).program
    ref_vs = [ref_validate(s, r.decls) for s in r.statements]
    _, my_vs = program(src)
    assert lower_program(ref_vs).source == lower_program(my_vs).source
    assert "tlang" in sys.modules


def test_same_source_different_slot_maps_are_distinct_kernels():
    # per-component kernels of A(i,j) = A(j,i): k=1 and k=2 emit the same
    # text (load slot 0, store slot 1) over different components
    _, (v,) = program("tensor A dim 3 rank 2;\nA(i, j) = A(j, i);\n")
    p1 = lower_program([v], components=[{1}])
    p2 = lower_program([v], components=[{2}])
    assert p1.source == p2.source and p1.key != p2.key
    assert get_kernel(p1) is not get_kernel(p2)
    assert get_kernel(p1).cache_key == get_kernel(p2).cache_key  # cubin shared on disk


def test_movable_loads_refused_when_a_slot_is_read_and_written():
    from paper_1804_10120_b200.lowering import Variant

    _, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) += B(i);\n")
    plan = lower_program(vs, variant=Variant(ldmode=1))
    assert plan.variant.ldmode == 0 and "#define TLK_LDMODE 0" in plan.source
    _, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) = B(i);\n")
    plan = lower_program(vs, variant=Variant(ldmode=1))
    assert plan.variant.ldmode == 1 and "#define TLK_LDMODE 1" in plan.source


@pytest.mark.parametrize("hoist", [False, True])
@pytest.mark.parametrize("restrict", [False, True])
def test_variants_compile(hoist, restrict):
    from paper_1804_10120_b200.lowering import Variant

    _, vs = program(manifest()["cases"]["c4_p3"]["source"])
    k = get_kernel(lower_program(vs, variant=Variant(restrict=restrict, hoist=hoist, ldmode=1)))
    assert "DFMA" not in _sass(k)


def _defines(src: str) -> dict:
    out = {}
    for ln in src.splitlines():
        if ln.startswith("#define TLK_"):
            parts = ln.split(None, 2)
            # the generated header comes first; the template's #ifndef
            # defaults after it must not override it
            out.setdefault(parts[1], parts[2] if len(parts) > 2 else "")
    return out


@pytest.mark.parametrize("name,depth,tile,staged,ws", [
    ("c1_dtg", 3, 256, 8, 1), ("c2_maxwell", 3, 256, 9, 0), ("c3_christoffel", 3, 256, 18, 1),
    ("c4_p2", 2, 256, 34, 1), ("c4_p3", 2, 256, 32, 1)])
def test_staged_policy_ring_layout(name, depth, tile, staged, ws, monkeypatch):
    # policy 2's ring (warp-specialised except for multi-statement light
    # programs; 2-deep for 32+ reads), its staged share, and the ring's
    # read-slot ordinals: the first `staged` read slots in slot order,
    # numbered densely
    monkeypatch.setenv("TLK_POLICY", "2")
    _, vs = program(manifest()["cases"][name]["source"])
    plan = lower_program(vs)
    var = plan.variant
    assert var.stage == depth and var.stage_threads == tile and var.stage_ws == ws
    d = _defines(plan.source)
    assert int(d.get("TLK_STAGE_WS", "0")) == ws
    rord = [int(x) for x in d["TLK_RORD"].strip("{}").split(",")]
    assert int(d["TLK_NREAD"]) == staged == sum(1 for r in rord if r >= 0)
    reads = [j for j, fl in enumerate(plan.slot_flags) if fl & SLOT_READ]
    assert [rord[j] for j in reads[:staged]] == list(range(staged))
    assert all(rord[j] == -1 for j in range(len(rord)) if j not in reads[:staged])
    assert depth * staged * tile * 8 <= 224 * 1024
    assert int(d["TLK_STAGE_THREADS"]) == tile and int(d["TLK_THREADS"]) == 256


def test_contraction_class_policy_stages_40_reads_in_128_point_tiles(monkeypatch):
    # contract1 (90 reads, 81 writes): policy 1 left it unstaged (a 3-deep
    # ring of 3/4 of its reads leaves 4 warps per SM); policy 2 stages 40
    # reads through a 2-deep ring of 128-point tiles, warp-specialised
    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.lowering import choose_variant

    monkeypatch.setenv("TLK_POLICY", "2")

    src = {e.name: e.source for e in tb.builtin_suite()}["contract1"]
    _, vs = program(src)
    var = lower_program(vs).variant
    assert (var.stage, var.stage_threads, var.stage_reads, var.stage_ws) == (2, 128, 40, 1)
    assert choose_variant(90, 81, 405, 0, 0, policy=1).stage == 3  # then refused by the warp rule


@pytest.mark.parametrize("name,vec,threads,hoist,ldmode", [
    ("c1_dtg", 1, 512, True, 0), ("c2_maxwell", 1, 512, True, 0),
    ("c3_christoffel", 1, 128, False, 1), ("c4_p2", 1, 128, False, 1),
    ("c4_p3", 1, 128, True, 1), ("suite_outer3", 1, 512, True, 0),
    ("suite_assign3", 1, 512, True, 0), ("suite_contract1", 1, 128, False, 1)])
def test_default_policy_is_one_shot_flat(name, vec, threads, hoist, ldmode):
    # policy 3 (the default): the plain entry over a one-shot grid, no TMA
    # ring, no size class; the launch geometry travels in the source for
    # C-ABI callers that pass none (tlb_exec_host, the harness bindings)
    _, vs = program(manifest()["cases"][name]["source"])
    plan = lower_program(vs)
    var = plan.variant
    assert (var.stage, var.waves, var.vec, var.threads, var.hoist, var.ldmode, var.small_n) == \
        (0, 0, vec, threads, hoist, ldmode, 0)
    d = _defines(plan.source)
    assert d["TLK_GRID_WAVES"] == "0" and d["TLK_VEC"] == str(vec)
    assert d["TLK_THREADS"] == str(threads) and "TLK_NSTAGE" not in d
    k = get_kernel(plan)
    assert k.max_blocks == 1 << 62 and k.vec == 1 and k.small is None


def test_spilling_programs_are_lowered_in_output_groups():
    # contract3 (761 values live under program-wide value numbering: 5.7 KB
    # of spills per thread) is split into output groups — non-inlined device
    # functions of <= 64 live values; contract2 (94 live) is not
    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.lowering import _max_live

    src = {e.name: e.source for e in tb.builtin_suite()}
    _, vs = program(src["contract3"])
    plan = lower_program(vs)
    assert plan.variant.vn == 1 and plan.source.count("__noinline__ void tlk_grp") == 3
    assert plan.flops_per_point == 8667  # algorithmic count, unchanged by recomputation
    _, vs = program(src["contract2"])
    plan = lower_program(vs)
    assert plan.variant.vn == 0 and "tlk_grp" not in plan.source
    from paper_1804_10120_b200.lowering import Instr

    # the live-range estimate itself
    ins = [Instr("ld", 0, slot=0), Instr("ld", 1, slot=1), Instr("mul", 2, 0, 1),
           Instr("st", a=2, slot=2), Instr("ld", 3, slot=3), Instr("st", a=3, slot=4)]
    assert _max_live(ins) == 2


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="no cuobjdump")
def test_output_groups_remove_the_spills():
    from paper_1804_10120_b200 import bench as tb

    _, vs = program({e.name: e.source for e in tb.builtin_suite()}["contract3"])
    k = get_kernel(lower_program(vs))
    out = subprocess.run(["cuobjdump", "-res-usage", str(k.cubin_path)], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    line = next(out[i + 1] for i, ln in enumerate(out) if "tlk_flat_v1" in ln)
    stack = int(line.split("STACK:")[1].split()[0])
    assert stack < 1024  # call frames only (5736 bytes of spills ungrouped)


def test_read_modify_write_programs_run_hoisted_one_shot():
    _, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) += B(i);\n")
    var = lower_program(vs).variant
    assert (var.vec, var.waves, var.threads, var.restrict, var.hoist, var.ldmode) == \
        (1, 0, 128, False, True, 0)


def test_stage_refused_for_read_write_and_read_free_programs():
    from paper_1804_10120_b200.lowering import Variant

    _, vs = program("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\nA(i) += B(i);\n")
    assert lower_program(vs, variant=Variant(stage=3)).variant.stage == 0
    _, vs = program("tensor A dim 3 rank 2;\nA(i,j) = 1.5;\n")
    plan = lower_program(vs, variant=Variant(stage=3))
    assert plan.variant.stage == 0 and "#define TLK_NSTAGE" not in plan.source


def test_stage_ring_clamped_to_shared_memory():
    # 4 x 256-point tiles of 64 reads would need 512 KB: depth, then tile,
    # shrink until the ring fits the 224 KB budget
    from paper_1804_10120_b200.lowering import STAGE_SMEM_MAX, Variant

    _, vs = program(manifest()["cases"]["c4_p3"]["source"])
    plan = lower_program(vs, variant=Variant(stage=4, stage_threads=256))
    var = plan.variant
    assert var.stage >= 2
    assert var.stage * plan.reads * var.stage_threads * 8 <= STAGE_SMEM_MAX


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="no cuobjdump")
@pytest.mark.parametrize("ws", [0, 1])
def test_staged_entries_use_bulk_copies_without_spills(ws):
    from paper_1804_10120_b200.lowering import Variant

    _, vs = program(manifest()["cases"]["c4_p2"]["source"])
    # the staged entry is a variant (policy 3 does not pick it; policy 2 did)
    k = get_kernel(lower_program(vs, variant=Variant(stage=2, stage_threads=256,
                                                     stage_reads=34, stage_ws=ws, ldmode=1)))
    sass = _sass(k)
    # the staged batch entry is opt-in (measured slower): not in default modules
    assert "tlk_stage_v1" in sass and "tlk_stage_batch_v1" not in sass
    assert "tlk_stage_v1" not in _sass(get_kernel(lower_program(vs)))

    opt = get_kernel(lower_program(vs, variant=Variant(stage=3, batch_vec=3)))
    assert "tlk_stage_batch_v1" in _sass(opt)
    assert "UBLKCP" in sass  # cp.async.bulk (TMA engine)
    assert "SYNCS" in sass  # mbarrier operations
    assert "LDL" not in sass and "STL" not in sass
    assert "DFMA" not in sass


def test_statement_parts():
    # independent statements (no field in common, transitively) form parts
    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.lowering import statement_parts

    assert statement_parts(tb.load(tb.P2)[1]) == [[0], [1]]
    assert statement_parts(tb.load(tb.MAXWELL)[1]) == [[0, 1, 2, 7], [3, 4, 5, 6]]
    assert statement_parts(tb.load(tb.P3)[1]) == [[0, 1, 2]]  # chained through Gamma, db
    _, vs = tb.load(tb.P2)
    # two names for one storage join their statements into one part
    assert statement_parts(vs, {"K": "dg"}) == [[0, 1]]


def test_split_policy_keeps_field_order_and_emits_parts():
    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.lowering import Variant

    for text, parts in ((tb.P2, 2), (tb.MAXWELL, 2)):
        _, vs = tb.load(text)
        plan = lower_program(vs)
        assert plan.variant.split == 1 and "y" in plan.variant.tag()
        assert f"#define TLK_PARTS {parts}" in plan.source
        assert "tlk_part(const unsigned part" in plan.source
        flat = lower_program(vs, variant=Variant(**{**plan.variant.__dict__, "split": 0}))
        # callers bind fields by the plan's order: splitting must not change it
        assert [f.name for f in plan.fields] == [f.name for f in flat.fields]
        assert plan.bytes_per_point == flat.bytes_per_point
        assert plan.flops_per_point == flat.flops_per_point
        assert sorted(zip(plan.slot_field, plan.slot_comp, plan.slot_flags)) == \
            sorted(zip(flat.slot_field, flat.slot_comp, flat.slot_flags))
    # a single part, or output groups, never split
    _, vs = tb.load(tb.P3)
    assert lower_program(vs).variant.split == 0
    _, vs = tb.load(tb.P2)
    assert lower_program(vs, variant=Variant(split=1, vn=1)).variant.split == 0


def test_split_kernel_compiles_with_fewer_registers():
    # P2's parts alone need fewer registers than the fused body (128 -> 89)
    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.lowering import Variant

    if not shutil.which("cuobjdump"):
        pytest.skip("no cuobjdump")
    _, vs = tb.load(tb.P2)
    plan = lower_program(vs)
    flat = lower_program(vs, variant=Variant(**{**plan.variant.__dict__, "split": 0}))

    def regs(p):
        k = get_kernel(p)
        path = k.cubin_path
        if not path.exists():
            path.write_bytes(k.cubin())
        out = subprocess.run(["cuobjdump", "-res-usage", str(path)], capture_output=True,
                             text=True, check=True).stdout.splitlines()
        for i, line in enumerate(out):
            if "tlk_flat_v1" in line:
                return int(out[i + 1].split("REG:")[1].split()[0])
        raise AssertionError("no tlk_flat_v1")

    assert regs(plan) < regs(flat)


@pytest.mark.parametrize("name", ["c1_dtg", "c2_maxwell", "c3_christoffel", "p2", "p3"])
def test_c_abi_default_geometry_matches_the_python_launch(name):
    # tlb_launch_default reads TLK_VEC / TLK_GRID_WAVES (and a staged ring)
    # from the source; the Python Kernel launches the plan's variant: the two
    # must name the same entry and grid (tlb_runtime.cpp tlb_launch_default)
    import re

    from paper_1804_10120_b200 import bench as tb
    from paper_1804_10120_b200.runtime import ONE_SHOT, Kernel

    _, vs = tb.load(tb.PROGRAMS[name])
    plan = lower_program(vs)
    k = Kernel(plan)

    def define(key, dflt):
        m = re.search(rf"^#define {key} (\S+)", plan.source, re.M)
        return int(m.group(1)) if m else dflt

    waves = define("TLK_GRID_WAVES", 1)
    staged = define("TLK_NSTAGE", 0) > 0
    c_vec = 3 if staged else (0 if define("TLK_VEC", 2) == 2 else 1)
    c_mb = ONE_SHOT if waves == 0 else (-waves if waves > 1 else 0)
    assert (k.vec, k.max_blocks) == (c_vec, c_mb)


def test_split_policy_keeps_programs_with_a_tiny_part_fused():
    # a part streaming < SPLIT_MIN_ARRAYS arrays would be block-dispatch bound
    from paper_1804_10120_b200.lowering import Variant

    src = ("tensor G dim 3 rank 3 sym(1,2);\ntensor I dim 3 rank 2 sym(0,1);\n"
           "tensor D dim 3 rank 2 sym(0,1) inner rank 1;\n"
           "tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;\n"
           "G(sym<1,2>, i, j, k) = 0.5*Sum(l, I(i,l)*(D(j,l)(k)+D(l,k)(j)-D(j,k)(l)));\n"
           "A(i) = B(i);\n")
    _, vs = program(src)
    plan = lower_program(vs)
    assert plan.variant.split == 0  # the copy part: 6 arrays x 128 threads x 8 B
    # an explicit variant still splits (tests, tuning)
    assert lower_program(vs, variant=Variant(vec=1, waves=0, split=1)).variant.split == 1
    # 18 arrays per 128-thread block (18 KB) measured -1 to -2 % split: fused too
    _, vs = program(src.replace("tensor A dim 3 rank 1;\ntensor B dim 3 rank 1;",
                                "tensor A dim 3 rank 2;\ntensor B dim 3 rank 2;")
                    .replace("A(i) = B(i);", "A(i,j) = B(i,j);"))
    assert lower_program(vs).variant.split == 0
