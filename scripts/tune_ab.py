"""Interleaved A/B of lowering variants on one B200: for each (program, N)
every variant runs ROUNDS times in round-robin order (so clock and thermal
drift hit all variants alike), each time K eager launches back to back
bracketed by CUDA events; reported: median and min per variant, and every
variant's output compared bitwise with the first's.

Cases come from the CASES env var (JSON list of
{"program": name, "n": points, "variants": {label: {Variant overrides}}}),
overrides applied on top of the policy variant; default: the round-2
warp-specialisation candidates.

Usage: python scripts/tune_ab.py  -> JSON lines"""

from __future__ import annotations

import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1804_10120_b200 import bench as tb  # noqa: E402
from paper_1804_10120_b200.lowering import Variant, lower_program  # noqa: E402
from paper_1804_10120_b200.runtime import fill_uniform, get_kernel  # noqa: E402

ROUNDS = int(os.environ.get("ROUNDS", "7"))
K = int(os.environ.get("K", "10"))

DEFAULT = [
    {"program": "p2", "n": 1 << 28, "variants": {
        "policy": {}, "ws_s2": {"stage_ws": 1, "stage": 2},
        "ws_s2_r40": {"stage_ws": 1, "stage": 2, "stage_reads": 40},
        "ws_s2_r30": {"stage_ws": 1, "stage": 2, "stage_reads": 30}}},
    {"program": "p3", "n": 1 << 26, "variants": {
        "policy": {}, "ws_s2": {"stage_ws": 1, "stage": 2}}},
    {"program": "c3_christoffel", "n": 1 << 21, "variants": {
        "policy": {"small_n": 0}, "ws": {"small_n": 0, "stage_ws": 1}}},
    {"program": "c3_christoffel", "n": 1 << 26, "variants": {
        "policy": {}, "ws": {"stage_ws": 1}}},
    {"program": "c1_dtg", "n": 1 << 26, "variants": {
        "policy": {}, "ws": {"stage_ws": 1}}},
    {"program": "c2_maxwell", "n": 1 << 26, "variants": {
        "policy": {}, "ws": {"stage_ws": 1}}},
]


def source(name: str) -> str:
    if name in tb.PROGRAMS:
        return tb.PROGRAMS[name]
    return {e.name: e.source for e in tb.builtin_suite()}[name]


def run(case):
    name, n = case["program"], int(case["n"])
    prog, vs = tb.load(case.get("source") or source(name))
    base = lower_program(vs)
    if case.get("staged_only") and not base.variant.stage:
        print(json.dumps({"program": name, "N": n, "skipped": "not staged by the policy",
                          "variant": base.variant.tag()}), flush=True)
        return
    bufs = []
    for k, info in enumerate(base.fields):
        b = torch.zeros(info.n_components, n, dtype=torch.float64, device="cuda")
        if k not in base.lhs_fields:
            for c in range(info.n_components):
                fill_uniform(b[c], 0xC0FFEE, (k << 8) | c)
        bufs.append(b)
    bases = [b.data_ptr() for b in bufs]
    pitches = [n if info.n_components > 1 else 0 for info in base.fields]
    stream = torch.cuda.current_stream().cuda_stream
    kerns, plans, same, launch_kw = {}, {}, {}, {}
    want = None
    for label, over in case["variants"].items():
        if "__policy__" in over or "__env__" in over:
            # the lowering policy's own choice under TLK_POLICY=k / other env
            envs = dict(over.get("__env__", {}))
            if "__policy__" in over:
                envs["TLK_POLICY"] = str(over["__policy__"])
            saved = {k: os.environ.get(k) for k in envs}
            os.environ.update(envs)
            import importlib

            from paper_1804_10120_b200 import lowering as _lw
            _lw.VN_LIVE_BUDGET = int(os.environ.get("TLK_VN_BUDGET", "64"))
            plan = lower_program(vs)
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k)
                else:
                    os.environ[k] = v
            _lw.VN_LIVE_BUDGET = int(os.environ.get("TLK_VN_BUDGET", "64"))
            del importlib
        else:
            var = Variant(**{**base.variant.__dict__,
                             **{k: v for k, v in over.items() if not k.startswith("__")}})
            plan = lower_program(vs, variant=var)
        kern = get_kernel(plan)
        lk = dict(over.get("__launch__", {}))
        if lk.get("max_blocks") == "all":  # non-persistent: one thread per point (pair)
            lk["max_blocks"] = -(-n // (lk.get("vec", 1) * kern.threads))
        elif isinstance(lk.get("max_blocks"), str) and lk["max_blocks"].startswith("tiles"):
            per = int(lk["max_blocks"][5:] or 1)  # "tilesK": K tiles per staged block
            lk["max_blocks"] = max(1, n // plan.variant.stage_threads // per)
        launch_kw[label] = lk
        for k in base.lhs_fields:
            bufs[k].zero_()
        kern.launch(n, bases, pitches, stream, **lk)
        torch.cuda.synchronize()
        out = torch.cat([bufs[k][:, ::1009].flatten() for k in base.lhs_fields])
        if want is None:
            want = out.clone()
        same[label] = bool(torch.equal(out.view(torch.int64), want.view(torch.int64)))
        kerns[label], plans[label] = kern, plan
    ts = {label: [] for label in kerns}
    for _ in range(ROUNDS):
        for label, kern in kerns.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(K):
                kern.launch(n, bases, pitches, stream, **launch_kw[label])
            b.record()
            b.synchronize()
            ts[label].append(a.elapsed_time(b) / 1e3 / K)
    for label, t in ts.items():
        med = statistics.median(t)
        bpp = plans[label].bytes_per_point
        print(json.dumps({"program": name, "N": n, "shape": label,
                          "variant": plans[label].variant.tag(),
                          "us_median": round(med * 1e6, 2), "us_min": round(min(t) * 1e6, 2),
                          "tbs_median": round(bpp * n / med / 1e12, 4),
                          "tbs_best": round(bpp * n / min(t) / 1e12, 4),
                          "bitwise_same": same[label],
                          "us_all": [round(x * 1e6, 1) for x in t]}), flush=True)
    del bufs, kerns
    torch.cuda.empty_cache()


def main():
    cases = json.loads(os.environ["CASES"]) if os.environ.get("CASES") else DEFAULT
    if os.environ.get("SUITE_WS"):  # every suite statement: policy vs warp-specialised ring
        n = int(os.environ["SUITE_WS"])
        cases = [{"program": e.name, "n": n, "staged_only": True,
                  "variants": {"policy": {}, "ws": {"stage_ws": 1},
                               "ws_s2": {"stage_ws": 1, "stage": 2}}}
                 for e in tb.builtin_suite()]
        cases += [{"program": "c2_maxwell", "n": n, "variants": {
            "policy": {}, "ws": {"stage_ws": 1}, "ws_r12": {"stage_ws": 1, "stage_reads": 12},
            "ws_r14": {"stage_ws": 1, "stage_reads": 14},
            "ws_r18_s2": {"stage_ws": 1, "stage_reads": 18, "stage": 2}}},
            {"program": "p2", "n": n, "variants": {
                "policy": {}, "ws_s2": {"stage_ws": 1, "stage": 2},
                "ws_s2_r32": {"stage_ws": 1, "stage": 2, "stage_reads": 32},
                "ws_s2_r36": {"stage_ws": 1, "stage": 2, "stage_reads": 36},
                "ws_s2_t128_r40": {"stage_ws": 1, "stage": 2, "stage_reads": 40,
                                   "stage_threads": 128},
                "ws_s3_t128_r40": {"stage_ws": 1, "stage": 3, "stage_reads": 40,
                                   "stage_threads": 128}}}]
        cases += [{"program": c, "n": n, "variants": {
            "policy": {}, "ws_s2_t128_r40": {"stage_ws": 1, "stage": 2, "stage_reads": 40,
                                             "stage_threads": 128},
            "ws_s2_r24": {"stage_ws": 1, "stage": 2, "stage_reads": 24}}}
            for c in ("contract1", "contract2")]
    if os.environ.get("POLICY_AB"):  # round-1 vs round-2 policy, every program
        sizes = [int(x) for x in os.environ["POLICY_AB"].split(",")]
        names = [e.name for e in tb.builtin_suite()] + list(tb.PROGRAMS)
        pa, pb = os.environ.get("POLICY_PAIR", "1,2").split(",")
        cases = [{"program": nm, "n": n, "variants": {f"policy{pa}": {"__policy__": int(pa)},
                                                      f"policy{pb}": {"__policy__": int(pb)}}}
                 for n in sizes for nm in names]
    if os.environ.get("ONESHOT"):  # one-shot grids: flat entry shapes vs staged entry
        sizes = [int(x) for x in os.environ["ONESHOT"].split(",")]
        names = os.environ.get("PROGS", "c1_dtg,c2_maxwell,c3_christoffel,p2,p3,kij,"
                                        "contract1,outer3,assign3").split(",")
        cases = []
        for n in sizes:
            for nm in names:
                v = {"policy": {},
                     "v1_np": {"stage": 0, "__launch__": {"vec": 1, "max_blocks": "all"}},
                     "v1_np_t128": {"stage": 0, "threads": 128,
                                    "__launch__": {"vec": 1, "max_blocks": "all"}},
                     "v1_np_t512": {"stage": 0, "threads": 512,
                                    "__launch__": {"vec": 1, "max_blocks": "all"}},
                     "v2_np": {"stage": 0, "__launch__": {"vec": 2, "max_blocks": "all"}}}
                if lower_program(tb.load(source(nm))[1]).variant.stage:
                    v["staged_np1"] = {"__launch__": {"vec": 3, "max_blocks": "tiles1"}}
                    v["staged_np4"] = {"__launch__": {"vec": 3, "max_blocks": "tiles4"}}
                cases.append({"program": nm, "n": n, "variants": v})
    if os.environ.get("CHUNKS"):  # block-local chunks in one-shot grids
        sizes = [int(x) for x in os.environ["CHUNKS"].split(",")]
        cases = [{"program": nm, "n": n, "variants": {
            "policy": {}, "chunk2": {"chunk": 2}, "chunk4": {"chunk": 4},
            "chunk8": {"chunk": 8}, "chunk4_t256": {"chunk": 4, "threads": 256}}}
            for n in sizes for nm in ("p2", "c3_christoffel", "c1_dtg", "c2_maxwell", "p3",
                                      "assign3", "outer3")]
    if os.environ.get("SPLITS"):  # independent statement parts (Variant.split)
        sizes = [int(x) for x in os.environ["SPLITS"].split(",")]
        cases = [{"program": nm, "n": n, "variants": {"policy": {}, "split": {"split": 1}}}
                 for n in sizes for nm in ("p2", "c2_maxwell")]
    if os.environ.get("SPLIT_THREADS"):  # block size of split programs (policy: split)
        sizes = [int(x) for x in os.environ["SPLIT_THREADS"].split(",")]
        cases = [{"program": nm, "n": n, "variants": {
            "policy": {}, "nosplit": {"split": 0}, "split_t128": {"threads": 128},
            "split_t256": {"threads": 256}, "split_t512": {"threads": 512}}}
            for n in sizes for nm in ("p2", "c2_maxwell")]
    if os.environ.get("SPLIT_MINB"):  # register caps (launch-bound min blocks) of split P2
        sizes = [int(x) for x in os.environ["SPLIT_MINB"].split(",")]
        cases = [{"program": "p2", "n": n, "variants": {
            "policy": {}, "minb6": {"minb": 6}, "minb7": {"minb": 7}, "minb8": {"minb": 8}}}
            for n in sizes]
    if os.environ.get("VNGROUPS"):  # output groups (Variant.vn) for the contractions
        sizes = [int(x) for x in os.environ["VNGROUPS"].split(",")]
        cases = [{"program": nm, "n": n, "variants": {
            "ungrouped": {"vn": 0},
            "budget48": {"__env__": {"TLK_VN_BUDGET": "48"}},
            "budget64": {"__env__": {"TLK_VN_BUDGET": "64"}},
            "budget96": {"__env__": {"TLK_VN_BUDGET": "96"}},
            "budget128": {"__env__": {"TLK_VN_BUDGET": "128"}}}}
            for n in sizes for nm in ("contract2", "contract3")]
    if os.environ.get("RMW"):  # read-modify-write programs: policy geometry vs one-shot shapes
        sizes = [int(x) for x in os.environ["RMW"].split(",")]
        srcs = {
            "rmw_add": "tensor A dim 3 rank 2;\ntensor B dim 3 rank 2;\nA(i, j) += B(i, j);\n",
            "rmw_scale": "tensor A dim 3 rank 2 sym(0,1);\nA(sym<0,1>, i, j) *= 2.0;\n",
            "rmw_gamma": tb.CHRISTOFFEL.replace(") = 0.5*", ") += 0.5*"),
            "rmw_dtg": tb.DTG.replace(") = -2*", ") += -2*"),
        }
        cases = []
        for n in sizes:
            for nm, src in srcs.items():
                cases.append({"program": nm, "n": n, "source": src, "variants": {
                    "policy": {},
                    "v1_np_t512": {"vec": 1, "waves": 0, "threads": 512, "hoist": True},
                    "v1_np_t128": {"vec": 1, "waves": 0, "threads": 128},
                    "v1_np_t256": {"vec": 1, "waves": 0, "threads": 256},
                    "v2_np_t256": {"vec": 2, "waves": 0, "threads": 256},
                    "v1_np_t128_h1": {"vec": 1, "waves": 0, "threads": 128, "hoist": True},
                    "v1_np_t256_h1": {"vec": 1, "waves": 0, "threads": 256, "hoist": True},
                    "v2_np_t256_h1": {"vec": 2, "waves": 0, "threads": 256, "hoist": True}}})
    if os.environ.get("HEAVY"):  # policy-3 heavier kernels: load flavour, hoist, register cap
        sizes = [int(x) for x in os.environ["HEAVY"].split(",")]
        cases = []
        for n in sizes:
            for nm in os.environ.get("PROGS", "c3_christoffel,p2,p3,contract1").split(","):
                cases.append({"program": nm, "n": n, "variants": {
                    "policy3": {},
                    "hoist": {"hoist": True},
                    "ldcs": {"ldmode": 0},
                    "minb4": {"minb": 4},
                    "minb6": {"minb": 6},
                    "minb8": {"minb": 8},
                    "t64": {"threads": 64},
                    "t256_minb3": {"threads": 256, "minb": 3},
                    "v2_t128": {"vec": 2, "__launch__": {"vec": 2}}}})
    if os.environ.get("WRITEDOM"):  # write-dominated / copy programs: launch shapes
        sizes = [int(x) for x in os.environ["WRITEDOM"].split(",")]
        cases = []
        for n in sizes:
            for nm in ("outer1", "outer2", "outer3", "assign1", "assign3"):
                cases.append({"program": nm, "n": n, "variants": {
                    "p2_v1_w4_t256": {"__policy__": 2},
                    "v1_w4_t256_h1": {"vec": 1, "waves": 4, "threads": 256, "hoist": True,
                                      "small_n": 0},
                    "v1_np_t256": {"vec": 1, "waves": 0, "threads": 256, "small_n": 0},
                    "v1_np_t512": {"vec": 1, "waves": 0, "threads": 512, "small_n": 0},
                    "v1_np_t512_h1": {"vec": 1, "waves": 0, "threads": 512, "hoist": True,
                                      "small_n": 0},
                    "v2_np_t256": {"vec": 2, "waves": 0, "threads": 256, "small_n": 0},
                    "v2_np_t512": {"vec": 2, "waves": 0, "threads": 512, "small_n": 0},
                    "v2_w4_t256": {"vec": 2, "waves": 4, "threads": 256, "small_n": 0}}})
    if os.environ.get("NONPERSISTENT"):  # grid-stride vs one-shot grids of the flat entries
        n = int(os.environ["NONPERSISTENT"])
        names = ["assign1", "assign3", "outer1", "outer3", "add3", "kij", "c1_dtg", "c2_maxwell",
                 "c3_christoffel", "p2", "contract1"]
        cases = [{"program": nm, "n": n, "variants": {
            "policy": {},
            "flat_v1_w4": {"stage": 0, "__launch__": {"vec": 1, "max_blocks": -4}},
            "flat_v1_np": {"stage": 0, "__launch__": {"vec": 1, "max_blocks": "all"}},
            "flat_v2_w1": {"stage": 0, "__launch__": {"vec": 2, "max_blocks": 0}},
            "flat_v2_np": {"stage": 0, "__launch__": {"vec": 2, "max_blocks": "all"}}}}
            for nm in names]
    for case in cases:
        run(case)


if __name__ == "__main__":
    main()
