"""Soak test of the staged entries: random programs (the fuzz generator of
tests/helpers.py), random sizes (log-uniform, 1 .. 2^22 points) and random
ring shapes (depth 2-4, tiles 64-256, any staged share), each result checked
bitwise — against the CPU oracle up to 2^18 points, above that against the
plain flat entry of the same program.  Runs for --seconds and prints one
JSON summary line.
Usage: PYTHONPATH=.:tests python scripts/soak.py [--seconds 300]"""

import argparse
import json
import random
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

from helpers import FUZZ_DECLS, device_env, env_to_host, fuzz_statement, random_host_env, same_bits  # noqa: E402
from oracle import numpy_eval  # noqa: E402
from paper_1804_10120_b200.evaluator import _bind  # noqa: E402
from paper_1804_10120_b200.ir import ValidationError, validate_statement  # noqa: E402
from paper_1804_10120_b200.lowering import Variant, lower_program  # noqa: E402
from paper_1804_10120_b200.parser import parse_program  # noqa: E402
from paper_1804_10120_b200.runtime import Batch, Kernel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=300)
ap.add_argument("--seed", type=int, default=7)
ap.add_argument("--mode", choices=("staged", "default"), default="staged",
                help="staged: random TMA ring shapes; default: the lowering policy in force "
                     "through the public eval_program (one-shot grids, block shrink)")
args = ap.parse_args()
rng = random.Random(args.seed)
prog = parse_program(FUZZ_DECLS).program
stats = {"cases": 0, "staged": 0, "oracle_checked": 0, "flat_checked": 0, "batch_cases": 0,
         "mismatches": []}
t_end = time.time() + args.seconds
stream = torch.cuda.current_stream().cuda_stream


def run(stmts, env, variant, n):
    _, _, stores = _bind(stmts, env)
    k = Kernel(lower_program(stmts, variant=variant))
    k.launch(n, [s.base for s in stores], [s.pitch for s in stores], stream)
    torch.cuda.synchronize()
    return k


while time.time() < t_end:
    stmts = []
    while len(stmts) < rng.randint(1, 3):
        res = parse_program(FUZZ_DECLS + fuzz_statement(rng))
        if not res.ok:
            continue
        try:
            stmts.append(validate_statement(res.program.statements[0], res.program.decls))
        except ValidationError:
            continue
    if args.mode == "default":
        # the public API under the default policy: oracle up to 2^19 points,
        # above that the round-1 persistent 2-point entry of the same program
        from paper_1804_10120_b200 import eval_program

        n = int(2 ** rng.uniform(0, 22))
        host = random_host_env(prog, n, rng.randrange(1 << 30))
        env = device_env(prog, host)
        eval_program(stmts, env)
        torch.cuda.synchronize()
        got = env_to_host(env)
        stats["cases"] += 1
        try:  # programs the policy runs as independent statement parts
            from paper_1804_10120_b200.evaluator import plan_for

            stats["split"] = stats.get("split", 0) + plan_for(stmts, env).variant.split
        except Exception:
            pass
        if n <= 1 << 19:
            want = {key: a.copy() for key, a in host.items()}
            numpy_eval.eval_program(stmts, want)
            stats["oracle_checked"] += 1
        else:
            env2 = device_env(prog, host)
            run(stmts, env2, Variant(restrict=False), n)
            want = env_to_host(env2)
            stats["flat_checked"] += 1
        for key in want:
            if not same_bits(got[key], want[key]):
                stats["mismatches"].append({"n": n, "field": key, "mode": "default",
                                            "stmts": [str(v.stmt) for v in stmts]})
                break
        continue
    if rng.random() < 0.3:
        # multi-domain batch (plain or staged batch entry) vs the oracle
        var = Variant(stage=rng.choice([0, 2, 3]), stage_threads=rng.choice([64, 128, 256]),
                      stage_reads=rng.choice([0, 1, 3]), batch_vec=rng.choice([1, 2, 3]),
                      batch_threads=rng.choice([0, 64, 128]))
        sizes = [int(2 ** rng.uniform(0, 13)) for _ in range(rng.randint(1, 40))]
        hosts = [random_host_env(prog, m, rng.randrange(1 << 30)) for m in sizes]
        envs = [device_env(prog, h) for h in hosts]
        k = Kernel(lower_program(stmts, variant=var))
        bases, pitches = [], []
        for env in envs:
            _, _, stores = _bind(stmts, env)
            bases.append([st.base for st in stores])
            pitches.append([st.pitch for st in stores])
        Batch(k, bases, pitches, sizes, stream).launch(stream)
        torch.cuda.synchronize()
        stats["batch_cases"] += 1
        for env, h in zip(envs, hosts):
            want = {key: a.copy() for key, a in h.items()}
            numpy_eval.eval_program(stmts, want)
            got = env_to_host(env)
            bad = [key for key in want if not same_bits(got[key], want[key])]
            if bad:
                stats["mismatches"].append({"batch": True, "sizes": sizes, "variant": var.tag(),
                                            "field": bad[0],
                                            "stmts": [str(v.stmt) for v in stmts]})
                break
        continue
    n = int(2 ** rng.uniform(0, 22))
    var = Variant(stage=rng.choice([2, 3, 4]), stage_threads=rng.choice([64, 128, 256]),
                  stage_reads=rng.choice([0, 1, 2, 5, 9, 17]), hoist=rng.random() < 0.5)
    if lower_program(stmts, variant=var).variant.stage == 0 and rng.random() < 0.85:
        continue  # mostly programs the staged entry can take (no read-write slot)
    host = random_host_env(prog, n, rng.randrange(1 << 30))
    env = device_env(prog, host)
    k = run(stmts, env, var, n)
    got = env_to_host(env)
    stats["cases"] += 1
    stats["staged"] += int(k.vec == 3)
    if n <= 1 << 18:
        want = {key: a.copy() for key, a in host.items()}
        numpy_eval.eval_program(stmts, want)
        stats["oracle_checked"] += 1
    else:
        env2 = device_env(prog, host)
        run(stmts, env2, Variant(), n)
        want = env_to_host(env2)
        stats["flat_checked"] += 1
    for key in want:
        if not same_bits(got[key], want[key]):
            stats["mismatches"].append({"n": n, "variant": var.tag(), "field": key,
                                        "stmts": [str(v.stmt) for v in stmts]})
            break
    del env
print(json.dumps(stats))
