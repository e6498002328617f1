"""Quick infrastructure check on a GPU box: library, NVRTC, launch, batch,
host staging, fill.  Prints JSON lines; used during development."""
import json, time
import numpy as np
import torch
from paper_1804_10120_b200 import parse_program, validate_statement, TensorField, ScalarField
from paper_1804_10120_b200 import eval_statement, eval_batch, eval_program
from paper_1804_10120_b200.runtime import fill_uniform, get_kernel
from paper_1804_10120_b200.evaluator import kernel_for

SRC = """tensor dtg dim 3 rank 2 sym(0,1);
field alpha;
tensor K dim 3 rank 2 sym(0,1);
tensor db dim 3 rank 2;
dtg(sym<0,1>, i, j) = -2*alpha*K(i,j) + db(i,j) + db(j,i);
"""
r = parse_program(SRC)
prog = r.program
v = validate_statement(prog.statements[0], prog.decls)
N = 64**3
rng = np.random.default_rng(0xC0FFEE)
env = {}
for it in prog.items:
    name = getattr(it, "name", None)
    if name in prog.decls.tensors:
        f = TensorField(name, prog.decls.tensors[name], N)
        if name != "dtg":
            f.data.copy_(torch.from_numpy(rng.uniform(0, 1, tuple(f.data.shape))))
        env[name] = f
    elif name in prog.decls.scalar_fields:
        f = ScalarField(name, N)
        f.data.copy_(torch.from_numpy(rng.uniform(0, 1, N)))
        env[name] = f
eval_statement(v, env)
torch.cuda.synchronize()
h = {k: f.data.cpu().numpy() for k, f in env.items()}
a, K, db = h["alpha"], h["K"][:, 0], h["db"][:, 0]
want = np.zeros((6, 1, N))
n = 0
comp = {(0,0):0,(1,0):1,(2,0):2,(1,1):3,(2,1):4,(2,2):5}
def kc(i, j):
    return comp[(max(i,j), min(i,j))] if False else comp[tuple(sorted((i,j), reverse=True))]
for (i, j) in [(0,0),(1,0),(2,0),(1,1),(2,1),(2,2)]:
    want[n, 0] = -2.0 * a * K[kc(i, j)] + db[i + 3*j] + db[j + 3*i]
    n += 1
got = h["dtg"]
print(json.dumps({"dtg_bitwise": bool((got == want).all()), "maxdiff": float(np.abs(got-want).max())}))
k = kernel_for(v, env)
print(json.dumps({"attrs": k.attrs("tlk_flat_v2")}))
# timing
for _ in range(3): eval_statement(v, env)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): eval_statement(v, env)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"dtg_ms": ms, "GBs": 176 * N / ms / 1e6}))
# big
N2 = 2**26
big = {}
for idx, name in enumerate(["dtg", "alpha", "K", "db"]):
    if name == "alpha":
        f = ScalarField(name, N2)
    else:
        f = TensorField(name, prog.decls.tensors[name], N2)
    fill_uniform(f.data.view(-1), 0xC0FFEE, idx)
    big[name] = f
for _ in range(3): eval_statement(v, big)
torch.cuda.synchronize()
e0.record()
for _ in range(10): eval_statement(v, big)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(json.dumps({"dtg_big_ms": ms, "GBs": 176 * N2 / ms / 1e6}))
# host staged
henv = {k: (f.to("cpu")) for k, f in env.items()}
t = time.time()
eval_statement(v, henv)
print(json.dumps({"host_staged_s": time.time()-t, "bitwise": bool((henv["dtg"].data.numpy() == want).all())}))
# batch
envs = []
for d in range(8):
    e = {k: f.to("cuda") for k, f in env.items()}
    e["dtg"].data.zero_()
    envs.append(e)
eval_batch([v], envs)
torch.cuda.synchronize()
print(json.dumps({"batch_ok": all(bool((e["dtg"].data.cpu().numpy() == want).all()) for e in envs)}))
