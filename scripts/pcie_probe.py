"""Raw host<->device copy ceilings on this box (pinned memory), for the e2e
leg's context: H2D alone, D2H alone, both directions at once."""
import json
import time

import torch

n = 1 << 30  # 8 GiB of fp64
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


gb = 8 * n / 1e9
print(json.dumps({
    "h2d_gbs": gb / t(lambda: d.copy_(h, non_blocking=True)),
    "d2h_gbs": gb / t(lambda: h2.copy_(d2, non_blocking=True)),
    "bidir_each_gbs": gb / t(both),
}))
