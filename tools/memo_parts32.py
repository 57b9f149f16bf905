"""Step cost split on C4 with the compact (u32) key stream (library phase events)
and a plain fill of the same u32 key buffer."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_1511_07983_b200 import rk, workloads as W  # noqa: E402

gpu, ks = W.config("C4")
c = rk.Context(0)
c.rk_set_gpu_params(gpu)
c.rk_set_kernels(ks)
N = math.factorial(12)
_, _, idx, key = c.rk_heuristic_order()
cand = torch.tensor([key], dtype=torch.int64, device="cuda")
rec = torch.zeros(8, dtype=torch.int64, device="cuda")
k32 = torch.empty(N, dtype=torch.int32, device="cuda")
ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
hist = torch.zeros(256, dtype=torch.int64, device="cuda")
base = c.rk_key_lower_bound()


def step():
    c.rk_sweep_pass1_async(0, N, cand, rec, None)
    hist.zero_()
    c.rk_sweep_pass2_32_async(0, N, cand, rec, 256, hist, k32, base, ovf, rec)


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


step()
torch.cuda.synchronize()
c.rk_set_timing(True)
ms = t(step)
ph = c.rk_timing_read()
c.rk_set_timing(False)
print("step", round(ms, 4), {k: round(v[0] / v[1], 4) for k, v in ph.items() if v[1]})
print("fill u32 1.92GB", round(t(lambda: k32.fill_(1)), 4), "ovf", int(ovf.item()))
