"""Pass-2 cost split on C4: keys only / histogram only / neither / both."""
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
cand = torch.zeros(1, dtype=torch.int64, device="cuda")
_, _, idx, key = c.rk_heuristic_order()
cand[0] = key
rec = torch.zeros(8, dtype=torch.int64, device="cuda")
keys = torch.empty(N, dtype=torch.int64, device="cuda")
hist = torch.zeros(256, dtype=torch.int64, device="cuda")
c.rk_sweep_pass1_async(0, N, cand, rec, keys)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


print("pass1", t(lambda: c.rk_sweep_pass1_async(0, N, cand, rec, keys)))
print("keys+hist", t(lambda: c.rk_sweep_pass2_async(0, N, cand, rec, 256, hist, keys, rec)))
print("keys only", t(lambda: c.rk_sweep_pass2_async(0, N, cand, rec, 256, None, keys, rec)))
print("hist only", t(lambda: c.rk_sweep_pass2_async(0, N, cand, rec, 256, hist, None, rec)))
print("neither", t(lambda: c.rk_sweep_pass2_async(0, N, cand, rec, 256, None, None, rec)))
print("torch fill 3.83GB", t(lambda: keys.fill_(1)))
