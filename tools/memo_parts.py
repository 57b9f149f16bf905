"""Step cost split on C4 (library phase events): memo tables, key stream
(with and without keys), histogram; and a plain fill of the same key buffer."""
import json
import math
import os
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


def phases(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    c.rk_set_timing(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    r = c.rk_timing_read()
    c.rk_set_timing(False)
    return {k: round(v[0] / v[1], 4) for k, v in r.items() if v[1]}


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


def step(k):
    c.rk_sweep_pass1_async(0, N, cand, rec, k)
    hist.zero_()
    c.rk_sweep_pass2_async(0, N, cand, rec, 256, hist, k, rec)


print("step with keys", t(lambda: step(keys)), phases(lambda: step(keys)))
print("step without keys", t(lambda: step(None)), phases(lambda: step(None)))
print("torch fill 3.83GB", t(lambda: keys.fill_(1)))
print("torch zero 3.83GB", t(lambda: keys.zero_()))

g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "c4_oracle.json")))
cand[0] = g["cand_key"]
step(keys)
torch.cuda.synchronize()
want = [g["stats"][f] for f in ("key_min", "key_max", "argmin", "argmax", "n_lt", "n_eq", "n_gt", "evaluated")]
got = [int(x) for x in rec.cpu().tolist()]
print("parity vs C4 oracle golden:", "OK" if got == want and hist.cpu().tolist() == g["hist"] else f"MISMATCH {got} {want}",
      os.environ.get("RK_LIB", "default"))
