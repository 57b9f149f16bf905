import math, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_07983_b200 import rk, workloads as W
gpu, ks = W.config("C4")
c = rk.Context(0); c.rk_set_gpu_params(gpu); c.rk_set_kernels(ks)
N = math.factorial(12)
keys = torch.empty(N, dtype=torch.int64, device="cuda")
st = c.rk_eval_range(0, N, 0, keys_dev=keys)
h = torch.zeros(256, dtype=torch.int64, device="cuda")
for _ in range(3): c.rk_histogram(keys, N, st.key_min, st.key_max, 256, h)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): c.rk_histogram(keys, N, st.key_min, st.key_max, 256, h)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"hist_ms": ms, "GBps": 8 * N / ms / 1e6, "mass_ok": int(h.sum().item()) == 23 * N}))
