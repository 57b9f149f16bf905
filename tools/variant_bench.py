"""Time rk_eval_kernel on C4 (12!) for one librk build (RK_LIB=path) and check
the result against tests/golden/c4_oracle.json.  Dev tool for kernel variants."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_07983_b200 import rk, workloads as W

g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c4_oracle.json")))
gpu, ks = W.config("C4")
c = rk.Context(0)
c.rk_set_gpu_params(gpu)
c.rk_set_kernels(ks)
N = math.factorial(12)
keys = torch.empty(N, dtype=torch.int64, device="cuda")
cand = torch.tensor([g["cand_key"]], dtype=torch.int64, device="cuda")
rec = torch.zeros(8, dtype=torch.int64, device="cuda")
with_keys = os.environ.get("NOKEYS") is None
for _ in range(3):
    c.rk_eval_range_async(0, N, cand, rec, keys if with_keys else None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    c.rk_eval_range_async(0, N, cand, rec, keys if with_keys else None)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
want = tuple(g["stats"][f] for f in ("key_min", "key_max", "argmin", "argmax", "n_lt", "n_eq", "n_gt", "evaluated"))
ok = st.as_tuple() == want
print(json.dumps({"lib": os.environ.get("RK_LIB", "default"), "ms": ms, "perms_per_s": N / ms * 1e3, "parity": ok}))
