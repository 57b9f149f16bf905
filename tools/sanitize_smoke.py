"""Small end-to-end exercise of every device entry point, for compute-sanitizer."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_07983_b200 import rk, workloads as W

c = rk.Context(0)
for name in ("C1", "C2"):
    gpu, ks = W.config(name)
    c.rk_set_gpu_params(gpu)
    c.rk_set_kernels(ks)
    N = math.factorial(len(ks))
    order, _, idx, key = c.rk_heuristic_order()
    keys = torch.empty(N, dtype=torch.int64, device="cuda")
    st = c.rk_eval_range(0, N, key, keys_dev=keys)
    st2 = c.rk_eval_range(5, N - 11, key, keys_dev=keys[:N - 11])
    h = torch.zeros(256, dtype=torch.int64, device="cuda")
    c.rk_histogram(keys, N, st.key_min, st.key_max, 256, h)
    c.rk_select_keys(keys, N, st.key_min, st.key_max, [0, (N - 1) // 2, N - 1])
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    c.rk_eval_range_async(0, N, None, rec)
    h2 = torch.zeros(64, dtype=torch.int64, device="cuda")
    c.rk_eval_range_hist_async(0, N, None, None, rec, 64, h2)
    k32 = torch.empty(N, dtype=torch.int32, device="cuda")
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    c.rk_eval_range32_async(0, N, None, rec, k32, c.rk_key_lower_bound(), ovf)
    c.rk_histogram32_async(k32, N, c.rk_key_lower_bound(), rec, 64, h2)
    c.rk_simulate_order(order)
    c.rk_percentile(order, 0, N)
    recs = torch.zeros((2, 8), dtype=torch.int64, device="cuda")
    c.rk_eval_range_async(0, N // 2, None, recs[0])
    c.rk_eval_range_async(N // 2, N - N // 2, None, recs[1])
    c.rk_merge_stats_async(recs, 2, rec)
c.rk_set_gpu_params(W.GTX580)
c.rk_eval_batch(W.c5_sets(8))
c.rk_heuristic_batch(W.c5_sets(8))
# memoised step (levels, suffix rows, run pass, row multiset CAS, key stream): C3 through the public API
from paper_1511_07983_b200.sweep import Sweeper
gpu, ks = W.config("C3")
rep = Sweeper(gpu).run(ks)
assert sum(rep.hist) == rep.n_orders
c.rk_set_gpu_params((13, 32768, 49152, 48, 8, 411, 100))  # generic (runtime-S) variant
c.rk_set_kernels(W.W4)
c.rk_eval_range(0, 24, 0)
torch.cuda.synchronize()
print("sanitize smoke OK")
