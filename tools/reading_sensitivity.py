"""sensitivity of the results to reading L4 (round-robin cursor
persists across kernels in a round [default] vs restarts at SM 0 per kernel).
Full spaces on the GPU under both readings; prints one JSON line."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_07983_b200 import rk, workloads as W

c = rk.Context(0)
out = {}
for name in ("C2", "C3", "C4"):
    gpu, ks = W.config(name)
    N = math.factorial(len(ks))
    res = {}
    keys = {}
    for flag in (0, 1):
        c.rk_set_gpu_params(list(gpu) + [flag])
        c.rk_set_kernels(ks)
        order, _, idx, key = c.rk_heuristic_order()
        kd = torch.empty(N, dtype=torch.int64, device="cuda")
        st = c.rk_eval_range(0, N, key, keys_dev=kd)
        keys[flag] = kd
        res[flag] = {"best_T": st.key_min / gpu[6], "argmin": st.argmin, "worst_T": st.key_max / gpu[6],
                     "heuristic_percentile": 100.0 * (st.n_eq + st.n_gt) / N,
                     "median_T": c.rk_select_keys(kd, N, st.key_min, st.key_max, [(N - 1) // 2])[0] / gpu[6]}
    diff = int((keys[0] != keys[1]).sum().item())
    out[name] = {"persist": res[0], "per_kernel": res[1], "orders_with_different_time": diff, "orders": N,
                 "same_argmin": res[0]["argmin"] == res[1]["argmin"]}
    del keys
sets = W.c5_sets(4096)
F = math.factorial(9)
for flag in (0, 1):
    c.rk_set_gpu_params(list(W.GTX580) + [flag])
    r = c.rk_eval_batch(sets)
    p = sorted(100.0 * (st.n_eq + st.n_gt) / F for st, _ in r)
    out.setdefault("C5_heuristic_percentile", {})["per_kernel" if flag else "persist"] = {
        "median": p[len(p) // 2], "mean": sum(p) / len(p), "frac_ge_90": sum(x >= 90 for x in p) / len(p)}
print(json.dumps(out))
