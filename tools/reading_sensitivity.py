"""sensitivity of the results to the readings of L4/L5.

Readings (rk_gpu_params.flags): 0 = binding readings (next-fit cursor that
persists across kernels within a round; a block that fits nowhere closes the
round), 1 = cursor restarts at SM 0 per kernel, 2 = strict round robin, 4 =
skip-ahead, and the combinations 3, 5, 6, 7.  Full spaces of C2-C4 on the GPU
under every reading (the default through the memoised step, the others
through the per-order policy kernels), plus the C5 batch's heuristic
percentiles.  Prints one JSON line (profiles/r02_reading_sensitivity.json)."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_07983_b200 import rk, workloads as W

FLAGS = {0: "binding", 1: "cursor_per_kernel", 2: "strict_rr", 3: "strict_rr+cursor_per_kernel",
         4: "skip_ahead", 5: "skip_ahead+cursor_per_kernel", 6: "strict_rr+skip_ahead", 7: "all"}
c = rk.Context(0)
out = {"readings": FLAGS}
for name in ("C2", "C3", "C4"):
    gpu, ks = W.config(name)
    N = math.factorial(len(ks))
    res, base = {}, None
    for flag in FLAGS:
        c.rk_set_gpu_params(list(gpu) + [flag])
        c.rk_set_kernels(ks)
        order, _, idx, key = c.rk_heuristic_order()
        kd = torch.empty(N, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = c.rk_eval_range(0, N, key, keys_dev=kd)
        dt = time.perf_counter() - t0
        r = {"best_T": st.key_min / gpu[6], "argmin": st.argmin, "worst_T": st.key_max / gpu[6],
             "heuristic_percentile": 100.0 * (st.n_eq + st.n_gt) / N,
             "median_T": c.rk_select_keys(kd, N, st.key_min, st.key_max, [(N - 1) // 2])[0] / gpu[6],
             "eval_s": round(dt, 4), "orders_per_s": N / dt}
        if base is None:
            base = kd
        else:
            r["orders_with_different_time"] = int((kd != base).sum().item())
            del kd
        res[FLAGS[flag]] = r
    out[name] = {"orders": N, **res}
    del base
sets = W.c5_sets(4096)
F = math.factorial(9)
for flag in FLAGS:
    c.rk_set_gpu_params(list(W.GTX580) + [flag])
    r = c.rk_eval_batch(sets)
    p = sorted(100.0 * (st.n_eq + st.n_gt) / F for st, _ in r)
    out.setdefault("C5_heuristic_percentile", {})[FLAGS[flag]] = {
        "median": p[len(p) // 2], "mean": sum(p) / len(p), "frac_ge_90": sum(x >= 90 for x in p) / len(p)}
print(json.dumps(out))
