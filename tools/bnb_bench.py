"""Branch-and-bound exact optimum (rk_best_order) on n = 12..16 generator sets:
wall time, nodes visited vs the n!*n exhaustive placements, and (n <= 13)
agreement with the exhaustive device sweep.  Writes one JSON line per case."""
import json
import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1511_07983_b200 import rk  # noqa: E402
from paper_1511_07983_b200 import workloads as W  # noqa: E402


def main():
    ns = [int(x) for x in sys.argv[1:]] or [12, 13, 14, 15, 16]
    c = rk.Context(0)
    for name in ("C2", "C3", "C4"):
        gpu, ks = W.config(name)
        c.rk_set_gpu_params(gpu)
        c.rk_set_kernels(ks)
        _, _, hidx, hkey = c.rk_heuristic_order()
        for seed in (None, hidx):
            t0 = time.perf_counter()
            o, idx, key, nodes = c.rk_best_order(seed)
            dt = time.perf_counter() - t0
            print(json.dumps({"config": name, "n": 12, "seeded": seed is not None, "s": round(dt, 4), "key": key,
                              "index": idx, "nodes": nodes, "frac_of_tree": nodes / (12 * math.factorial(12))}),
                  flush=True)
    for n in ns:
        for rep in range(2):
            ks = W.gen_g(W.SplitMix64(W.SEED_BASE + 1000 * n + rep), n)
            c.rk_set_gpu_params(W.GTX580)
            c.rk_set_kernels(ks)
            _, _, hidx, hkey = c.rk_heuristic_order()
            t0 = time.perf_counter()
            o, idx, key, nodes = c.rk_best_order(hidx)
            dt = time.perf_counter() - t0
            rec = {"n": n, "rep": rep, "s": round(dt, 4), "key": key, "index": idx, "heur_key": hkey,
                   "nodes": nodes, "frac_of_tree": nodes / (n * math.factorial(n))}
            if n <= 13:
                N = math.factorial(n)
                r = torch.zeros(8, dtype=torch.int64, device="cuda")
                cd = torch.zeros(1, dtype=torch.int64, device="cuda")
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                c.rk_eval_range_async(0, N, cd, r)
                torch.cuda.synchronize()
                rec["full_sweep_s"] = round(time.perf_counter() - t0, 4)
                st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(r.cpu().numpy().tobytes()))
                rec["agrees_full_sweep"] = (st.key_min, st.argmin) == (key, idx)
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
