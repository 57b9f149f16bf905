"""Config C5 (BASELINE.json configs[4]): 4096 random 9-kernel sets, each set's
full 9! space vs its Algorithm 1 order (rk_eval_batch).  Prints one JSON line:
evaluations/s and the percentile distribution of the heuristic."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_07983_b200 import rk, workloads as W

import numpy as np
sets = np.array(W.c5_sets(int(os.environ.get("C5_SETS", "4096"))), dtype=np.int64)  # (sets, 9, 6), host-resident
c = rk.Context(0)
c.rk_set_gpu_params(W.GTX580)
res = c.rk_eval_batch(sets)  # warm-up (also validates)
times = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = c.rk_eval_batch(sets)
    times.append(time.perf_counter() - t0)
F = math.factorial(9)
pct = sorted(100.0 * (st.n_eq + st.n_gt) / F for st, _ in res)
q = lambda p: pct[min(len(pct) - 1, int(p * len(pct)))]
print(json.dumps({"config": "C5", "sets": len(sets), "evaluations": len(sets) * F,
                  "seconds": min(times), "evals_per_s": len(sets) * F / min(times),
                  "note": "synchronous rk_eval_batch incl. host validation + table packing, device Algorithm 1 per set, upload, D2H",
                  "heuristic_percentile": {"min": pct[0], "p10": q(0.1), "median": q(0.5), "p90": q(0.9),
                                           "max": pct[-1], "mean": sum(pct) / len(pct),
                                           "frac_ge_90": sum(p >= 90 for p in pct) / len(pct)}}))
