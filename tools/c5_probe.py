"""C5 batch timing breakdown: rk_eval_batch memoised vs direct (RK_NO_MEMO=1),
with Algorithm 1 on device (default) and with given candidate indices."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_07983_b200 import rk, workloads as W

import numpy as np
sets = np.array(W.c5_sets(4096), dtype=np.int64)  # (sets, 9, 6), host-resident
os.environ["RK_NO_MEMO"] = "1"
cd = rk.Context(0)
del os.environ["RK_NO_MEMO"]
cm = rk.Context(0)
out = {}
for name, c in (("memo", cm), ("direct", cd)):
    c.rk_set_gpu_params(W.GTX580)
    res = c.rk_eval_batch(sets)
    idx = [0] * len(sets)
    for label, kw in (("alg1_on_device", {}), ("given_candidates", {"cand_index": idx})):
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c.rk_eval_batch(sets, **kw)
            ts.append(time.perf_counter() - t0)
        out[f"{name}_{label}_ms"] = round(min(ts) * 1e3, 3)
    out[f"{name}_launches"] = c.launches
print(json.dumps(out))
