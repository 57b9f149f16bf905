"""Where the C5 call's host time goes: array marshalling, record conversion, and the C call."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1511_07983_b200 import rk, workloads as W

sets = np.array(W.c5_sets(4096), dtype=np.int64)
c = rk.Context(0)
c.rk_set_gpu_params(W.GTX580)
c.rk_eval_batch(sets)
best = {}
def t(name, f, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t0) * 1e3)
    best[name] = round(min(ts), 3)
t("marshal_ms", lambda: rk.kernels_array(sets))
out = (rk.rk_stats * 4096)()
t("records_ms", lambda: [rk.Stats(*r) for r in np.frombuffer(out, dtype=np.uint64).reshape(4096, 8).tolist()])
t("call_total_ms", lambda: c.rk_eval_batch(sets))
idx = [0] * 4096
t("call_given_cand_ms", lambda: c.rk_eval_batch(sets, cand_index=idx))
t("heuristic_batch_ms", lambda: c.rk_heuristic_batch(sets) if hasattr(c, "rk_heuristic_batch") else None)
print(json.dumps(best))
