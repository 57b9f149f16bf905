"""Full-space statistics (no keys stored) for generator sets with n = 13..15:
memoised path vs the plan state, timed with CUDA events; one JSON line each."""
import json
import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1511_07983_b200 import rk, workloads as W  # noqa: E402

c = rk.Context(0)
for n in [int(x) for x in sys.argv[1:]] or [13, 14]:
    ks = W.gen_g(W.SplitMix64(W.SEED_BASE + 1000 * n), n)
    c.rk_set_gpu_params(W.GTX580)
    t0 = time.perf_counter()
    c.rk_set_kernels(ks)
    plan_s = time.perf_counter() - t0
    on, P, nodes = c.rk_memo_info()
    N = math.factorial(n)
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    cd = torch.zeros(1, dtype=torch.int64, device="cuda")
    c.rk_eval_range_async(0, N, cd, rec)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    c.rk_eval_range_async(0, N, cd, rec)
    b.record()
    torch.cuda.synchronize()
    st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
    _, idx, key, _ = c.rk_best_order(c.rk_heuristic_order()[2])
    print(json.dumps({"n": n, "orders": N, "memo": on, "levels": P, "nodes_last": nodes[-1] if nodes else None,
                      "plan_s": round(plan_s, 3), "sweep_ms": round(a.elapsed_time(b), 2),
                      "orders_per_s": N / (a.elapsed_time(b) / 1e3), "key_min": st.key_min, "argmin": st.argmin,
                      "evaluated": st.evaluated, "bnb_agrees": (key, idx) == (st.key_min, st.argmin)}), flush=True)
