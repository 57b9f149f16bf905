"""C6 (B200 preset, run-length SM state) full-space sweep timing, and the
run-length state's cost on C4 (RK_FORCE_RUNS=1 in a child process) against
the register-state variant.  One JSON line per measurement."""
import json
import math
import os
import subprocess
import sys

import torch

sys.path.insert(0, ".")
from paper_1511_07983_b200 import rk  # noqa: E402
from paper_1511_07983_b200 import workloads as W  # noqa: E402


def time_sweep(name, reps=5):
    gpu, ks = W.config(name)
    c = rk.Context(0)
    c.rk_set_gpu_params(gpu)
    c.rk_set_kernels(ks)
    N = math.factorial(len(ks))
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    cd = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        c.rk_eval_range_async(0, N, cd, rec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c.rk_eval_range_async(0, N, cd, rec)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    _, _, hidx, _ = c.rk_heuristic_order()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    _, idx, key, nodes = c.rk_best_order(hidx)
    ev[1].record()
    torch.cuda.synchronize()
    return {"config": name, "S_reduced": None, "force_runs": os.environ.get("RK_FORCE_RUNS") == "1",
            "sweep_ms": round(ms, 3), "orders_per_s": N / ms * 1e3, "bnb_ms": round(ev[0].elapsed_time(ev[1]), 3),
            "bnb_nodes": nodes}


def main():
    if len(sys.argv) > 1:
        print(json.dumps(time_sweep(sys.argv[1])), flush=True)
        return
    for name in ("C6", "C4"):
        print(json.dumps(time_sweep(name)), flush=True)
    env = dict(os.environ, RK_FORCE_RUNS="1")
    subprocess.run([sys.executable, __file__, "C4"], env=env, check=True)


if __name__ == "__main__":
    main()
