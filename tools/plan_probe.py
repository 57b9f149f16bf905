"""Cost of rk_set_kernels on C4 (validation, table packing, H2D, the one-sync memo
plan) and of the other per-call pieces of Sweeper.run."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1511_07983_b200 import workloads as W  # noqa: E402
from paper_1511_07983_b200.sweep import Sweeper  # noqa: E402

gpu, ks = W.config("C4")
sw = Sweeper(gpu, device=0, compact_keys=True)
for _ in range(3):
    sw.run(ks)
torch.cuda.synchronize()
out = {}
R = 20
t0 = time.perf_counter()
for _ in range(R):
    sw.ctx.rk_set_kernels(ks)
torch.cuda.synchronize()
out["rk_set_kernels_ms"] = (time.perf_counter() - t0) / R * 1e3
t0 = time.perf_counter()
for _ in range(R):
    sw.heuristic()
out["heuristic_ms"] = (time.perf_counter() - t0) / R * 1e3
sw.set_kernels(ks)
_, idx = sw.heuristic()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(R):
    sw.step_device(idx)
torch.cuda.synchronize()
out["step_device_wall_ms"] = (time.perf_counter() - t0) / R * 1e3
t0 = time.perf_counter()
for _ in range(R):
    sw.run(ks)
out["run_wall_ms"] = (time.perf_counter() - t0) / R * 1e3
print(json.dumps(out))
