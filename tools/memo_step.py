"""One C4 step of the memoised path (for ncu): cand key, pass 1, pass 2, three times."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1511_07983_b200 import sweep, workloads as W  # noqa: E402

gpu, ks = W.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
sw = sweep.Sweeper(gpu, 0)
sw.set_kernels(ks)
_, idx = sw.heuristic()
print("memo", sw.ctx.rk_memo_info())
for _ in range(3):
    sw.step_device(idx)
torch.cuda.synchronize()
ev = {}
for _ in range(5):
    sw.step_device(idx, events=ev)
torch.cuda.synchronize()
for k, v in ev.items():
    print(k, sum(a.elapsed_time(b) for a, b in v) / len(v), "ms")
