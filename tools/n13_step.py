"""One memoised 13! step (compact keys) for ncu launch lists: a Generator-G set of
13 kernels (seed SEED_BASE + 13000), 3 steps."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1511_07983_b200 import workloads as W  # noqa: E402
from paper_1511_07983_b200.sweep import Sweeper  # noqa: E402

ks = W.gen_g(W.SplitMix64(W.SEED_BASE + 13000), 13)
sw = Sweeper(W.GTX580, device=0, compact_keys=True)
sw.set_kernels(ks)
_, idx = sw.heuristic()
print("memo", sw.ctx.rk_memo_info())
for _ in range(3):
    sw.step_device(idx)
torch.cuda.synchronize()
