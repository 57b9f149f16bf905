"""Per-set timing of Sweeper.run on fresh Generator-G 12-kernel sets (bench's fresh_sets e2e)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_07983_b200 import workloads as W
from paper_1511_07983_b200.sweep import Sweeper

gpu, ks = W.config("C4")
sw = Sweeper(gpu, compact_keys=os.environ.get("COMPACT", "0") == "1")
sw.run(ks)
out = []
for rep in range(2):
    for i in range(12):
        kset = W.gen_g(W.SplitMix64(W.SEED_BASE + 0x4000 + i), 12)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sw.run(kset)
        torch.cuda.synchronize()
        t = (time.perf_counter() - t0) * 1e3
        info = sw.ctx.rk_memo_info() if hasattr(sw, "ctx") else None
        out.append({"rep": rep, "set": i, "ms": round(t, 3), "memo_info": list(info) if info else None})
print(json.dumps(out))
