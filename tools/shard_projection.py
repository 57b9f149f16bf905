"""Strong-scaling projection of the memoised C4 step from one GPU (
VERDICT r01 item 4): for G in {1, 2, 4, 8}, run rank g's shard of the step
ALONE on this GPU (exactly the per-rank device work of a G-rank run: pass 1 on
the shard, pass 2 on the shard, the candidate key) and time it with CUDA
events; the slowest shard bounds the G-rank step.  Collectives are not
included (one GPU): the projection adds `--coll-us` per collective, 2 per step.
Prints one JSON line per G and a summary (profiles/r02_shard_projection.json)."""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1511_07983_b200 import workloads as W  # noqa: E402
from paper_1511_07983_b200.dist import shard_bounds  # noqa: E402
from paper_1511_07983_b200.sweep import Sweeper  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=0, help="a Generator-G set of n kernels (seed SEED_BASE + 1000 n) instead")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--gs", default="1,2,4,8")
ap.add_argument("--coll-us", type=float, default=15.0)
args = ap.parse_args()
if args.n:
    gpu, ks = W.GTX580, W.gen_g(W.SplitMix64(W.SEED_BASE + 1000 * args.n), args.n)
    args.config = f"G{args.n}"
else:
    gpu, ks = W.config(args.config)
N = math.factorial(len(ks))
sw = Sweeper(gpu, device=0, compact_keys=True)
sw.set_kernels(ks)
_, idx = sw.heuristic()
stream = torch.cuda.current_stream()
res = {}
for G in [int(x) for x in args.gs.split(",")]:
    per = []
    for g in range(G):
        sw.first, sw.count = shard_bounds(N, G, g)
        for _ in range(3):
            sw.step_device(idx, stream)
        torch.cuda.synchronize()
        sw.ctx.rk_set_timing(True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.reps):
            sw.step_device(idx, stream)
        b.record(stream)
        torch.cuda.synchronize()
        ph = sw.ctx.rk_timing_read()
        sw.ctx.rk_set_timing(False)
        per.append({"shard": g, "first": sw.first, "count": sw.count, "ms": a.elapsed_time(b) / args.reps,
                    **{k: v[0] / v[1] for k, v in ph.items() if v[1]}})
    worst = max(per, key=lambda x: x["ms"])
    res[G] = {"max_shard_ms": worst["ms"], "worst_shard": worst, "shards": per}
T1 = res[1]["max_shard_ms"]
summary = {}
for G, r in res.items():
    tG = r["max_shard_ms"] + (2 * args.coll_us / 1e3 if G > 1 else 0.0)
    summary[G] = {"per_rank_ms": r["max_shard_ms"], "projected_step_ms": tG, "projected_eff": T1 / (G * tG),
                  "tables_ms": r["worst_shard"].get("tables"), "extremes_ms": r["worst_shard"].get("extremes"),
                  "stream_ms": r["worst_shard"].get("stream"), "hist_ms": r["worst_shard"].get("hist")}
print(json.dumps({"config": args.config, "orders": N, "collective_us_assumed": args.coll_us, "summary": summary,
                  "detail": res}))
