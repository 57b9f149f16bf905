"""quality of Algorithm 1 at batch scale under the model.

For S random kernel sets (generator G, n kernels), run Algorithm 1 on the GPU
for every set, evaluate each set's full n! space, and report the distribution
of the heuristic order's percentile rank (ties count for the candidate,
SPEC:325) next to the paper's "well above the 90 percentile mark".

    python tools/heuristic_quality.py [--sets 100000] [--n 9]
"""
import argparse, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1511_07983_b200 import rk, workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--sets", type=int, default=100000)
ap.add_argument("--n", type=int, default=9)
ap.add_argument("--seed", type=int, default=0xF4)
ap.add_argument("--chunk", type=int, default=8192)
a = ap.parse_args()
t0 = time.time()
rng = W.SplitMix64(W.SEED_BASE + a.seed)
sets = [W.gen_g(rng, a.n) for _ in range(a.sets)]
tgen = time.time() - t0
c = rk.Context(0)
c.rk_set_gpu_params(W.GTX580)
F = math.factorial(a.n)
pct, dev, spd = [], [], []
t0 = time.time()
for i in range(0, a.sets, a.chunk):
    for st, ck in c.rk_eval_batch(sets[i:i + a.chunk]):  # Algorithm 1 on the device + full space per set
        pct.append(100.0 * (st.n_eq + st.n_gt) / F)
        dev.append(100.0 * (ck - st.key_min) / st.key_min)
        spd.append(st.key_max / ck)
dt = time.time() - t0
pct = np.array(pct)
print(json.dumps({
    "sets": a.sets, "n": a.n, "orders_evaluated": a.sets * F, "seconds": dt, "evals_per_s": a.sets * F / dt,
    "generation_seconds_host": tgen,
    "percentile": {"mean": float(pct.mean()), "median": float(np.median(pct)), "p10": float(np.percentile(pct, 10)),
                   "p90": float(np.percentile(pct, 90)), "frac_ge_90": float((pct >= 90).mean()),
                   "frac_eq_100": float((pct >= 100).mean())},
    "deviation_from_optimal_pct": {"mean": float(np.mean(dev)), "median": float(np.median(dev))},
    "speedup_over_worst": {"mean": float(np.mean(spd)), "median": float(np.median(spd))},
}))
