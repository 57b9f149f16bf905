"""Write the large-config oracle goldens (calls ONLY oracle/ + the input generator).

    python tests/golden/make_goldens.py C2 C3 C4 C5 [--threads N] [--c5-sets 256]

For each config: Algorithm 1's order (oracle's own implementation), its index and
exact key, the full-space statistics (min/argmin, max/argmax, counts vs the
candidate) and the B=256 histogram.  C5: per-set statistics for
the first --c5-sets sets.  The outputs are committed under tests/golden/ and
compared bit-exactly with the CUDA path by tests/test_gpu_parity.py.
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_1511_07983_b200 import workloads as W  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def one_config(name, threads, bins=256):
    gpu, ks = W.config(name)
    order, _ = O.heuristic(gpu, ks)
    cand_idx = O.rank(order)
    cand_key = O.simulate(gpu, ks, order).key
    t0 = time.time()
    s, keys = O.sweep(gpu, ks, cand_key=cand_key, threads=threads, keys=True)
    dt = time.time() - t0
    hist = O.histogram(keys, s.key_min, s.key_max, bins)
    # order statistics (SPEC:302 median = lower-middle; Fig. 1 ranking points):
    # a library sort of the oracle's keys
    import numpy as np
    N = len(keys)
    ranks = sorted({0, N - 1, (N - 1) // 2} | {N * q // 10 for q in range(1, 10)})
    srt = np.sort(keys)
    order_stats = {str(r): int(srt[r]) for r in ranks}
    del srt
    return {
        "_source": f"oracle/rk_oracle.cpp via tests/golden/make_goldens.py ({threads} threads, {dt:.1f} s, "
                   f"{platform.processor() or platform.machine()})",
        "config": name, "gpu": list(gpu), "kernels": [list(k) for k in ks],
        "cand_order": order, "cand_index": cand_idx, "cand_key": cand_key,
        "stats": {"key_min": s.key_min, "key_max": s.key_max, "argmin": s.argmin, "argmax": s.argmax,
                  "n_lt": s.n_lt, "n_eq": s.n_eq, "n_gt": s.n_gt, "evaluated": s.evaluated},
        "max_rel_err_naive_double": s.max_rel_err,
        "bins": bins, "hist": hist,
        "median_rank": (N - 1) // 2, "order_stats": order_stats,
    }


def c5(threads, n_sets):
    sets = W.c5_sets(n_sets)
    gpu = W.GTX580
    t0 = time.time()
    res = O.sweep_sets(gpu, sets, threads=threads)
    dt = time.time() - t0
    return {
        "_source": f"oracle/rk_oracle.cpp via tests/golden/make_goldens.py ({threads} threads, {dt:.1f} s); " +
                   (f"first {n_sets} of the 4096 C5 sets (labelled subset)" if n_sets < 4096 else "all 4096 C5 sets"),
        "config": "C5", "n_sets": n_sets, "n": 9, "gpu": list(gpu),
        "sets": [{"stats": list(st.as_tuple()), "cand_index": ci, "cand_key": ck} for st, ci, ck in res],
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--c5-sets", type=int, default=256)
    a = ap.parse_args()
    for c in a.configs:
        out = c5(a.threads, a.c5_sets) if c == "C5" else one_config(c, a.threads)
        fn = os.path.join(HERE, f"{c.lower()}_oracle.json")
        with open(fn, "w") as f:
            json.dump(out, f, indent=1)
        print("wrote", fn, out.get("_source"))


if __name__ == "__main__":
    main()
