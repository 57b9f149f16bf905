"""Shape of C4's suffix rows (120 keys per run) relative to the 256 Fig. 1
bins: bins spanned per run, distinct keys per run (dev diagnostic for the
memo histogram / counting passes)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_1511_07983_b200 import rk, workloads as W  # noqa: E402

gpu, ks = W.config("C4")
c = rk.Context(0)
c.rk_set_gpu_params(gpu)
c.rk_set_kernels(ks)
N = math.factorial(12)
_, _, idx, key = c.rk_heuristic_order()
cand = torch.tensor([key], dtype=torch.int64, device="cuda")
rec = torch.zeros(8, dtype=torch.int64, device="cuda")
keys = torch.empty(N, dtype=torch.int64, device="cuda")
c.rk_sweep_pass1_async(0, N, cand, rec, keys)
c.rk_sweep_pass2_async(0, N, cand, rec, 0, None, keys, rec)
torch.cuda.synchronize()
kmin, kmax = int(rec[0]), int(rec[1])
D = kmax - kmin
rows = keys.view(-1, 120)
span_bins = torch.zeros(258, dtype=torch.int64, device="cuda")
ndv_hist = torch.zeros(121, dtype=torch.int64, device="cuda")
inside = 0
for s in range(0, rows.shape[0], 1 << 20):
    r = rows[s:s + (1 << 20)]
    mn, mx = r.min(1).values, r.max(1).values
    b0 = torch.clamp(((mn - kmin) * 256) // D, max=255)
    b1 = torch.clamp(((mx - kmin) * 256) // D, max=255)
    span_bins += torch.bincount(b1 - b0, minlength=258)[:258]
    srt = r.sort(1).values
    ndv = 1 + (srt[:, 1:] != srt[:, :-1]).sum(1)
    ndv_hist += torch.bincount(ndv, minlength=121)[:121]
    inside += int(((mn <= key) & (mx >= key)).sum())
sb = span_bins.cpu().tolist()
nh = ndv_hist.cpu().tolist()
runs = rows.shape[0]
print("runs", runs, "bin width", D / 256, "row span (keys) mean",
      float((rows.max(1).values - rows.min(1).values).double().mean()))
print("bins spanned-1 histogram:", {i: v for i, v in enumerate(sb) if v})
print("distinct per row: mean", sum(i * v for i, v in enumerate(nh)) / runs, "max", max(i for i, v in enumerate(nh) if v))
print("rows containing the candidate:", inside, inside / runs)

# how many distinct rows (node, K_closed) among the runs? (a hash of each run's 120 keys)
w = torch.randint(1, 1 << 62, (120,), dtype=torch.int64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
hs = []
for s in range(0, rows.shape[0], 1 << 20):
    r = rows[s:s + (1 << 20)]
    hs.append((r * w).sum(1))
h = torch.cat(hs)
uq, cn = torch.unique(h, return_counts=True)
print("distinct rows (node, K_closed):", int(uq.numel()), "of", rows.shape[0])
cs = torch.sort(cn, descending=True).values
print("multiplicity: max", int(cs[0]), "top10", cs[:10].tolist(), "rows with m>=100:", int((cn >= 100).sum()),
      "runs in them:", int(cn[cn >= 100].sum()))
mins = rows.min(1).values
print("distinct row minima:", int(torch.unique(mins).numel()))
