"""Public API: evaluate the whole launch-order space of a kernel set.

``Sweeper(gpu).run(kernels)`` is the call a user makes: host kernel profiles
in, a Table-3-style report out (PAPER:236 columns; Fig. 1 histogram).  Every
step runs in librk's sm_100a kernels; across ranks the index space is sharded
(dist.py).  ``Sweeper.step_device`` is the same path with inputs resident and
no host synchronisation, as timed by bench.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import rk
from .dist import REC_WORDS, all_gather_records, all_reduce, all_reduce_hist, shard_bounds


@dataclass
class Report:
    """SweepReport in exact keys (T = key / rb_den)."""
    n_orders: int
    best_key: int
    best_index: int
    worst_key: int
    worst_index: int
    cand_order: list
    cand_index: int
    cand_key: int
    n_lt: int
    n_eq: int
    n_gt: int
    hist: list
    rb_den: int
    median_key: int | None = None  # lower-middle of the sorted keys
    # Fig. 1 ranking curve: [(rank, key)] at ranks k*N//(p-1), k < p-1, and N-1
    ranking_curve: list | None = None

    @property
    def percentile(self) -> float:  # ties count for the candidate
        return 100.0 * (self.n_eq + self.n_gt) / self.n_orders

    @property
    def speedup_over_worst(self) -> float:  # Table 3: worst / algorithm
        return self.worst_key / self.cand_key

    @property
    def deviation_pct(self) -> float:  # Table 3: (algorithm - optimal) / optimal
        return 100.0 * (self.cand_key - self.best_key) / self.best_key

    @property
    def gain_over_median_pct(self) -> float | None:
        """PAPER:257 "median sequence" comparison: the heuristic order's gain over
        the median order, 100 * (T_median - T_cand) / T_cand (half of the random
        orders are at least this much slower)."""
        if self.median_key is None:
            return None
        return 100.0 * (self.median_key - self.cand_key) / self.cand_key

    def time(self, key: int) -> float:
        return key / self.rb_den


class Sweeper:
    def __init__(self, gpu, device: int | None = None, bins: int = 256, group=None, compact_keys: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("Sweeper needs a CUDA device (no CPU fallback)")
        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.distributed else 1
        self.rank = dist.get_rank(group) if self.distributed else 0
        self.device = torch.cuda.current_device() if device is None else device
        self.dev = torch.device("cuda", self.device)
        self.ctx = rk.Context(self.device)
        self.gpu = tuple(int(x) for x in gpu)
        self.ctx.rk_set_gpu_params(self.gpu)
        self.bins = bins
        self.n = 0
        self.keys = None
        self.keys32 = None
        self.ovf = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # exact keys stored as u32 offsets from the set's exact lower bound: half the key bytes;
        # a key >= base + 2^32 sets the overflow flag and run() repeats the step with u64 keys
        self.compact_keys = compact_keys
        self.rec = torch.zeros(REC_WORDS, dtype=torch.int64, device=self.dev)
        self.glob = torch.zeros(REC_WORDS, dtype=torch.int64, device=self.dev)
        self.cand = torch.zeros(1, dtype=torch.int64, device=self.dev)
        # histogram with a count record appended: one all_reduce for N ranks
        self.hbuf = torch.zeros(bins + REC_WORDS, dtype=torch.int64, device=self.dev)
        self.hist = self.hbuf[:bins]
        self.fin = torch.zeros(REC_WORDS, dtype=torch.int64, device=self.dev)
        self.launches = 0

    def set_kernels(self, kernels):
        self.ctx.rk_set_kernels(kernels)
        self.n = len(kernels)
        self.total = math.factorial(self.n)
        self.first, self.count = shard_bounds(self.total, self.world, self.rank)
        # compact keys (u32 offsets from the exact lower bound) unless a
        # previous pass on this set overflowed; then u64 keys
        self.base = self.ctx.rk_key_lower_bound()
        self.memo = self.ctx.rk_memo_info()[0] and self.bins <= 32768
        self.ovf.zero_()
        if self.compact_keys:
            self.compact = True
            if self.keys32 is None or self.keys32.numel() < self.count:
                self.keys32 = torch.empty(max(1, self.count), dtype=torch.int32, device=self.dev)
            # the u64 buffer a set whose keys overflow the offsets falls back to: allocated up front
            # when modest (<= 8 GB), else on the first overflow
            if (self.keys is None or self.keys.numel() < self.count) and self.count * 8 <= (8 << 30):
                self.keys = torch.empty(max(1, self.count), dtype=torch.int64, device=self.dev)
        else:
            self._use_wide_keys()

    def _use_wide_keys(self):
        self.compact = False
        if self.keys is None or self.keys.numel() < self.count:
            self.keys = torch.empty(max(1, self.count), dtype=torch.int64, device=self.dev)

    def step_device(self, cand_index: int, stream=None, events=None):
        """Enqueue one pass of the hot path; no host sync.  Returns #our launches.
        events (optional dict) receives CUDA event pairs around pass 1 ("eval":
        memo tables + extremes, or the direct evaluation) and pass 2 ("hist":
        counts + histogram + keys, or the histogram of the stored keys).
        Collectives for N ranks: one all_gather of the 64-B
        extremes records (merged on device into the global record, whose
        extremes are the histogram range) and one all_reduce of the histogram
        with the count record appended (int64[bins + 8]); a 2-record device
        merge then gives the final record."""
        c = self.ctx
        L = 0
        c.rk_eval_index_async(cand_index, self.cand, stream)                                  # a5 candidate key
        L += c.launches
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if events is not None else None
        st = torch.cuda.current_stream() if stream is None else stream
        if ev:
            e0, e1 = ev(), ev()
            e0.record(st)
        memo = self.compact and self.memo
        if self.compact and not memo:                                                          # a1-a4 (u32 keys)
            c.rk_eval_range32_async(self.first, self.count, self.cand, self.rec, self.keys32, self.base, self.ovf,
                                    stream)
        else:                                                                                  # a1-a4 pass 1
            c.rk_sweep_pass1_async(self.first, self.count, self.cand, self.rec, None if memo else self.keys, stream)
        L += c.launches
        if ev:
            e1.record(st)
            events.setdefault("eval", []).append((e0, e1))
        multi = self.world > 1
        if multi:                                                                               # a6 combine
            recs = all_gather_records(self.rec, self.group)
            c.rk_merge_stats_async(recs, self.world, self.glob, stream)
            L += c.launches
            rng = self.glob
        else:
            rng = self.rec
        self.hbuf.zero_()
        counts = self.hbuf[self.bins:] if multi else self.rec  # where pass 2 adds the counts
        if ev:
            h0, h1 = ev(), ev()
            h0.record(st)
        if memo:                                                                               # a4 pass 2 (u32 keys)
            c.rk_sweep_pass2_32_async(self.first, self.count, self.cand, rng, self.bins, self.hist, self.keys32,
                                      self.base, self.ovf, counts, stream)
        elif self.compact:                                                                     # a4 histogram
            c.rk_histogram32_async(self.keys32, self.count, self.base, rng, self.bins, self.hist, stream)
        else:                                                                                  # a4 pass 2
            c.rk_sweep_pass2_async(self.first, self.count, self.cand, rng, self.bins, self.hist, self.keys, counts,
                                   stream)
        L += c.launches
        if ev:
            h1.record(st)
            events.setdefault("hist", []).append((h0, h1))
        if multi:
            all_reduce_hist(self.hbuf, self.group)
            both = torch.stack([self.glob, self.hbuf[self.bins:]])
            c.rk_merge_stats_async(both, 2, self.fin, stream)
            L += c.launches
        self.launches = L
        return L

    @property
    def record(self) -> torch.Tensor:
        """The step's final record (device int64[8] = rk_stats)."""
        return self.fin if self.world > 1 else self.rec

    def overflowed(self) -> bool:
        """Did a compact-key pass see a key >= base + 2^32 (on any rank)?"""
        f = self.ovf.clone()
        if self.world > 1:
            all_reduce(f, dist.ReduceOp.MAX, self.group)
        return bool(f.item())

    def heuristic(self):
        order, _, idx, _ = self.ctx.rk_heuristic_order(with_key=False)  # Algorithm 1 on the host
        return order, idx

    def run(self, kernels, median: bool = False, curve_points: int = 0) -> Report:
        """End to end: host profiles in (H2D), report out (D2H).  median=True adds
        the exact median key and the gain over the median order
        (PAPER:257); curve_points = p >= 2 adds the Fig. 1 ranking curve at ranks
        k*N//(p-1) (k < p-1) and N-1 (exact order statistics: a few extra passes
        over the keys)."""
        self.set_kernels(kernels)
        order, idx = self.heuristic()
        self.step_device(idx)
        # one D2H: record, candidate key, histogram and the compact-key overflow flag (with one rank the flag
        # is final; with N ranks the memoised pass decides it from the global range, the direct one per rank)
        out = torch.cat([self.record, self.cand, self.hist, self.ovf.to(torch.int64)]).cpu()
        if self.compact and (self.overflowed() if self.world > 1 else bool(out[-1].item())):
            self._use_wide_keys()  # rare: keys span >= 2^32 above the bound
            self.step_device(idx)
            out = torch.cat([self.record, self.cand, self.hist, self.ovf.to(torch.int64)]).cpu()
        out = out[:-1]
        st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(out[:REC_WORDS].numpy().tobytes()))
        rep = Report(n_orders=self.total, best_key=st.key_min, best_index=st.argmin, worst_key=st.key_max,
                     worst_index=st.argmax, cand_order=order, cand_index=idx,
                     cand_key=int(out[REC_WORDS].item()) & ((1 << 64) - 1), n_lt=st.n_lt, n_eq=st.n_eq,
                     n_gt=st.n_gt, hist=[int(x) for x in out[REC_WORDS + 1:].tolist()], rb_den=self.gpu[6])
        N = self.total
        ranks = []
        if median:
            ranks.append((N - 1) // 2)
        curve = []
        if curve_points >= 2:
            curve = sorted(set([k * N // (curve_points - 1) for k in range(curve_points - 1)] + [N - 1]))
        if ranks or curve:
            got = self.select(ranks + curve, st.key_min, st.key_max)
            if median:
                rep.median_key = got[0]
            if curve:
                rep.ranking_curve = [[r, k] for r, k in zip(curve, got[len(ranks):])]
        return rep

    def select(self, ranks, kmin: int, kmax: int):
        """Exact order statistics over all ranks' keys (after a step)."""
        if self.world == 1:
            if self.compact:
                return self.ctx.rk_select_keys32(self.keys32, self.base, self.count, kmin, kmax, ranks)
            return self.ctx.rk_select_keys(self.keys, self.count, kmin, kmax, ranks)

        def count_fn(lo, span, nb):
            h = torch.zeros(nb, dtype=torch.int64, device=self.dev)
            if self.compact:
                self.ctx.rk_range_histogram32(self.keys32, self.base, self.count, lo, span, nb, h)
            else:
                self.ctx.rk_range_histogram(self.keys, self.count, lo, span, nb, h)
            return h

        from .dist import select_keys_sharded
        return select_keys_sharded(count_fn, kmin, kmax, ranks, group=self.group)

    @property
    def h2d_bytes(self) -> int:
        """Bytes the host sends per run(): the packed kernel tables + params."""
        return rk.rk_table_bytes()

    @property
    def d2h_bytes(self) -> int:
        return 8 * (REC_WORDS + 1 + self.bins + 1)  # record, candidate key, histogram, overflow flag
