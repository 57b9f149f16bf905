"""Thin ctypes binding of librk (include/rk.h) — argument marshalling only.

Every function keeps the C name.  Device buffers are torch tensors on the
ctx's CUDA device (PyTorch is plumbing: memory, streams, process groups);
every step of the hot path runs in librk's sm_100a kernels.  If librk.so is
missing or a CUDA device is absent, compute calls raise — there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RK_LIB", os.path.join(HERE, "librk.so"))

RK_OK, RK_EINVAL, RK_EINFEASIBLE, RK_ETOOMANY, RK_EMISSINGRATIO, RK_EOVERFLOW, RK_ESTATE, RK_ECUDA, \
    RK_ENODEVICE, RK_EUNSUPPORTED = range(10)
STATUS_NAMES = ["RK_OK", "RK_EINVAL", "RK_EINFEASIBLE", "RK_ETOOMANY", "RK_EMISSINGRATIO", "RK_EOVERFLOW",
                "RK_ESTATE", "RK_ECUDA", "RK_ENODEVICE", "RK_EUNSUPPORTED"]

#: every symbol include/rk.h declares (checked by tests/test_abi.py)
EXPORTS = ["rk_create", "rk_destroy", "rk_last_error", "rk_set_gpu_params", "rk_set_kernels", "rk_eval_range",
           "rk_eval_range_async", "rk_eval_range_hist_async", "rk_eval_range32_async", "rk_key_lower_bound", "rk_histogram32_async",
           "rk_eval_index_async", "rk_merge_stats_async", "rk_histogram", "rk_histogram_async",
           "rk_select_keys", "rk_range_histogram", "rk_select_keys32", "rk_range_histogram32", "rk_heuristic_order", "rk_heuristic_batch", "rk_percentile", "rk_eval_batch", "rk_simulate_order", "rk_best_order", "rk_sweep_pass1_async", "rk_sweep_pass2_async", "rk_sweep_pass2_32_async", "rk_set_timing", "rk_timing_read", "rk_memo_info", "rk_memo_audit", "rk_rank", "rk_unrank",
           "rk_last_launch_count", "rk_table_bytes"]


class rk_gpu_params(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint32) for f in
                ("n_sm", "regs_per_sm", "shm_bytes_per_sm", "max_warps_per_sm", "max_blocks_per_sm", "rb_num",
                 "rb_den", "flags")]


RK_FLAG_CURSOR_PER_KERNEL = 1
RK_FLAG_STRICT_RR = 2
RK_FLAG_SKIP_AHEAD = 4
RK_PHASE_NAMES = ("tables", "stream", "hist", "direct", "extremes", "runs")  # RK_PHASE_* of rk.h
RK_N_PHASES = len(RK_PHASE_NAMES)


class rk_kernel(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint32) for f in
                ("grid_blocks", "threads_per_block", "regs_per_thread", "shm_bytes_per_block", "inst_per_block",
                 "mem_per_block")]


class rk_stats(ctypes.Structure):
    _fields_ = [("key_min", ctypes.c_uint64), ("key_max", ctypes.c_uint64), ("argmin", ctypes.c_uint64),
                ("argmax", ctypes.c_uint64), ("n_lt", ctypes.c_uint64), ("n_eq", ctypes.c_uint64),
                ("n_gt", ctypes.c_uint64), ("evaluated", ctypes.c_uint64)]

    def as_tuple(self):
        return (self.key_min, self.key_max, self.argmin, self.argmax, self.n_lt, self.n_eq, self.n_gt,
                self.evaluated)


assert ctypes.sizeof(rk_stats) == 64
STATS_BYTES = 64

_lib = None


def lib():
    """Load librk.so (built by paper_1511_07983_b200.build); raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"librk.so not built ({LIB_PATH}); run __graft_entry__.build() — no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
        sig = {
            "rk_create": ([P(vp), ctypes.c_int], ctypes.c_int),
            "rk_destroy": ([vp], None),
            "rk_last_error": ([vp], ctypes.c_char_p),
            "rk_last_launch_count": ([vp], u32),
            "rk_set_gpu_params": ([vp, P(rk_gpu_params)], ctypes.c_int),
            "rk_set_kernels": ([vp, P(rk_kernel), u32], ctypes.c_int),
            "rk_eval_range": ([vp, u64, u64, u64, P(rk_stats), vp, vp], ctypes.c_int),
            "rk_eval_range_async": ([vp, u64, u64, vp, vp, vp, vp], ctypes.c_int),
            "rk_eval_index_async": ([vp, u64, vp, vp], ctypes.c_int),
            "rk_eval_range_hist_async": ([vp, u64, u64, vp, vp, vp, u32, vp, vp], ctypes.c_int),
            "rk_eval_range32_async": ([vp, u64, u64, vp, vp, vp, u64, vp, vp], ctypes.c_int),
            "rk_key_lower_bound": ([vp, P(u64)], ctypes.c_int),
            "rk_histogram32_async": ([vp, vp, u64, u64, vp, u32, vp, vp], ctypes.c_int),
            "rk_table_bytes": ([], u32),
            "rk_merge_stats_async": ([vp, vp, u32, vp, vp], ctypes.c_int),
            "rk_histogram": ([vp, vp, u64, u64, u64, u32, vp, vp], ctypes.c_int),
            "rk_histogram_async": ([vp, vp, u64, vp, u32, vp, vp], ctypes.c_int),
            "rk_select_keys": ([vp, vp, u64, u64, u64, P(u64), u32, P(u64), vp], ctypes.c_int),
            "rk_range_histogram": ([vp, vp, u64, u64, u64, u32, vp, vp], ctypes.c_int),
            "rk_select_keys32": ([vp, vp, u64, u64, u64, u64, P(u64), u32, P(u64), vp], ctypes.c_int),
            "rk_range_histogram32": ([vp, vp, u64, u64, u64, u64, u32, vp, vp], ctypes.c_int),
            "rk_heuristic_order": ([vp, P(ctypes.c_int32), P(ctypes.c_int32), P(u64), P(u64)], ctypes.c_int),
            "rk_sweep_pass1_async": ([vp, u64, u64, vp, vp, vp, vp], ctypes.c_int),
            "rk_sweep_pass2_async": ([vp, u64, u64, vp, vp, u32, vp, vp, vp, vp], ctypes.c_int),
            "rk_sweep_pass2_32_async": ([vp, u64, u64, vp, vp, u32, vp, vp, u64, vp, vp, vp], ctypes.c_int),
            "rk_memo_info": ([vp, P(u32), P(u32), P(u32), u32], ctypes.c_int),
            "rk_memo_audit": ([vp, P(u64)], ctypes.c_int),
            "rk_set_timing": ([vp, ctypes.c_int], ctypes.c_int),
            "rk_timing_read": ([vp, P(ctypes.c_double), P(u32), u32], ctypes.c_int),
            "rk_best_order": ([vp, u64, P(ctypes.c_int32), P(u64), P(u64), P(u64), vp], ctypes.c_int),
            "rk_heuristic_batch": ([vp, P(rk_kernel), u32, u32, P(ctypes.c_int32), P(u64), vp], ctypes.c_int),
            "rk_percentile": ([vp, P(ctypes.c_int32), u64, u64, P(u64), P(u64)], ctypes.c_int),
            "rk_eval_batch": ([vp, P(rk_kernel), u32, u32, P(u64), P(rk_stats), P(u64), vp], ctypes.c_int),
            "rk_simulate_order": ([vp, P(ctypes.c_int32), P(u32), u32, P(u32), P(u64)], ctypes.c_int),
            "rk_rank": ([P(ctypes.c_int32), u32, P(u64)], ctypes.c_int),
            "rk_unrank": ([u64, u32, P(ctypes.c_int32)], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


class RkError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")
        self.status = status


def _ptr(t):
    """Raw pointer of a torch tensor / None."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)  # torch.cuda.Stream


class _KArr:
    """Contiguous rk_kernel array backed by numpy (keeps the buffer alive)."""

    def __init__(self, kernels):
        import numpy as np

        from itertools import chain

        if isinstance(kernels, np.ndarray):  # (..., 6) integer array: no per-field Python iteration
            a = kernels.reshape(-1, 6).astype(np.uint64) if kernels.size else np.zeros((1, 6), np.uint64)
        else:
            a = (np.fromiter(chain.from_iterable(kernels), dtype=np.uint64, count=6 * len(kernels)).reshape(-1, 6)
                 if len(kernels) else np.zeros((1, 6), np.uint64))
        if a.size and (a.max() > 0xFFFFFFFF):
            raise RkError(RK_EINVAL, "kernel field exceeds u32")
        self.buf = np.ascontiguousarray(a.astype(np.uint32))
        self._as_parameter_ = self.buf.ctypes.data_as(ctypes.POINTER(rk_kernel))


def kernels_array(kernels):
    return _KArr(kernels)


def rk_table_bytes() -> int:
    return int(lib().rk_table_bytes())


def rk_rank(order) -> int:
    o = (ctypes.c_int32 * len(order))(*order)
    v = ctypes.c_uint64()
    s = lib().rk_rank(o, len(order), ctypes.byref(v))
    if s:
        raise RkError(s, "rk_rank")
    return v.value


def rk_unrank(idx: int, n: int) -> list:
    o = (ctypes.c_int32 * n)()
    s = lib().rk_unrank(idx, n, o)
    if s:
        raise RkError(s, "rk_unrank")
    return list(o)


@dataclass
class Stats:
    key_min: int
    key_max: int
    argmin: int
    argmax: int
    n_lt: int
    n_eq: int
    n_gt: int
    evaluated: int

    @classmethod
    def from_c(cls, c: rk_stats):
        return cls(*c.as_tuple())

    def as_tuple(self):
        return (self.key_min, self.key_max, self.argmin, self.argmax, self.n_lt, self.n_eq, self.n_gt,
                self.evaluated)


class Context:
    """Owns an rk_ctx.  ``device=-1`` gives a host-only ctx (validation and
    Algorithm 1 only; every model evaluation raises RK_ENODEVICE)."""

    def __init__(self, device: int = 0):
        self._L = lib()
        h = ctypes.c_void_p()
        s = self._L.rk_create(ctypes.byref(h), device)
        if s:
            raise RkError(s, f"rk_create(device={device})")
        self.h = h
        self.device = device
        self.n = 0

    def close(self):
        if getattr(self, "h", None):
            self._L.rk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, s, what):
        if s:
            raise RkError(s, f"{what}: {self._L.rk_last_error(self.h).decode()}")

    @property
    def launches(self) -> int:
        return int(self._L.rk_last_launch_count(self.h))

    # -- inputs --------------------------------------------------------------
    def rk_set_gpu_params(self, gpu):
        g = [int(x) for x in gpu]
        p = rk_gpu_params(*(g + [0] * (8 - len(g))))  # 7-tuple (Table 1) or 8 with model flags
        self._chk(self._L.rk_set_gpu_params(self.h, ctypes.byref(p)), "rk_set_gpu_params")

    def rk_set_kernels(self, kernels):
        arr = kernels_array(kernels)
        self._chk(self._L.rk_set_kernels(self.h, arr, len(kernels)), "rk_set_kernels")
        self.n = len(kernels)

    # -- evaluation ----------------------------------------------------------
    def rk_eval_range(self, first: int, count: int, candidate_key: int = 0, keys_dev=None, stream=None) -> Stats:
        out = rk_stats()
        self._chk(self._L.rk_eval_range(self.h, first, count, candidate_key, ctypes.byref(out), _ptr(keys_dev),
                                        _stream(stream)), "rk_eval_range")
        return Stats.from_c(out)

    def rk_eval_range_async(self, first: int, count: int, cand_key_dev, stats_dev, keys_dev=None, stream=None):
        self._chk(self._L.rk_eval_range_async(self.h, first, count, _ptr(cand_key_dev), _ptr(stats_dev),
                                              _ptr(keys_dev), _stream(stream)), "rk_eval_range_async")

    def rk_eval_range_hist_async(self, first: int, count: int, cand_key_dev, stats_dev, range_dev, bins: int,
                                 hist_dev, stream=None):
        self._chk(self._L.rk_eval_range_hist_async(self.h, first, count, _ptr(cand_key_dev), _ptr(stats_dev),
                                                   _ptr(range_dev), bins, _ptr(hist_dev), _stream(stream)),
                  "rk_eval_range_hist_async")

    def rk_eval_range32_async(self, first: int, count: int, cand_key_dev, stats_dev, keys32_dev, key_base: int,
                              ovf_dev, stream=None):
        self._chk(self._L.rk_eval_range32_async(self.h, first, count, _ptr(cand_key_dev), _ptr(stats_dev),
                                                _ptr(keys32_dev), key_base, _ptr(ovf_dev), _stream(stream)),
                  "rk_eval_range32_async")

    def rk_key_lower_bound(self) -> int:
        v = ctypes.c_uint64()
        self._chk(self._L.rk_key_lower_bound(self.h, ctypes.byref(v)), "rk_key_lower_bound")
        return v.value

    def rk_histogram32_async(self, keys32_dev, count: int, key_base: int, range_dev, bins: int, hist_dev,
                             stream=None):
        self._chk(self._L.rk_histogram32_async(self.h, _ptr(keys32_dev), count, key_base, _ptr(range_dev), bins,
                                               _ptr(hist_dev), _stream(stream)), "rk_histogram32_async")

    def rk_eval_index_async(self, index: int, key_dev, stream=None):
        self._chk(self._L.rk_eval_index_async(self.h, index, _ptr(key_dev), _stream(stream)), "rk_eval_index_async")

    def rk_merge_stats_async(self, in_dev, n_records: int, out_dev, stream=None):
        self._chk(self._L.rk_merge_stats_async(self.h, _ptr(in_dev), n_records, _ptr(out_dev), _stream(stream)),
                  "rk_merge_stats_async")

    def rk_histogram(self, keys_dev, count: int, kmin: int, kmax: int, bins: int, hist_dev, stream=None):
        self._chk(self._L.rk_histogram(self.h, _ptr(keys_dev), count, kmin, kmax, bins, _ptr(hist_dev),
                                       _stream(stream)), "rk_histogram")

    def rk_histogram_async(self, keys_dev, count: int, range_dev, bins: int, hist_dev, stream=None):
        self._chk(self._L.rk_histogram_async(self.h, _ptr(keys_dev), count, _ptr(range_dev), bins, _ptr(hist_dev),
                                             _stream(stream)), "rk_histogram_async")

    def rk_select_keys(self, keys_dev, count: int, kmin: int, kmax: int, ranks, stream=None):
        m = len(ranks)
        r = (ctypes.c_uint64 * max(1, m))(*ranks)
        out = (ctypes.c_uint64 * max(1, m))()
        self._chk(self._L.rk_select_keys(self.h, _ptr(keys_dev), count, kmin, kmax, r, m, out, _stream(stream)),
                  "rk_select_keys")
        return list(out)[:m]

    def rk_range_histogram(self, keys_dev, count: int, lo: int, span: int, bins: int, hist_dev, stream=None):
        self._chk(self._L.rk_range_histogram(self.h, _ptr(keys_dev), count, lo, span, bins, _ptr(hist_dev),
                                             _stream(stream)), "rk_range_histogram")

    def rk_select_keys32(self, keys32_dev, key_base: int, count: int, kmin: int, kmax: int, ranks, stream=None):
        m = len(ranks)
        r = (ctypes.c_uint64 * max(1, m))(*ranks)
        out = (ctypes.c_uint64 * max(1, m))()
        self._chk(self._L.rk_select_keys32(self.h, _ptr(keys32_dev), key_base, count, kmin, kmax, r, m, out,
                                           _stream(stream)), "rk_select_keys32")
        return list(out)[:m]

    def rk_range_histogram32(self, keys32_dev, key_base: int, count: int, lo: int, span: int, bins: int, hist_dev,
                             stream=None):
        self._chk(self._L.rk_range_histogram32(self.h, _ptr(keys32_dev), key_base, count, lo, span, bins,
                                               _ptr(hist_dev), _stream(stream)), "rk_range_histogram32")

    def rk_heuristic_order(self, with_key: bool = True):
        """Algorithm 1 -> (order, round_of, index, key-or-None)."""
        n = self.n
        o = (ctypes.c_int32 * n)()
        r = (ctypes.c_int32 * n)()
        idx = ctypes.c_uint64()
        key = ctypes.c_uint64()
        self._chk(self._L.rk_heuristic_order(self.h, o, r, ctypes.byref(idx), ctypes.byref(key) if with_key else None),
                  "rk_heuristic_order")
        return list(o), list(r), idx.value, (key.value if with_key else None)

    def rk_sweep_pass1_async(self, first: int, count: int, cand_key_dev, rec_dev, keys_dev=None, stream=None):
        self._chk(self._L.rk_sweep_pass1_async(self.h, first, count, _ptr(cand_key_dev), _ptr(rec_dev),
                                               _ptr(keys_dev), _stream(stream)), "rk_sweep_pass1_async")

    def rk_sweep_pass2_async(self, first: int, count: int, cand_key_dev, range_dev, bins: int, hist_dev, keys_dev,
                             rec_dev, stream=None):
        self._chk(self._L.rk_sweep_pass2_async(self.h, first, count, _ptr(cand_key_dev), _ptr(range_dev), bins,
                                               _ptr(hist_dev), _ptr(keys_dev), _ptr(rec_dev), _stream(stream)),
                  "rk_sweep_pass2_async")

    def rk_sweep_pass2_32_async(self, first: int, count: int, cand_key_dev, range_dev, bins: int, hist_dev,
                                keys32_dev, key_base: int, ovf_dev, rec_dev, stream=None):
        self._chk(self._L.rk_sweep_pass2_32_async(self.h, first, count, _ptr(cand_key_dev), _ptr(range_dev), bins,
                                                  _ptr(hist_dev), _ptr(keys32_dev), key_base, _ptr(ovf_dev),
                                                  _ptr(rec_dev), _stream(stream)), "rk_sweep_pass2_32_async")

    def rk_set_timing(self, on: bool = True):
        self._chk(self._L.rk_set_timing(self.h, 1 if on else 0), "rk_set_timing")

    def rk_timing_read(self):
        """-> {phase: (summed ms, marks)} since the last read (RK_PHASE_* names)."""
        ms = (ctypes.c_double * RK_N_PHASES)()
        cnt = (ctypes.c_uint32 * RK_N_PHASES)()
        self._chk(self._L.rk_timing_read(self.h, ms, cnt, RK_N_PHASES), "rk_timing_read")
        return {name: (ms[i], cnt[i]) for i, name in enumerate(RK_PHASE_NAMES)}

    def rk_memo_info(self):
        """-> (on, P, [distinct nodes per level 0..P])"""
        on, lv = ctypes.c_uint32(), ctypes.c_uint32()
        nodes = (ctypes.c_uint32 * 17)()
        self._chk(self._L.rk_memo_info(self.h, ctypes.byref(on), ctypes.byref(lv), nodes, 17), "rk_memo_info")
        return bool(on.value), lv.value, list(nodes)[:lv.value + 1] if on.value else []

    def rk_memo_audit(self):
        """-> 8 counters of the race audit of the last pass 1's memo tables (rk.h)."""
        out = (ctypes.c_uint64 * 8)()
        self._chk(self._L.rk_memo_audit(self.h, out), "rk_memo_audit")
        return list(out)

    def rk_best_order(self, seed_index=None, stream=None):
        """Exact optimum by branch and bound -> (order, index, key, nodes);
        seed_index None = unseeded bound."""
        n = self.n
        o = (ctypes.c_int32 * n)()
        idx, key, nodes = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        seed = (1 << 64) - 1 if seed_index is None else int(seed_index)
        self._chk(self._L.rk_best_order(self.h, seed, o, ctypes.byref(idx), ctypes.byref(key), ctypes.byref(nodes),
                                        _stream(stream)), "rk_best_order")
        return list(o), idx.value, key.value, nodes.value

    def rk_heuristic_batch(self, sets, stream=None):
        """Algorithm 1 on the device for many sets -> (orders, indices).  sets: a list of
        kernel lists, or an integer array of shape (n_sets, n, 6)."""
        n = len(sets[0])
        arr = kernels_array(sets if hasattr(sets, "shape") else [k for s in sets for k in s])
        ns = len(sets)
        orders = (ctypes.c_int32 * (ns * n))()
        idx = (ctypes.c_uint64 * ns)()
        self._chk(self._L.rk_heuristic_batch(self.h, arr, n, ns, orders, idx, _stream(stream)), "rk_heuristic_batch")
        return [list(orders[q * n:(q + 1) * n]) for q in range(ns)], list(idx)

    def rk_percentile(self, order, first: int, count: int):
        o = (ctypes.c_int32 * len(order))(*order)
        nge = ctypes.c_uint64()
        key = ctypes.c_uint64()
        self._chk(self._L.rk_percentile(self.h, o, first, count, ctypes.byref(nge), ctypes.byref(key)),
                  "rk_percentile")
        return nge.value, key.value

    def rk_eval_batch(self, sets, cand_index=None, stream=None):
        """-> list of (Stats, cand_key) per set.  sets: a list of kernel lists, or an
        integer array of shape (n_sets, n, 6)."""
        n = len(sets[0])
        arr = kernels_array(sets if hasattr(sets, "shape") else [k for s in sets for k in s])
        ns = len(sets)
        out = (rk_stats * ns)()
        keys = (ctypes.c_uint64 * ns)()
        ci = (ctypes.c_uint64 * ns)(*cand_index) if cand_index is not None else None
        self._chk(self._L.rk_eval_batch(self.h, arr, n, ns, ci, out, keys, _stream(stream)), "rk_eval_batch")
        import numpy as np
        rows = np.frombuffer(out, dtype=np.uint64).reshape(ns, 8).tolist()  # field order of rk_stats
        return [(Stats(*r), k) for r, k in zip(rows, keys)]

    def rk_simulate_order(self, order, max_rounds: int = 4096):
        n = len(order)
        o = (ctypes.c_int32 * n)(*order)
        rounds = (ctypes.c_uint32 * (max_rounds * n))()
        nr = ctypes.c_uint32()
        key = ctypes.c_uint64()
        self._chk(self._L.rk_simulate_order(self.h, o, rounds, max_rounds, ctypes.byref(nr), ctypes.byref(key)),
                  "rk_simulate_order")
        R = nr.value
        return [[rounds[r * n + i] for i in range(n)] for r in range(R)], key.value
