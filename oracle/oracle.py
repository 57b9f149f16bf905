"""ctypes wrapper of ``oracle/rk_oracle.cpp`` — TEST INFRASTRUCTURE ONLY.

Inputs are plain sequences so this module imports nothing from the product
package:

* ``gpu``     = (n_sm, regs_per_sm, shm_per_sm, warps_per_sm, blocks_per_sm, rb_num, rb_den[, flags])
* ``kernels`` = [(grid_blocks, threads_per_block, regs_per_thread, shm_per_block,
                  inst_per_block A_i, mem_per_block M_i), ...]

(Table 1; GTX580 values PAPER:254; R_B = rb_num/rb_den.)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rk_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_EINVAL, OR_EINFEASIBLE, OR_ETOOMANY, OR_EMISSINGRATIO, OR_EOVERFLOW = range(6)


def build(force: bool = False) -> str:
    """Compile the oracle with plain g++ (no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["g++", "-std=c++17", "-O2", "-g", "-shared", "-fPIC", "-pthread", "-o", _LIB + ".tmp", _SRC]
        )
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        dp = ctypes.POINTER(ctypes.c_double)
        L.or_check_inputs.argtypes = [u32p, u32p, ctypes.c_int]
        L.or_unrank.argtypes = [ctypes.c_uint64, ctypes.c_int, i32p]
        L.or_unrank.restype = None
        L.or_rank.argtypes = [i32p, ctypes.c_int]
        L.or_rank.restype = ctypes.c_uint64
        L.or_factorial.argtypes = [ctypes.c_int]
        L.or_factorial.restype = ctypes.c_uint64
        L.or_simulate.argtypes = [u32p, u32p, ctypes.c_int, i32p, u32p, ctypes.c_int, i32p, u64p, u64p, dp, i32p]
        L.or_sweep.argtypes = [u32p, u32p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                               ctypes.c_int, u64p, u64p, dp]
        L.or_histogram.argtypes = [u64p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, u64p]
        L.or_heuristic.argtypes = [u32p, u32p, ctypes.c_int, i32p, i32p]
        L.or_pair_score.argtypes = [u32p, u32p, ctypes.c_int, ctypes.c_int, i32p, dp, dp]
        L.or_keys_of.argtypes = [u32p, u32p, ctypes.c_int, u64p, ctypes.c_uint64, ctypes.c_int, u64p]
        L.or_sweep_sets.argtypes = [u32p, u32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u64p]
        _lib = L
    return _lib


CURSOR_PER_KERNEL = 1  # L4 alt.: the round-robin cursor restarts at SM 0 for every kernel
STRICT_RR = 2          # L4 alt.: a block goes to the cursor's SM or nowhere (no scan)
SKIP_AHEAD = 4         # L5 alt.: a blocked kernel waits, later kernels keep filling the round


def _gpu_arr(gpu):
    """7-tuple (Table 1 GPU parameters) or 8-tuple with model-reading flags
    (CURSOR_PER_KERNEL | STRICT_RR | SKIP_AHEAD; rk_oracle.cpp OrGpu)."""
    assert len(gpu) in (7, 8)
    g = [int(x) for x in gpu] + ([0] if len(gpu) == 7 else [])
    return (ctypes.c_uint32 * 8)(*g)


def _kern_arr(kernels):
    flat = []
    for k in kernels:
        assert len(k) == 6
        flat.extend(int(x) for x in k)
    return (ctypes.c_uint32 * max(1, len(flat)))(*flat)


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle error {code}")
        self.code = code


def _chk(code: int):
    if code != OR_OK:
        raise OracleError(code)


def check_inputs(gpu, kernels) -> int:
    return lib().or_check_inputs(_gpu_arr(gpu), _kern_arr(kernels), len(kernels))


def factorial(n: int) -> int:
    return int(lib().or_factorial(n))


def unrank(idx: int, n: int) -> list[int]:
    o = (ctypes.c_int32 * max(1, n))()
    lib().or_unrank(idx, n, o)
    return list(o)[:n]


def rank(order) -> int:
    o = (ctypes.c_int32 * max(1, len(order)))(*order)
    return int(lib().or_rank(o, len(order)))


@dataclass
class SimResult:
    key: int                 # exact K = sum_r max(den*I_r, num*M_r)
    t_naive: float           # SPEC:210 literal double formula
    rounds: list             # p[r][i]
    trace: list | None       # [(round, sm)] per block in dispatch order


def simulate(gpu, kernels, order, trace: bool = False, max_rounds: int = 4096) -> SimResult:
    n = len(kernels)
    rounds = (ctypes.c_uint32 * (max_rounds * max(1, n)))()
    nr = ctypes.c_int32()
    lo, hi, tn = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_double()
    tot = sum(int(k[0]) for k in kernels)
    tr = (ctypes.c_int32 * max(2, 2 * tot))() if trace else None
    o = (ctypes.c_int32 * max(1, n))(*order)
    _chk(lib().or_simulate(_gpu_arr(gpu), _kern_arr(kernels), n, o, rounds, max_rounds, ctypes.byref(nr),
                           ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(tn), tr))
    R = nr.value
    rl = [[rounds[r * n + i] for i in range(n)] for r in range(R)]
    t = [(tr[2 * b], tr[2 * b + 1]) for b in range(tot)] if trace else None
    return SimResult(key=(hi.value << 64) | lo.value, t_naive=tn.value, rounds=rl, trace=t)


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
    max_rel_err: float = 0.0

    def as_tuple(self):
        return (self.key_min, self.key_max, self.argmin, self.argmax, self.n_lt, self.n_eq, self.n_gt, self.evaluated)


def sweep(gpu, kernels, first: int = 0, count: int | None = None, cand_key: int = 0, threads: int = 1,
          keys: bool = False):
    """Returns (Stats, keys-list-or-None)."""
    import numpy as np

    n = len(kernels)
    if count is None:
        count = factorial(n) - first
    st = (ctypes.c_uint64 * 8)()
    err = ctypes.c_double()
    karr = np.zeros(count if keys else 0, dtype=np.uint64)
    kp = karr.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) if keys else None
    _chk(lib().or_sweep(_gpu_arr(gpu), _kern_arr(kernels), n, first, count, cand_key, threads, st, kp,
                        ctypes.byref(err)))
    s = Stats(*[int(x) for x in st], max_rel_err=err.value)
    return s, (karr if keys else None)


def keys_of(gpu, kernels, indices, threads: int = 1):
    """Keys of explicit lexicographic indices (numpy uint64 array in, out)."""
    import numpy as np

    idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
    out = np.zeros(len(idx), dtype=np.uint64)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    _chk(lib().or_keys_of(_gpu_arr(gpu), _kern_arr(kernels), len(kernels), idx.ctypes.data_as(u64p), len(idx),
                          threads, out.ctypes.data_as(u64p)))
    return out


def histogram(keys, kmin: int, kmax: int, bins: int):
    import numpy as np

    k = np.ascontiguousarray(keys, dtype=np.uint64)
    h = np.zeros(bins, dtype=np.uint64)
    _chk(lib().or_histogram(k.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(k), kmin, kmax, bins,
                            h.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return [int(x) for x in h]


def heuristic(gpu, kernels):
    """Algorithm 1 -> (order, round_of)."""
    n = len(kernels)
    o = (ctypes.c_int32 * max(1, n))()
    r = (ctypes.c_int32 * max(1, n))()
    _chk(lib().or_heuristic(_gpu_arr(gpu), _kern_arr(kernels), n, o, r))
    return list(o)[:n], list(r)[:n]


def pair_score(gpu, kernels, i: int, j: int):
    """ScoreGen(K_i, K_j) and ProfileCombine ratio -> (feasible, score, r_comb)."""
    f, s, rc = ctypes.c_int32(), ctypes.c_double(), ctypes.c_double()
    _chk(lib().or_pair_score(_gpu_arr(gpu), _kern_arr(kernels), i, j, ctypes.byref(f), ctypes.byref(s),
                             ctypes.byref(rc)))
    return bool(f.value), s.value, rc.value


def sweep_sets(gpu, sets, threads: int = 1):
    """Per set: (Stats, cand_index, cand_key) with the candidate = Algorithm 1's order."""
    import numpy as np

    n = len(sets[0])
    flat = [k for s in sets for k in s]
    out = np.zeros(10 * len(sets), dtype=np.uint64)
    _chk(lib().or_sweep_sets(_gpu_arr(gpu), _kern_arr(flat), n, len(sets), threads,
                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    res = []
    for s in range(len(sets)):
        o = [int(x) for x in out[10 * s:10 * s + 10]]
        res.append((Stats(*o[:8]), o[8], o[9]))
    return res
