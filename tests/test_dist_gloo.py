"""Multi-rank host logic over gloo on CPU (world_size 2 and 3): index-space
shards, the record all_gather layout and the histogram all_reduce of
paper_1511_07983_b200.dist.  Per-rank shard results come from the oracle (test
infrastructure); the product's collective helpers move them."""
import math
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1511_07983_b200 import dist as D
from paper_1511_07983_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pack(t):
    """oracle Stats tuple -> the 8 int64 words of an rk_stats record (64 B)."""
    return [x if x < (1 << 63) else x - (1 << 64) for x in t]


def _unpack(w):
    return tuple(x & ((1 << 64) - 1) for x in w)


def _merge(records):
    """Reference merge for the test: lexicographic (key, idx) min / (key, -idx) max."""
    recs = [_unpack(r) for r in records]
    recs = [r for r in recs if r[7] > 0]
    kmin, amin = min((r[0], r[2]) for r in recs)
    kmax, amax = max(((r[1], -r[3]) for r in recs))
    return (kmin, kmax, amin, -amax, sum(r[4] for r in recs), sum(r[5] for r in recs), sum(r[6] for r in recs),
            sum(r[7] for r in recs))


def _worker(rank, world, port, cfg, q):
    import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gpu, ks = W.config(cfg)
    N = math.factorial(len(ks))
    cand = O.simulate(gpu, ks, O.heuristic(gpu, ks)[0]).key
    first, count = D.shard_bounds(N, world, rank)
    st, keys = O.sweep(gpu, ks, first, count, cand_key=cand, keys=True)
    rec = torch.tensor(_pack(st.as_tuple()), dtype=torch.int64)
    allrecs = D.all_gather_records(rec)
    g = _merge([tuple(int(v) for v in row) for row in allrecs.tolist()])
    hist = torch.tensor(O.histogram(keys, g[0], g[1], 64), dtype=torch.int64)
    D.all_reduce_hist(hist)
    t = D.max_over_ranks(float(rank + 1), torch.device("cpu"))
    if rank == 0:
        q.put((g, hist.tolist(), t, allrecs.shape))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sweep_over_gloo_equals_unsharded(world):
    import oracle as O

    cfg = "C2"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    t0 = time.time()
    while True:
        try:
            g, hist, tmax, shape = q.get(timeout=2)
            break
        except queue.Empty:
            assert not any(p.exitcode not in (None, 0) for p in procs), "a rank failed"
            assert time.time() - t0 < 240, "timeout"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gpu, ks = W.config(cfg)
    cand = O.simulate(gpu, ks, O.heuristic(gpu, ks)[0]).key
    full, keys = O.sweep(gpu, ks, cand_key=cand, keys=True)
    assert g == full.as_tuple()
    assert hist == O.histogram(keys, full.key_min, full.key_max, 64)
    assert tmax == float(world) and tuple(shape) == (world, D.REC_WORDS)


def test_shard_bounds_partition():
    for total in (1, 24, 40320, math.factorial(12)):
        for world in (1, 2, 3, 4, 7, 8):
            b = [D.shard_bounds(total, world, r) for r in range(world)]
            assert b[0][0] == 0 and sum(c for _, c in b) == total
            for (f0, c0), (f1, _) in zip(b, b[1:]):
                assert f0 + c0 == f1
            assert max(c for _, c in b) - min(c for _, c in b) <= 1


def _sel_worker(rank, world, port, q):
    import numpy as np

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    allkeys = rng.integers(10 ** 10, 10 ** 10 + 10 ** 7, 50000).astype(np.int64)
    allkeys[:5] = [10 ** 10, 10 ** 10 + 10 ** 7 - 1, 10 ** 10 + 3, 10 ** 10 + 3, 10 ** 10 + 3]
    first, count = D.shard_bounds(len(allkeys), world, rank)
    mine = allkeys[first:first + count]

    def count_fn(lo, span, nb):  # test-side counter (the GPU uses rk_range_histogram)
        x = mine[(mine >= lo) & (mine < lo + span)] - lo
        return torch.from_numpy(np.bincount((x * nb) // span, minlength=nb).astype(np.int64))

    ranks = [0, len(allkeys) - 1, (len(allkeys) - 1) // 2, 1, 2, 3, 12345]
    got = D.select_keys_sharded(count_fn, int(allkeys.min()), int(allkeys.max()), ranks, bins=64)
    if rank == 0:
        q.put((got, [int(v) for v in np.sort(allkeys)[ranks]]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 3])
def test_sharded_order_statistics_over_gloo(world):
    import queue
    import time
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sel_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    t0 = time.time()
    while True:
        try:
            got, want = q.get(timeout=2)
            break
        except queue.Empty:
            assert not any(p.exitcode not in (None, 0) for p in procs), "a rank failed"
            assert time.time() - t0 < 240, "timeout"
    for p in procs:
        p.join(timeout=60)
    assert got == want
