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
    """oracle Stats tuple -> the 7 int64 words of an rk_stats record (56 B)."""
    kmin, kmax, amin, amax, lt, eq, gt, ev = t
    w = [kmin, kmax, amin | (amax << 32), lt, eq, gt, ev]
    return [x if x < (1 << 63) else x - (1 << 64) for x in w]


def _unpack(w):
    w = [x & ((1 << 64) - 1) for x in w]
    return (w[0], w[1], w[2] & 0xFFFFFFFF, w[2] >> 32, w[3], w[4], w[5], w[6])


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
