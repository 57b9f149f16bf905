"""The multi-rank CUDA path executed: world 2 and 3
ranks, each running the product's step (Sweeper.run -> rk_sweep_pass1/2 on its
contiguous shard, the record all_gather + device merge, the histogram+count
all_reduce + final merge) on the one GPU of the test box, the collectives over
gloo (CUDA tensors staged through host memory).  No rank's kernel waits on
another rank's kernel: the exchanges are the host collectives.  The merged
report, histogram and median must equal the oracle goldens of the full space."""
import json
import math
import os
import queue
import socket
import time

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1511_07983_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q, compact=False):
    from paper_1511_07983_b200.sweep import Sweeper

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    gpu, ks = W.config(cfg)
    sw = Sweeper(gpu, device=0, compact_keys=compact)
    rep = sw.run(ks, median=True)
    launches = sw.launches
    rep2 = sw.run(ks)  # a second step on the same Sweeper (buffers reused)
    if rank == 0:
        q.put((rep.__dict__, rep2.__dict__, launches, sw.first, sw.count))
    else:
        q.put(("shard", rank, sw.first, sw.count, rep.__dict__))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, cfg, compact=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q, compact)) for r in range(world)]
    for p in procs:
        p.start()
    got, shards, t0 = None, {}, time.time()
    while got is None or len(shards) < world - 1:
        try:
            m = q.get(timeout=2)
        except queue.Empty:
            assert not any(p.exitcode not in (None, 0) for p in procs), "a rank failed"
            assert time.time() - t0 < 600, "timeout"
            continue
        if m[0] == "shard":
            shards[m[1]] = m[2:]
        else:
            got = m
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return got, shards


@pytest.mark.parametrize("world,cfg,compact", [(2, "C3", False), (3, "C3", False), (2, "C4", False), (3, "C4", False),
                                               (2, "C4", True), (3, "C3", True)])
def test_multi_rank_cuda_step_equals_oracle_golden(world, cfg, compact):
    """compact=True: the bench's form (exact u32 key offsets; the overflow test on
    the merged global range, so every rank decides alike)."""
    with open(os.path.join(GOLD, f"{cfg.lower()}_oracle.json")) as f:
        g = json.load(f)
    (rep, rep2, launches, first, count), shards = _run(world, cfg, compact)
    N = math.factorial(len(W.config(cfg)[1]))
    assert first == 0 and count == N // world
    assert sorted(shards) == list(range(1, world)) and sum(c for _, c, _ in shards.values()) + count == N
    st = g["stats"]
    for r in (rep, rep2):
        assert (r["best_key"], r["worst_key"], r["best_index"], r["worst_index"]) == \
            (st["key_min"], st["key_max"], st["argmin"], st["argmax"])
        assert (r["n_lt"], r["n_eq"], r["n_gt"]) == (st["n_lt"], st["n_eq"], st["n_gt"])
        assert r["cand_key"] == g["cand_key"] and r["cand_index"] == g["cand_index"]
        if g.get("bins", 256) == 256 and "hist" in g:
            assert r["hist"] == g["hist"]
        assert sum(r["hist"]) == N
    # every rank holds the same merged report
    for _, _, other in shards.values():
        assert other["best_key"] == rep["best_key"] and other["hist"] == rep["hist"]
    if "order_stats" in g and str((N - 1) // 2) in g["order_stats"]:
        assert rep["median_key"] == g["order_stats"][str((N - 1) // 2)]
    assert launches > 0
