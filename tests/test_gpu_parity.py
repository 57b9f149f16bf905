"""GPU parity: the CUDA path (through the C-ABI) vs the oracle, element by
element on the same seeded inputs.  Bit-exact keys, round partitions,
argmin/argmax, counts, histograms; doubles K/den within 1e-12 of the oracle's
naive SPEC:210 double (O5).
"""
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402
from paper_1511_07983_b200 import rk  # noqa: E402
from paper_1511_07983_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
NCPU = os.cpu_count() or 1


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the -m gpu suite needs a B200 (no CPU fallback)")
    c = rk.Context(0)
    yield c
    c.close()


def gpu_keys(ctx, gpu, ks, first=0, count=None, cand=0):
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    n = len(ks)
    if count is None:
        count = math.factorial(n) - first
    keys = torch.zeros(max(count, 1), dtype=torch.int64, device="cuda")
    st = ctx.rk_eval_range(first, count, cand, keys_dev=keys)
    return st, keys[:count].cpu().numpy().view(np.uint64)


def check_full_space(ctx, gpu, ks, cand=None, bins=(1, 4, 256)):
    n = len(ks)
    if cand is None:
        cand = O.simulate(gpu, ks, O.heuristic(gpu, ks)[0]).key
    st, keys = gpu_keys(ctx, gpu, ks, cand=cand)
    ost, okeys = O.sweep(gpu, ks, cand_key=cand, threads=NCPU, keys=True)
    assert np.array_equal(keys, okeys), "per-order keys differ"
    assert st.as_tuple() == ost.as_tuple()
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    for B in bins:
        h = torch.zeros(B, dtype=torch.int64, device="cuda")
        ctx.rk_histogram(kd, len(keys), st.key_min, st.key_max, B, h)
        torch.cuda.synchronize()
        assert h.cpu().tolist() == O.histogram(okeys, ost.key_min, ost.key_max, B)
    return st


def test_w4_golden(ctx):
    g = _gold("w4.json")
    st, keys = gpu_keys(ctx, g["gpu"], g["kernels"], cand=100 * g["heuristic"]["T"])
    assert [int(k) for k in keys] == [100 * row[3] for row in g["orders"]]
    assert st.key_min == 100 * g["stats"]["best"] and st.argmin == g["stats"]["argmin"]
    assert st.key_max == 100 * g["stats"]["worst"] and st.argmax == g["stats"]["argmax"]
    assert st.n_eq + st.n_gt == 24 and st.n_lt == 0
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    for B, want in ((4, g["hist4"]), (8, g["hist8"])):
        h = torch.zeros(B, dtype=torch.int64, device="cuda")
        ctx.rk_histogram(kd, 24, st.key_min, st.key_max, B, h)
        assert h.cpu().tolist() == want
    order, round_of, idx, key = ctx.rk_heuristic_order()
    assert order == g["heuristic"]["order"] and idx == g["heuristic"]["index"] and key == 100 * g["heuristic"]["T"]
    nge, k2 = ctx.rk_percentile(order, 0, 24)
    assert k2 == key and 100.0 * nge / 24 == g["heuristic"]["percentile"]
    for row in g["orders"]:
        rounds, key = ctx.rk_simulate_order([int(c) for c in row[1]])
        assert key == 100 * row[3]
        assert rounds == O.simulate(g["gpu"], g["kernels"], [int(c) for c in row[1]]).rounds


def test_w2_cursor_and_counterexamples(ctx):
    w = _gold("w2_cursor.json")
    ctx.rk_set_gpu_params(w["gpu"])
    ctx.rk_set_kernels(w["kernels"])
    rounds, key = ctx.rk_simulate_order(w["order"])
    assert rounds == w["rounds"] and key == w["T"]
    c = _gold("counterexamples.json")
    ctx.rk_set_gpu_params(c["C1"]["gpu"])
    ctx.rk_set_kernels(c["C1"]["kernels"])
    for order, T, rr in c["C1"]["cases"]:
        assert ctx.rk_simulate_order(order) == (rr, T)
    c2 = c["C2"]
    ctx.rk_set_gpu_params(c2["gpu"])
    ctx.rk_set_kernels(c2["kernels"])
    assert ctx.rk_simulate_order(c2["with_X_first"]["order"])[1] == c2["with_X_first"]["T"]
    ctx.rk_set_kernels([c2["kernels"][i] for i in c2["without_X"]["kernels_idx"]])
    assert ctx.rk_simulate_order(c2["without_X"]["order"])[1] == c2["without_X"]["T"]


def test_c1_random_sets(ctx):
    for ks in W.c1_random_sets():
        check_full_space(ctx, W.GTX580, ks, bins=(3,))


def test_c2_full_space_vs_oracle_and_golden(ctx):
    gpu, ks = W.config("C2")
    g = _gold("c2_oracle.json")
    st = check_full_space(ctx, gpu, ks, cand=g["cand_key"])
    assert list(st.as_tuple()) == [g["stats"][f] for f in
                                   ("key_min", "key_max", "argmin", "argmax", "n_lt", "n_eq", "n_gt", "evaluated")]


def test_c3_full_space_vs_oracle(ctx):
    gpu, ks = W.config("C3")
    g = _gold("c3_oracle.json")
    st = check_full_space(ctx, gpu, ks, cand=g["cand_key"], bins=(256,))
    assert st.evaluated == 3628800 and st.key_min == g["stats"]["key_min"] and st.argmin == g["stats"]["argmin"]


GPUS = [W.GTX580, (8, 65536, 102400, 64, 16, 7, 2), (3, 16384, 16384, 32, 4, 5, 1), (32, 65536, 98304, 64, 32, 1, 1),
        (13, 32768, 49152, 48, 8, 411, 100), (1, 65536, 49152, 48, 2, 1, 1), (5, 65536, 65536, 64, 3, 9, 4)]


@pytest.mark.parametrize("gi", range(len(GPUS)))
def test_random_sets_many_gpu_shapes(ctx, gi):
    gpu = GPUS[gi]
    sets = W.random_small_sets(0xD00D + gi, 30, 1, 7, gpu=gpu)
    done = 0
    for ks in sets:
        if not all(W.feasible(gpu, k) for k in ks):
            continue
        try:
            ctx.rk_set_gpu_params(gpu)
            ctx.rk_set_kernels(ks)
        except rk.RkError as e:
            assert e.status == rk.RK_EUNSUPPORTED
            continue
        check_full_space(ctx, gpu, ks, bins=(7,))
        done += 1
    assert done >= 5


@pytest.mark.parametrize("seed", range(4))
def test_round_partitions_random_orders(ctx, seed):
    rng = W.SplitMix64(0x9A27 + seed)
    for gi, gpu in enumerate(GPUS):
        for ks in W.random_small_sets(0x51 + seed * 31 + gi, 4, 1, 12, gpu=gpu):
            if not all(W.feasible(gpu, k) for k in ks):
                continue
            try:
                ctx.rk_set_gpu_params(gpu)
                ctx.rk_set_kernels(ks)
            except rk.RkError as e:
                assert e.status == rk.RK_EUNSUPPORTED
                continue
            for _ in range(5):
                order = list(range(len(ks)))
                for i in range(len(order) - 1, 0, -1):
                    j = rng.below(i + 1)
                    order[i], order[j] = order[j], order[i]
                rounds, key = ctx.rk_simulate_order(order)
                o = O.simulate(gpu, ks, order)
                assert rounds == o.rounds and key == o.key
                T = key / gpu[6]
                assert abs(T - o.t_naive) <= 1e-12 * T  # north_star 1e-12 on the float time


def test_ranges_edges_and_sharding(ctx):
    gpu, ks = W.config("C2")
    full, fkeys = gpu_keys(ctx, gpu, ks, cand=12130259200)
    N = 40320
    for first, count in ((0, 1), (1, 1), (5, 7), (7, 13), (40319, 1), (12345, 6789), (0, 0), (40314, 6)):
        st, keys = gpu_keys(ctx, gpu, ks, first, count, cand=12130259200)
        assert np.array_equal(keys, fkeys[first:first + count])
        if count:
            ost, _ = O.sweep(gpu, ks, first, count, cand_key=12130259200)
            assert st.as_tuple() == ost.as_tuple()
        else:
            assert st.evaluated == 0
    # G shards merged on the device == unsharded (deterministic merge)
    for G in (2, 3, 8):
        recs = torch.zeros((G, 8), dtype=torch.int64, device="cuda")  # 64 B per record
        bounds = [N * g // G for g in range(G + 1)]
        cand = torch.tensor([12130259200], dtype=torch.int64, device="cuda")
        for g in range(G):
            ctx.rk_eval_range_async(bounds[g], bounds[g + 1] - bounds[g], cand, recs[g])
        out = torch.zeros(8, dtype=torch.int64, device="cuda")
        ctx.rk_merge_stats_async(recs, G, out)
        torch.cuda.synchronize()
        assert rk.Stats.from_c(rk.rk_stats.from_buffer_copy(out.cpu().numpy().tobytes())).as_tuple() == full.as_tuple()


def test_small_n(ctx):
    for n in (1, 2, 3):
        for ks in W.random_small_sets(0x5A + n, 5, n, n):
            check_full_space(ctx, W.GTX580, ks, bins=(2,))


def test_errors_through_abi(ctx):
    ctx.rk_set_gpu_params(W.GTX580)
    with pytest.raises(rk.RkError) as e:
        ctx.rk_set_kernels([(16, 128, 20, 65536, 311, 100)])
    assert e.value.status == rk.RK_EINFEASIBLE
    ctx.rk_set_kernels(W.W4)
    with pytest.raises(rk.RkError) as e:
        ctx.rk_eval_range(20, 5)
    assert e.value.status == rk.RK_EINVAL


def test_c4_full_space_bench_config_vs_oracle_golden(ctx):
    """12! in the launch configuration bench.py times (rk_sweep_pass1/2: the
    memoised step with keys, counts and the fused histogram): aggregates +
    histogram vs the full multi-core oracle run (tests/golden/c4_oracle.json);
    per-order keys by the SURVEY §8(d) protocol — 10^6 random indices plus the
    first and last 10^5 indices of every shard of an 8-way split — each
    computed by the oracle one by one (O.keys_of)."""
    g = _gold("c4_oracle.json")
    gpu, ks = W.config("C4")
    assert g["kernels"] == [list(k) for k in ks]
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    assert ctx.rk_memo_info()[0], "the bench configuration runs the memoised step"
    order, _, idx, key = ctx.rk_heuristic_order()
    assert order == g["cand_order"] and idx == g["cand_index"] and key == g["cand_key"]
    N = math.factorial(12)
    keys = torch.empty(N, dtype=torch.int64, device="cuda")
    cand = torch.tensor([key], dtype=torch.int64, device="cuda")
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    hist = torch.zeros(g["bins"], dtype=torch.int64, device="cuda")
    ctx.rk_sweep_pass1_async(0, N, cand, rec, keys)
    ctx.rk_sweep_pass2_async(0, N, cand, rec, g["bins"], hist, keys, rec)
    torch.cuda.synchronize()
    st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
    assert list(st.as_tuple()) == [g["stats"][f] for f in
                                   ("key_min", "key_max", "argmin", "argmax", "n_lt", "n_eq", "n_gt", "evaluated")]
    assert hist.cpu().tolist() == g["hist"]
    rng = np.random.default_rng(12)
    parts = [rng.integers(0, N, 10 ** 6)]
    for s in range(8):
        lo, hi = s * N // 8, (s + 1) * N // 8
        parts += [np.arange(lo, lo + 10 ** 5), np.arange(hi - 10 ** 5, hi)]
    sample = np.concatenate(parts).astype(np.uint64)
    want = O.keys_of(gpu, ks, sample, threads=NCPU)
    got = keys[torch.from_numpy(sample.view(np.int64)).cuda()].cpu().numpy().view(np.uint64)
    bad = np.nonzero(got != want)[0]
    assert len(bad) == 0, f"{len(bad)} of {len(sample)} sampled keys differ, e.g. index {sample[bad[0]]}"
    # O5: the reported doubles K/den are within 1e-12 of the naive SPEC:210 double
    for i, k in zip(sample[:200].tolist(), want[:200].tolist()):
        r = O.simulate(gpu, ks, O.unrank(i, 12))
        assert abs(r.t_naive - k / gpu[6]) <= 1e-12 * r.t_naive


def test_memo_with_cursor_per_kernel_reading_vs_oracle(monkeypatch):
    """Memoisation under RK_FLAG_CURSOR_PER_KERNEL (the L4 alternative; the
    level/suffix tables and the run pass all use the flag): full spaces of C2,
    C3 and random n = 6..8 sets over the GPU shapes, memoisation forced on,
    every key and statistic vs the block-by-block oracle."""
    ctx = _direct_ctx(monkeypatch, "RK_FORCE_MEMO")
    try:
        cases = [W.config("C2"), W.config("C3")]
        for gi, gpu in enumerate(GPUS[:5]):
            for ks in W.random_small_sets(0xC0C0 + gi, 3, 6, 8, gpu=gpu):
                if all(W.feasible(gpu, k) for k in ks):
                    cases.append((gpu, ks))
        checked = 0
        for gpu, ks in cases:
            g = list(gpu) + [rk.RK_FLAG_CURSOR_PER_KERNEL]
            try:
                ctx.rk_set_gpu_params(g)
                ctx.rk_set_kernels(ks)
            except rk.RkError as e:
                assert e.status == rk.RK_EUNSUPPORTED
                continue
            if not ctx.rk_memo_info()[0]:
                continue
            check_full_space(ctx, g, ks, bins=(64,))
            checked += 1
        assert checked >= 6
    finally:
        ctx.close()


def test_c5_batch_vs_oracle_golden(ctx):
    g = _gold("c5_oracle.json")
    sets = W.c5_sets(g["n_sets"])
    ctx.rk_set_gpu_params(W.GTX580)
    res = ctx.rk_eval_batch(sets)
    for (st, ck), want in zip(res, g["sets"]):
        assert list(st.as_tuple()) == want["stats"]
        assert ck == want["cand_key"]
    idx = [w["cand_index"] for w in g["sets"]]
    res2 = ctx.rk_eval_batch(sets, cand_index=idx)
    assert [r[0].as_tuple() for r in res2] == [r[0].as_tuple() for r in res]


def test_c5_full_batch_properties(ctx):
    sets = W.c5_sets(4096)
    ctx.rk_set_gpu_params(W.GTX580)
    res = ctx.rk_eval_batch(sets)
    F = math.factorial(9)
    for st, ck in res:
        assert st.evaluated == F and st.n_lt + st.n_eq + st.n_gt == F
        assert st.key_min <= ck <= st.key_max and st.n_eq >= 1


def test_symmetry_reduction_equivalence(ctx):
    """gcd(N_SM, grids) SMs act as one super-SM.  The reduced and
    unreduced device paths give bit-identical keys; odd grids (g = 1) still match
    the oracle."""
    gpu, ks = W.config("C2")  # g = 16 -> 1 super-SM
    _, k_red = gpu_keys(ctx, gpu, ks)
    os.environ["RK_NO_REDUCE"] = "1"
    try:
        c2 = rk.Context(0)
        c2.rk_set_gpu_params(gpu)
        c2.rk_set_kernels(ks)
        keys = torch.zeros(40320, dtype=torch.int64, device="cuda")
        c2.rk_eval_range(0, 40320, 0, keys_dev=keys)
        assert np.array_equal(keys.cpu().numpy().view(np.uint64), k_red)
        c2.close()
    finally:
        del os.environ["RK_NO_REDUCE"]
    rng = W.SplitMix64(0x0DD)
    for _ in range(6):
        sets = W.random_small_sets(rng.next(), 1, 5, 7)
        ks = [(k[0] + (rng.below(7) if rng.below(2) else 0),) + tuple(k[1:]) for k in sets[0]]
        check_full_space(ctx, W.GTX580, ks, bins=(5,))


DEGENERATE = {
    # all R_i >= R_B: every order has the same key (same-side theorem)
    "same_side": (W.GTX580, [(32, 256, 20, 0, 1110 * 8, 100 * 8), (48, 128, 32, 8192, 2400 * 4, 100 * 4),
                             (16, 512, 16, 16384, 600 * 16, 100 * 16), (64, 64, 24, 0, 800 * 2, 100 * 2)]),
    # identical kernels differing only in N_tblk
    "identical": (W.GTX580, [(t, 256, 24, 12288, 311 * 8, 100 * 8) for t in (16, 48, 80, 128, 32)]),
    # total blocks <= N_SM: one round for every order
    "one_round": (W.GTX580, [(3, 256, 24, 0, 311, 100), (5, 128, 20, 4096, 1110, 100), (8, 64, 16, 0, 2400, 100)]),
    # zero register and zero shared-memory demand (magic / numerator-mask path)
    "zero_demand": (W.GTX580, [(24, 128, 0, 0, 311, 100), (40, 256, 0, 8192, 1110, 100), (17, 64, 8, 0, 150, 100),
                               (33, 96, 0, 16384, 2400, 100)]),
    # one block per SM per kernel and one super-SM: SC == 1 (full-round division fallback)
    "sc_one": (W.GTX580, [(48, 128, 20, 49152, 311, 100), (32, 128, 20, 40000, 1110, 100),
                          (64, 1024, 32, 0, 600, 100)]),
    # N_blk_SM = 1 (no binary search), many rounds, odd grids
    "one_slot": ((7, 65536, 65536, 64, 1, 3, 2), [(9, 64, 8, 0, 7, 3), (13, 128, 16, 1024, 5, 9), (4, 32, 8, 0, 11, 2),
                                                  (21, 256, 4, 0, 2, 5)]),
    # many full single-kernel rounds (nfull > 0) with large grids
    "long_grids": (W.GTX580, [(2000, 256, 32, 16384, 311, 100), (1600, 128, 20, 0, 1110, 100),
                              (3000, 512, 16, 4096, 150, 100), (800, 64, 63, 24576, 2400, 100)]),
}


@pytest.mark.parametrize("name", sorted(DEGENERATE))
def test_degenerate_and_edge_inputs(ctx, name):
    gpu, ks = DEGENERATE[name]
    st = check_full_space(ctx, gpu, ks, bins=(1, 3, 256))
    if name in ("same_side", "identical"):
        assert st.key_min == st.key_max and st.argmin == 0 and st.argmax == 0
    if name == "one_round":
        for p in range(math.factorial(len(ks))):
            rounds, _ = ctx.rk_simulate_order(O.unrank(p, len(ks)))
            assert len(rounds) == 1


def test_max_n12_many_rounds_one_sm(ctx):
    # n = 12 on a 1-SM GPU with 2 block slots: sampled indices vs the oracle
    gpu = (1, 65536, 49152, 48, 2, 1, 1)
    ks = [(1 + (i % 3), 32 * (1 + i % 4), 8, 1024 * (i % 5), 3 + i, 2 + (7 * i) % 5) for i in range(12)]
    N = math.factorial(12)
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    keys = torch.empty(N, dtype=torch.int64, device="cuda")
    st = ctx.rk_eval_range(0, N, 0, keys_dev=keys)
    assert st.evaluated == N
    rng = np.random.default_rng(5)
    idx = np.concatenate([rng.integers(0, N, 3000), [0, N - 1, st.argmin, st.argmax]])
    kh = keys[torch.from_numpy(idx).cuda()].cpu().numpy().view(np.uint64)
    for i, k in zip(idx.tolist(), kh.tolist()):
        assert O.simulate(gpu, ks, O.unrank(i, 12)).key == k
    assert int(kh[-2]) == st.key_min and int(kh[-1]) == st.key_max


def test_order_statistics_median_and_ranks(ctx):
    """median = lower-middle of the sorted times; Fig. 1 ranking curve =
    keys at chosen ranks.  rk_select_keys vs a library sort of the oracle keys."""
    g = _gold("w4.json")
    st, keys = gpu_keys(ctx, g["gpu"], g["kernels"])
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    # hand distribution {126464:16, 129664:2, 131264:2, 132864:4}: ranks 11 (median), 16, 18, 20, 23
    got = ctx.rk_select_keys(kd, 24, st.key_min, st.key_max, [11, 15, 16, 18, 20, 23, 0])
    assert got == [100 * t for t in (126464, 126464, 129664, 131264, 132864, 132864, 126464)]
    for name in ("C2", "C3"):
        gpu, ks = W.config(name)
        st, keys = gpu_keys(ctx, gpu, ks)
        _, okeys = O.sweep(gpu, ks, threads=NCPU, keys=True)
        srt = np.sort(okeys)
        N = len(srt)
        ranks = [0, N - 1, (N - 1) // 2, N // 3, 7 * N // 9, 1, N - 2] + [int(x) for x in
                                                                           np.random.default_rng(3).integers(0, N, 20)]
        kd = torch.from_numpy(keys.view(np.int64)).cuda()
        assert ctx.rk_select_keys(kd, N, st.key_min, st.key_max, ranks) == [int(srt[r]) for r in ranks]
        # the range-histogram building block: counts in [lo, lo+span) match a direct count
        lo, span = int(srt[N // 4]), int(srt[3 * N // 4] - srt[N // 4]) + 1
        h = torch.zeros(64, dtype=torch.int64, device="cuda")
        ctx.rk_range_histogram(kd, N, lo, span, 64, h)
        torch.cuda.synchronize()
        inside = okeys[(okeys >= lo) & (okeys < lo + span)]
        assert int(h.sum().item()) == len(inside)


def test_histogram_bin_count_equals_key_span(ctx):
    """Regression: bins == kmax - kmin (the 32-bit magic would be 2^32)."""
    gpu, ks = W.config("C2")
    st, keys = gpu_keys(ctx, gpu, ks)
    _, okeys = O.sweep(gpu, ks, threads=NCPU, keys=True)
    D = st.key_max - st.key_min
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    lo = int(np.sort(okeys)[100])
    sub = okeys[okeys >= lo]
    for B in (D, D - 1, D + 1) if D <= 65536 else ():
        h = torch.zeros(B, dtype=torch.int64, device="cuda")
        ctx.rk_histogram(kd, len(keys), st.key_min, st.key_max, B, h)
        assert h.cpu().tolist() == O.histogram(okeys, st.key_min, st.key_max, B)
    # unit-width range bins: span == bins
    span = 4096
    h = torch.zeros(span, dtype=torch.int64, device="cuda")
    ctx.rk_range_histogram(kd, len(keys), lo, span, span, h)
    want = np.bincount((sub[sub < lo + span] - np.uint64(lo)).astype(np.int64), minlength=span)
    assert h.cpu().numpy().tolist() == want.tolist()


@pytest.mark.parametrize("D,B", [(1000, 1000), (999, 1000), (1001, 1000), (5, 256), (1 << 33, 256), (1 << 40, 4096),
                                 ((1 << 62) + 12345, 7), (65536, 65536)])
def test_histogram_exact_on_synthetic_keys(ctx, D, B):
    """rk_histogram on arbitrary key arrays (every BinCalc path: 32-bit magic,
    64-bit reciprocal, 128-bit) vs the oracle's integer formula (O7)."""
    rng = np.random.default_rng(D % 1000 + B)
    kmin = 10 ** 9 + 17
    keys = (np.uint64(kmin) + rng.integers(0, D + 1, 100000, dtype=np.uint64)).astype(np.uint64)
    keys[:3] = [kmin, kmin + D, kmin + D // 2]
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    h = torch.zeros(B, dtype=torch.int64, device="cuda")
    ctx.rk_histogram(kd, len(keys), kmin, kmin + D, B, h)
    assert h.cpu().tolist() == O.histogram(keys, kmin, kmin + D, B)


def test_public_sweeper_report_vs_oracle():
    """The user-level call (Sweeper.run: host profiles in, Table-3 report out)."""
    from paper_1511_07983_b200.sweep import Sweeper
    for name in ("C2", "C3"):
        gpu, ks = W.config(name)
        rep = Sweeper(gpu, bins=64).run(ks, median=True)
        order, _ = O.heuristic(gpu, ks)
        cand = O.simulate(gpu, ks, order).key
        st, keys = O.sweep(gpu, ks, cand_key=cand, threads=NCPU, keys=True)
        N = len(keys)
        assert (rep.best_key, rep.best_index, rep.worst_key, rep.worst_index) == (st.key_min, st.argmin, st.key_max,
                                                                                st.argmax)
        assert rep.cand_order == order and rep.cand_key == cand and rep.cand_index == O.rank(order)
        assert (rep.n_lt, rep.n_eq, rep.n_gt) == (st.n_lt, st.n_eq, st.n_gt)
        assert rep.hist == O.histogram(keys, st.key_min, st.key_max, 64)
        assert rep.median_key == int(np.sort(keys)[(N - 1) // 2])  # SPEC:302 lower-middle
        assert abs(rep.percentile - 100.0 * (st.n_eq + st.n_gt) / N) < 1e-12
        assert rep.speedup_over_worst == st.key_max / cand


def test_compact_keys_histogram32_select32_and_overflow_flag(ctx):
    gpu, ks = W.config("C3")
    st, keys = gpu_keys(ctx, gpu, ks)
    N = len(keys)
    base = ctx.rk_key_lower_bound()
    sI = sum(k[0] * k[4] for k in ks)
    sM = sum(k[0] * k[5] for k in ks)
    assert base == max(gpu[6] * sI, gpu[5] * sM) <= st.key_min
    k32 = torch.empty(N, dtype=torch.int32, device="cuda")
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    ctx.rk_eval_range32_async(0, N, None, rec, k32, base, ovf)
    torch.cuda.synchronize()
    assert int(ovf.item()) == 0
    got = k32.cpu().numpy().view(np.uint32).astype(np.uint64) + np.uint64(base)
    assert np.array_equal(got, keys)
    assert rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes())).as_tuple()[:4] == \
        st.as_tuple()[:4]
    h = torch.zeros(256, dtype=torch.int64, device="cuda")
    ctx.rk_histogram32_async(k32, N, base, rec, 256, h)
    assert h.cpu().tolist() == O.histogram(keys, st.key_min, st.key_max, 256)
    srt = np.sort(keys)
    ranks = [0, N - 1, (N - 1) // 2, 12345]
    assert ctx.rk_select_keys32(k32, base, N, st.key_min, st.key_max, ranks) == [int(srt[r]) for r in ranks]
    # a base too far below the keys must raise the overflow flag
    ovf.zero_()
    ctx.rk_eval_range32_async(0, N, None, rec, k32, st.key_max - (1 << 32), ovf)
    torch.cuda.synchronize()
    assert int(ovf.item()) == 1


def test_public_sweeper_compact_keys_mode():
    from paper_1511_07983_b200.sweep import Sweeper
    gpu, ks = W.config("C2")
    a = Sweeper(gpu, bins=32).run(ks, median=True)
    b = Sweeper(gpu, bins=32, compact_keys=True).run(ks, median=True)
    assert a == b


def _set13():
    return W.gen_g(W.SplitMix64(W.SEED_BASE + 13), 13)


def test_n13_u64_indices_around_2_pow_32(ctx):
    """13! = 6.2e9 orders needs u64 indices."""
    gpu, ks = W.GTX580, _set13()
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    first, count = (1 << 32) - 3001, 6007
    keys = torch.empty(count, dtype=torch.int64, device="cuda")
    cand = O.simulate(gpu, ks, O.unrank(1 << 32, 13)).key
    st = ctx.rk_eval_range(first, count, cand, keys_dev=keys)
    ost, okeys = O.sweep(gpu, ks, first, count, cand_key=cand, threads=NCPU, keys=True)
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), okeys)
    assert st.as_tuple() == ost.as_tuple() and st.argmin >= first


def test_n13_full_space_two_pass_histogram(ctx):
    gpu, ks = W.GTX580, _set13()
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    N = math.factorial(13)
    order, _, idx, key = ctx.rk_heuristic_order()
    assert key == O.simulate(gpu, ks, order).key
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    cd = torch.tensor([key], dtype=torch.int64, device="cuda")
    ctx.rk_eval_range_async(0, N, cd, rec)  # pass 1: no keys stored (50 GB)
    hist = torch.zeros(256, dtype=torch.int64, device="cuda")
    rec2 = torch.zeros(8, dtype=torch.int64, device="cuda")
    ctx.rk_eval_range_hist_async(0, N, cd, rec2, rec, 256, hist)  # pass 2: fused binning
    torch.cuda.synchronize()
    st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
    assert torch.equal(rec, rec2)
    assert st.evaluated == N == st.n_lt + st.n_eq + st.n_gt and st.n_eq >= 1
    assert int(hist.sum().item()) == N
    # the extremes are real orders with exactly those keys (oracle, one by one)
    assert O.simulate(gpu, ks, O.unrank(st.argmin, 13)).key == st.key_min
    assert O.simulate(gpu, ks, O.unrank(st.argmax, 13)).key == st.key_max
    # no sampled order beats the minimum or exceeds the maximum
    rng = np.random.default_rng(13)
    for i in rng.integers(0, N, 300).tolist():
        assert st.key_min <= O.simulate(gpu, ks, O.unrank(i, 13)).key <= st.key_max
    # sharded (3 contiguous shards, device merge) == unsharded
    recs = torch.zeros((3, 8), dtype=torch.int64, device="cuda")
    for g in range(3):
        ctx.rk_eval_range_async(N * g // 3, N * (g + 1) // 3 - N * g // 3, cd, recs[g])
    out = torch.zeros(8, dtype=torch.int64, device="cuda")
    ctx.rk_merge_stats_async(recs, 3, out)
    torch.cuda.synchronize()
    assert torch.equal(out, rec)


def test_fused_histogram_pass_matches_oracle(ctx):
    gpu, ks = W.config("C3")
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    N = math.factorial(10)
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    ctx.rk_eval_range_async(0, N, None, rec)
    _, okeys = O.sweep(gpu, ks, threads=NCPU, keys=True)
    st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
    for B in (1, 7, 256, 32768):
        hist = torch.zeros(B, dtype=torch.int64, device="cuda")
        ctx.rk_eval_range_hist_async(0, N, None, None, rec, B, hist)
        torch.cuda.synchronize()
        assert hist.cpu().tolist() == O.histogram(okeys, st.key_min, st.key_max, B)
    # a sub-range accumulates only its own orders
    hist = torch.zeros(64, dtype=torch.int64, device="cuda")
    ctx.rk_eval_range_hist_async(1000, 5000, None, None, rec, 64, hist)
    torch.cuda.synchronize()
    assert hist.cpu().tolist() == O.histogram(okeys[1000:6000], st.key_min, st.key_max, 64)


def test_n16_tail_of_the_space(ctx):
    gpu = W.GTX580
    ks = W.gen_g(W.SplitMix64(W.SEED_BASE + 16), 16)
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    N = math.factorial(16)
    for first in (N - 2500, (N // 7) * 3):
        keys = torch.empty(2500, dtype=torch.int64, device="cuda")
        st = ctx.rk_eval_range(first, 2500, 0, keys_dev=keys)
        ost, okeys = O.sweep(gpu, ks, first, 2500, threads=NCPU, keys=True)
        assert np.array_equal(keys.cpu().numpy().view(np.uint64), okeys)
        assert st.as_tuple() == ost.as_tuple()


def test_c4_order_statistics_vs_oracle_golden(ctx):
    g = _gold("c4_oracle.json")
    if "order_stats" not in g:
        pytest.skip("golden predates order statistics")
    gpu, ks = W.config("C4")
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    N = math.factorial(12)
    keys = torch.empty(N, dtype=torch.int64, device="cuda")
    st = ctx.rk_eval_range(0, N, 0, keys_dev=keys)
    ranks = [int(r) for r in g["order_stats"]]
    got = ctx.rk_select_keys(keys, N, st.key_min, st.key_max, ranks)
    assert got == [g["order_stats"][str(r)] for r in ranks]
    assert g["median_rank"] == (N - 1) // 2


@pytest.mark.parametrize("gi", range(4))
def test_device_algorithm1_matches_oracle(ctx, gi):
    """Algorithm 1 on the GPU (one thread per set) == the oracle's."""
    gpu = [W.GTX580, (8, 65536, 102400, 64, 16, 7, 2), (24, 32768, 49152, 48, 8, 311, 100),
           (16, 32768, 49152, 48, 8, 411, 100)][gi]
    ctx.rk_set_gpu_params(gpu)
    for n in (1, 2, 3, 5, 8, 9, 12, 16):
        sets = [ks for ks in W.random_small_sets(0xF4 + 100 * gi + n, 60, n, n, gpu=gpu)
                if all(W.feasible(gpu, k) for k in ks)]
        if not sets:
            continue
        orders, idx = ctx.rk_heuristic_batch(sets)
        for ks, o, i in zip(sets, orders, idx):
            want, _ = O.heuristic(gpu, ks)
            assert o == want and i == O.rank(want)


def test_device_algorithm1_c5_and_configs(ctx):
    ctx.rk_set_gpu_params(W.GTX580)
    sets = W.c5_sets(4096)
    orders, idx = ctx.rk_heuristic_batch(sets)
    g = _gold("c5_oracle.json")
    assert idx[:g["n_sets"]] == [s["cand_index"] for s in g["sets"]]
    for ks, o in list(zip(sets, orders))[:512]:
        assert o == O.heuristic(W.GTX580, ks)[0]


def test_cursor_per_kernel_reading_vs_oracle(ctx):
    """model-reading variant (RK_FLAG_CURSOR_PER_KERNEL)."""
    w = _gold("w2_cursor.json")
    ctx.rk_set_gpu_params(list(w["gpu"]) + [rk.RK_FLAG_CURSOR_PER_KERNEL])
    ctx.rk_set_kernels(w["kernels"])
    assert ctx.rk_simulate_order(w["order"]) == (w["rejected_reading_rounds"], w["T_rejected_reading"])
    for gpu in (W.GTX580, (13, 32768, 49152, 48, 8, 411, 100), (8, 65536, 102400, 64, 16, 7, 2)):
        for ks in W.random_small_sets(0xF3 + gpu[0], 6, 3, 7, gpu=gpu):
            if not all(W.feasible(gpu, k) for k in ks):
                continue
            check_full_space(ctx, list(gpu) + [1], ks, bins=(16,))
    gpu, ks = W.config("C2")
    check_full_space(ctx, list(gpu) + [1], ks, bins=(256,))


def _check_best(ctx, gpu, ks, want_key, want_idx, seeds=(None,)):
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    for seed in seeds:
        order, idx, key, nodes = ctx.rk_best_order(seed)
        assert (key, idx) == (want_key, want_idx), (seed, key, idx, want_key, want_idx)
        assert order == O.unrank(idx, len(ks))
        assert O.simulate(gpu, ks, order).key == key
        assert 1 <= nodes <= len(ks) * math.factorial(len(ks)) * 2
    return nodes


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_branch_and_bound_equals_full_sweep_goldens(ctx, name):
    """rk_best_order == the oracle's full-space (key_min, argmin)."""
    gpu, ks = W.config(name)
    g = _gold(f"{name.lower()}_oracle.json")
    _check_best(ctx, gpu, ks, g["stats"]["key_min"], g["stats"]["argmin"],
                seeds=(None, g["cand_index"], g["stats"]["argmin"], g["stats"]["argmax"]))


@pytest.mark.parametrize("gi", range(len(GPUS)))
def test_branch_and_bound_random_sets_vs_oracle(ctx, gi):
    gpu = GPUS[gi]
    done = 0
    for ks in W.random_small_sets(0xB0B + gi, 24, 1, 8, gpu=gpu):
        if not all(W.feasible(gpu, k) for k in ks):
            continue
        try:
            ctx.rk_set_gpu_params(gpu)
            ctx.rk_set_kernels(ks)
        except rk.RkError as e:
            assert e.status == rk.RK_EUNSUPPORTED
            continue
        ost, _ = O.sweep(gpu, ks, threads=NCPU)
        seed = int(np.random.default_rng(len(ks) + gi).integers(0, math.factorial(len(ks))))
        _check_best(ctx, gpu, ks, ost.key_min, ost.argmin, seeds=(None, seed))
        done += 1
    assert done >= 5


def test_branch_and_bound_ties_and_cursor_reading(ctx):
    # identical kernels: every order has the same key -> argmin 0, no pruning possible
    k = (20, 256, 20, 4096, 100, 30)
    _check_best(ctx, W.GTX580, [k] * 7, O.simulate(W.GTX580, [k] * 7, list(range(7))).key, 0)
    # the cursor-per-kernel reading (f3) through the same search
    gpu, ks = W.config("C2")
    g1 = list(gpu) + [rk.RK_FLAG_CURSOR_PER_KERNEL]
    ost, _ = O.sweep(g1, ks, threads=NCPU)
    _check_best(ctx, g1, ks, ost.key_min, ost.argmin)


def test_branch_and_bound_n13_vs_full_device_sweep(ctx):
    """n = 13 (6.2e9 orders): the search agrees with the exhaustive device sweep
    (itself parity-tested) and the oracle re-simulates the optimum."""
    gpu, ks = W.GTX580, _set13()
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    N = math.factorial(13)
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    cd = torch.zeros(1, dtype=torch.int64, device="cuda")
    ctx.rk_eval_range_async(0, N, cd, rec)
    torch.cuda.synchronize()
    st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
    _, _, hidx, _ = ctx.rk_heuristic_order()
    nodes = _check_best(ctx, gpu, ks, st.key_min, st.argmin, seeds=(None, hidx))
    assert nodes < 13 * N


# ---- run-length SM state (S' > 32, e.g. the 148-SM B200 preset) ----
BIG_GPUS = [W.B200, (33, 32768, 49152, 48, 8, 411, 100), (40, 65536, 102400, 64, 16, 7, 2),
            (148, 65536, 233472, 64, 32, 1, 1), (1000, 32768, 49152, 48, 8, 411, 100)]


@pytest.mark.parametrize("gi", range(len(BIG_GPUS)))
def test_runs_state_random_sets_vs_oracle(ctx, gi):
    gpu = BIG_GPUS[gi]
    rng = W.SplitMix64(0x5EED + gi)
    done = 0
    sets = [W.gen_b200(rng, 2 + q % 6, gpu=gpu) for q in range(10)] if gpu[0] >= 148 and gpu[3] >= 64 else \
        W.random_small_sets(0x5EED + gi, 12, 2, 7, gpu=gpu)
    for ks in sets:
        if not all(W.feasible(gpu, k) for k in ks):
            continue
        ctx.rk_set_gpu_params(gpu)
        ctx.rk_set_kernels(ks)
        check_full_space(ctx, gpu, ks, bins=(5,))
        o = O.unrank(len(ks) // 2, len(ks))
        r = O.simulate(gpu, ks, o)
        assert ctx.rk_simulate_order(o) == (r.rounds, r.key)
        done += 1
    assert done >= 5


def test_runs_state_c6_b200_preset(ctx):
    """C6 = the B200 preset with 12 generator kernels (S' = 37 super-SMs): the full
    device sweep's extremes and 2000 sampled keys re-simulated by the oracle, and
    the branch-and-bound optimum agrees with the sweep."""
    gpu, ks = W.config("C6")
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    N = math.factorial(12)
    keys = torch.zeros(N, dtype=torch.int64, device="cuda")
    st = ctx.rk_eval_range(0, N, 0, keys_dev=keys)
    assert st.evaluated == N
    assert O.simulate(gpu, ks, O.unrank(st.argmin, 12)).key == st.key_min
    assert O.simulate(gpu, ks, O.unrank(st.argmax, 12)).key == st.key_max
    rng = np.random.default_rng(6)
    idx = rng.integers(0, N, 2000)
    got = keys[torch.from_numpy(idx).cuda()].cpu().numpy().view(np.uint64)
    for i, k in zip(idx.tolist(), got.tolist()):
        assert k == O.simulate(gpu, ks, O.unrank(i, 12)).key, i
    _, _, hidx, _ = ctx.rk_heuristic_order()
    _check_best(ctx, gpu, ks, st.key_min, st.argmin, seeds=(hidx,))


def test_forced_runs_state_equals_register_state(monkeypatch):
    """RK_FORCE_RUNS=1 routes every S through the run-length state: same keys,
    partitions, statistics and optimum as the oracle on C2/C3 (S' = 1) and on
    random shapes with S' in 2..32."""
    monkeypatch.setenv("RK_FORCE_RUNS", "1")
    c = rk.Context(0)
    try:
        for name in ("C2", "C3"):
            gpu, ks = W.config(name)
            g = _gold(f"{name.lower()}_oracle.json")
            c.rk_set_gpu_params(gpu)
            c.rk_set_kernels(ks)
            st = c.rk_eval_range(0, math.factorial(len(ks)), g["cand_key"])
            assert list(st.as_tuple()) == [g["stats"][f] for f in
                                           ("key_min", "key_max", "argmin", "argmax", "n_lt", "n_eq", "n_gt",
                                            "evaluated")]
            _check_best(c, gpu, ks, g["stats"]["key_min"], g["stats"]["argmin"])
        for gpu in GPUS:
            for ks in W.random_small_sets(0xF0 + gpu[0], 4, 3, 7, gpu=gpu):
                if not all(W.feasible(gpu, k) for k in ks):
                    continue
                try:
                    c.rk_set_gpu_params(gpu)
                    c.rk_set_kernels(ks)
                except rk.RkError as e:
                    assert e.status == rk.RK_EUNSUPPORTED
                    continue
                check_full_space(c, gpu, ks, bins=(3,))
                for q in range(3):
                    o = O.unrank(q * 7 % math.factorial(len(ks)), len(ks))
                    r = O.simulate(gpu, ks, o)
                    assert c.rk_simulate_order(o) == (r.rounds, r.key)
        # cursor-per-kernel reading through the run-length state
        gpu, ks = W.config("C2")
        check_full_space(c, list(gpu) + [1], ks, bins=(16,))
        # batch path (C5 subset) through the run-length state
        g5 = _gold("c5_oracle.json")
        sets = W.c5_sets(64)
        c.rk_set_gpu_params(W.GTX580)
        res = c.rk_eval_batch(sets, [s["cand_index"] for s in g5["sets"][:64]])
        for q in range(64):
            assert list(res[q][0].as_tuple()) == g5["sets"][q]["stats"] and res[q][1] == g5["sets"][q]["cand_key"]
    finally:
        c.close()


# ---- suffix memoisation: memoised keys == direct keys == oracle ----
def _direct_ctx(monkeypatch, var="RK_NO_MEMO"):
    monkeypatch.setenv(var, "1")
    c = rk.Context(0)
    monkeypatch.delenv(var)
    return c


def test_memo_plan_info(ctx, monkeypatch):
    gpu, ks = W.config("C4")
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    on, P, nodes = ctx.rk_memo_info()
    assert on and P == 7 and nodes[0] == 1 and nodes[1] == 12
    # distinct nodes never exceed the number of prefixes n!/(n-j)!
    assert all(nodes[j] <= math.factorial(12) // math.factorial(12 - j) for j in range(P + 1))
    ctx.rk_set_kernels(ks[:5])  # n < 6: direct
    assert ctx.rk_memo_info()[0] is False
    d = _direct_ctx(monkeypatch)
    try:
        d.rk_set_gpu_params(gpu)
        d.rk_set_kernels(ks)
        assert d.rk_memo_info()[0] is False
    finally:
        d.close()


def test_memo_keys_equal_direct_keys(monkeypatch):
    """Every key and statistic of the memoised path equals the direct evaluation's
    (itself pinned to the oracle) on C2-C4 and random sets n = 6..9 over 7 GPU
    shapes (memoisation forced on), on full spaces and on ragged ranges."""
    d = _direct_ctx(monkeypatch)
    ctx = _direct_ctx(monkeypatch, "RK_FORCE_MEMO")
    try:
        cases = [W.config(c) for c in ("C2", "C3", "C4")]
        # huge per-block work: suffix rows span >= 2^32 (the 64-bit decode path)
        for ks in W.random_small_sets(0x91DE, 4, 7, 8):
            wide = [(k[0], k[1], k[2], k[3], min(k[4] * 797, (1 << 32) - 1), min(k[5] * 787, (1 << 32) - 1)) for k in ks]
            if W.key_bound(W.GTX580, wide) < (1 << 62):
                cases.append((W.GTX580, wide))
        for gi, gpu in enumerate(GPUS):
            for ks in W.random_small_sets(0xDEC0 + gi, 6, 6, 9, gpu=gpu):
                if all(W.feasible(gpu, k) for k in ks):
                    cases.append((gpu, ks))
        checked = 0
        for gpu, ks in cases:
            try:
                ctx.rk_set_gpu_params(gpu)
                ctx.rk_set_kernels(ks)
            except rk.RkError as e:
                assert e.status == rk.RK_EUNSUPPORTED
                continue
            d.rk_set_gpu_params(gpu)
            d.rk_set_kernels(ks)
            N = math.factorial(len(ks))
            cand = O.simulate(gpu, ks, O.unrank(N // 3, len(ks))).key
            rng = np.random.default_rng(len(ks) * 7 + checked)
            ranges = [(0, N)]
            for _ in range(3):
                f0 = int(rng.integers(0, N))
                ranges.append((f0, int(rng.integers(1, min(50000, N - f0) + 1))))
            for first, count in ranges:
                k1 = torch.zeros(count, dtype=torch.int64, device="cuda")
                k2 = torch.zeros(count, dtype=torch.int64, device="cuda")
                s1 = ctx.rk_eval_range(first, count, cand, keys_dev=k1)
                s2 = d.rk_eval_range(first, count, cand, keys_dev=k2)
                assert s1.as_tuple() == s2.as_tuple(), (gpu, ks, first, count)
                assert torch.equal(k1, k2)
                # the two-pass API with the fused histogram == histogram of the direct keys
                for B in (7, 256):
                    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
                    cd = torch.tensor([cand], dtype=torch.int64, device="cuda")
                    h1 = torch.zeros(B, dtype=torch.int64, device="cuda")
                    ctx.rk_sweep_pass1_async(first, count, cd, rec, None)
                    ctx.rk_sweep_pass2_async(first, count, cd, rec, B, h1, None, rec)
                    h2 = torch.zeros(B, dtype=torch.int64, device="cuda")
                    d.rk_histogram(k2, count, s2.key_min, s2.key_max, B, h2)
                    torch.cuda.synchronize()
                    assert torch.equal(h1, h2), (first, count, B)
                    assert rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes())).as_tuple() \
                        == s2.as_tuple()
            if ctx.rk_memo_info()[0]:
                checked += 1
        assert checked >= 10
    finally:
        d.close()
        ctx.close()


def test_memo_two_pass_api_and_fused_histogram(ctx):
    """rk_sweep_pass1/2 (the bench step): record, keys and histogram equal the
    oracle golden for C4; pass 2 without keys gives the same histogram."""
    gpu, ks = W.config("C4")
    g = _gold("c4_oracle.json")
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    N = math.factorial(12)
    cand = torch.tensor([g["cand_key"]], dtype=torch.int64, device="cuda")
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    keys = torch.zeros(N, dtype=torch.int64, device="cuda")
    hist = torch.zeros(256, dtype=torch.int64, device="cuda")
    ctx.rk_sweep_pass1_async(0, N, cand, rec, keys)
    ctx.rk_sweep_pass2_async(0, N, cand, rec, 256, hist, keys, rec)
    torch.cuda.synchronize()
    st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
    assert list(st.as_tuple()) == [g["stats"][f] for f in
                                   ("key_min", "key_max", "argmin", "argmax", "n_lt", "n_eq", "n_gt", "evaluated")]
    assert hist.cpu().tolist() == g["hist"]
    h2 = torch.zeros(256, dtype=torch.int64, device="cuda")
    ctx.rk_histogram(keys, N, st.key_min, st.key_max, 256, h2)
    assert torch.equal(hist, h2)
    rec2 = torch.zeros(8, dtype=torch.int64, device="cuda")
    h3 = torch.zeros(256, dtype=torch.int64, device="cuda")
    ctx.rk_sweep_pass1_async(0, N, cand, rec2, None)
    ctx.rk_sweep_pass2_async(0, N, cand, rec2, 256, h3, None, rec2)
    torch.cuda.synchronize()
    assert torch.equal(rec2, rec) and torch.equal(h3, hist)
    # order statistics over the memoised keys == the oracle's
    ranks = sorted(int(r) for r in g["order_stats"])
    got = ctx.rk_select_keys(keys, N, st.key_min, st.key_max, ranks)
    assert got == [g["order_stats"][str(r)] for r in ranks]


def test_memo_run_length_nodes_vs_oracle_and_direct(monkeypatch):
    """Memoisation over run-length SM states (S' > 32, e.g. the B200 preset):
    full spaces vs the oracle (memoisation forced on small sets) and C6's every
    key vs the direct run-length kernel."""
    fm = _direct_ctx(monkeypatch, "RK_FORCE_MEMO")
    d = _direct_ctx(monkeypatch)
    try:
        done = 0
        for gi, gpu in enumerate(BIG_GPUS[:3]):
            rng = W.SplitMix64(0x7A11 + gi)
            for q in range(3):
                ks = W.gen_b200(rng, 6 + q % 2, gpu=gpu) if gpu[3] >= 64 else \
                    W.random_small_sets(0x7A11 + gi * 7 + q, 1, 6, 7, gpu=gpu)[0]
                if not all(W.feasible(gpu, k) for k in ks):
                    continue
                fm.rk_set_gpu_params(gpu)
                fm.rk_set_kernels(ks)
                assert fm.rk_memo_info()[0]
                check_full_space(fm, gpu, ks, bins=(9,))
                done += 1
        assert done >= 5
        gpu, ks = W.config("C6")
        N = math.factorial(12)
        for c in (fm, d):
            c.rk_set_gpu_params(gpu)
            c.rk_set_kernels(ks)
        assert fm.rk_memo_info()[0] and not d.rk_memo_info()[0]
        k1 = torch.zeros(N, dtype=torch.int64, device="cuda")
        k2 = torch.zeros(N, dtype=torch.int64, device="cuda")
        s1 = fm.rk_eval_range(0, N, 0, keys_dev=k1)
        s2 = d.rk_eval_range(0, N, 0, keys_dev=k2)
        assert s1.as_tuple() == s2.as_tuple() and torch.equal(k1, k2)
    finally:
        fm.close()
        d.close()


def test_memo_plan_switching_sets_in_one_context(ctx):
    """Plans are kept only for byte-identical tables: alternating kernel sets (and
    GPU parameters) in one context give the oracle goldens every time."""
    c2, c3 = _gold("c2_oracle.json"), _gold("c3_oracle.json")
    fields = ("key_min", "key_max", "argmin", "argmax", "n_lt", "n_eq", "n_gt", "evaluated")
    for name, gold in (("C2", c2), ("C3", c3), ("C2", c2), ("C3", c3)):
        gpu, ks = W.config(name)
        ctx.rk_set_gpu_params(gpu)
        ctx.rk_set_kernels(ks)
        st = ctx.rk_eval_range(0, math.factorial(len(ks)), gold["cand_key"])
        assert list(st.as_tuple()) == [gold["stats"][f] for f in fields], name
    # the same kernels under the cursor-per-kernel reading (different tables) and back
    gpu, ks = W.config("C2")
    ost, _ = O.sweep(list(gpu) + [1], ks, cand_key=c2["cand_key"], threads=NCPU)
    ctx.rk_set_gpu_params(list(gpu) + [1])
    ctx.rk_set_kernels(ks)
    assert ctx.rk_eval_range(0, 40320, c2["cand_key"]).as_tuple() == ost.as_tuple()
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    assert list(ctx.rk_eval_range(0, 40320, c2["cand_key"]).as_tuple()) == [c2["stats"][f] for f in fields]


def test_memo_n14_full_space_vs_branch_and_bound_and_oracle(ctx):
    """14! = 8.7e10 orders: the memoised full-space statistics
    agree with the branch-and-bound optimum, the oracle re-simulates the extremes,
    and sampled orders lie within them."""
    n = 14
    ks = W.gen_g(W.SplitMix64(W.SEED_BASE + 1000 * n), n)
    ctx.rk_set_gpu_params(W.GTX580)
    ctx.rk_set_kernels(ks)
    assert ctx.rk_memo_info()[0]
    N = math.factorial(n)
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    cd = torch.zeros(1, dtype=torch.int64, device="cuda")
    ctx.rk_eval_range_async(0, N, cd, rec)
    torch.cuda.synchronize()
    st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
    assert st.evaluated == N
    _, _, hidx, _ = ctx.rk_heuristic_order()
    _, idx, key, _ = ctx.rk_best_order(hidx)
    assert (key, idx) == (st.key_min, st.argmin)
    assert O.simulate(W.GTX580, ks, O.unrank(st.argmin, n)).key == st.key_min
    assert O.simulate(W.GTX580, ks, O.unrank(st.argmax, n)).key == st.key_max
    rng = np.random.default_rng(14)
    for i in rng.integers(0, N, 200).tolist():
        assert st.key_min <= O.simulate(W.GTX580, ks, O.unrank(i, n)).key <= st.key_max


def test_device_algorithm1_unspecified_branches_hand_golden(ctx):
    """rk_heuristic_batch (device Algorithm 1) on the hand-derived branch goldens:
    ties, no feasible pair, lone kernel,
    equal-shm insertion, bonus clamp."""
    g = _gold("alg1_branches.json")
    ctx.rk_set_gpu_params(g["gpu"])
    for case in g["cases"]:
        orders, idx = ctx.rk_heuristic_batch([case["kernels"]])
        assert orders[0] == case["order"], case["name"]
        assert idx[0] == O.rank(case["order"])
        # the same set as a whole batch of copies (one thread per set)
        orders, _ = ctx.rk_heuristic_batch([case["kernels"]] * 37)
        assert all(o == case["order"] for o in orders)


F3 = _gold("readings_f3.json")
POLICY_FLAGS = [2, 3, 4, 5, 6, 7]  # strict RR (2) / skip-ahead (4), with and without cursor-per-kernel (1)


def test_policy_readings_hand_golden_through_abi(ctx):
    """strict round robin and skip-ahead (rk.h RK_FLAG_STRICT_RR /
    RK_FLAG_SKIP_AHEAD) reproduce the hand traces of tests/golden/readings_f3.json:
    round partitions and T of every case and reading, and the full space of each
    case against the oracle."""
    for case in F3["cases"]:
        for flags, want in case["readings"].items():
            gpu = list(case["gpu"]) + [int(flags)]
            ctx.rk_set_gpu_params(gpu)
            ctx.rk_set_kernels(case["kernels"])
            rounds, key = ctx.rk_simulate_order(case["order"])
            assert rounds == want["rounds"] and key == want["T"] * case["gpu"][6], (case["name"], flags)
            check_full_space(ctx, gpu, case["kernels"], bins=(5,))


@pytest.mark.parametrize("flags", POLICY_FLAGS)
def test_policy_full_spaces_vs_oracle(ctx, flags):
    """Per-order policy kernels vs the block-by-block oracle: every key, the
    statistics and histograms on C1 (W4 + random sets), C2 and random sets
    over the GPU shapes (symmetry reduction on, S' <= 32)."""
    for ks in [W.W4] + W.c1_random_sets()[:16]:
        check_full_space(ctx, list(W.GTX580) + [flags], ks, bins=(3,))
    done = 0
    for gi, gpu in enumerate(GPUS):
        for ks in W.random_small_sets(0xF300 + 16 * flags + gi, 6, 2, 7, gpu=gpu):
            if not all(W.feasible(gpu, k) for k in ks):
                continue
            ctx.rk_set_gpu_params(list(gpu) + [flags])
            ctx.rk_set_kernels(ks)
            check_full_space(ctx, list(gpu) + [flags], ks, bins=(7,))
            done += 1
    assert done >= 10
    gpu, ks = W.config("C2")
    check_full_space(ctx, list(gpu) + [flags], ks, bins=(256,))


@pytest.mark.parametrize("flags", [2, 4, 6])
def test_policy_c3_full_space_and_c4_samples_vs_oracle(ctx, flags):
    """C3 (3.6M orders) element by element; C4 (12!) on 20,000 random indices
    plus both ends (the oracle computes them one by one), under each policy."""
    gpu, ks = W.config("C3")
    check_full_space(ctx, list(gpu) + [flags], ks, bins=(256,))
    gpu, ks = W.config("C4")
    g = list(gpu) + [flags]
    ctx.rk_set_gpu_params(g)
    ctx.rk_set_kernels(ks)
    N = math.factorial(12)
    rng = np.random.default_rng(flags)
    sample = np.concatenate([rng.integers(0, N, 20000), np.arange(0, 500), np.arange(N - 500, N)]).astype(np.uint64)
    want = O.keys_of(g, ks, sample, threads=NCPU)
    idx = torch.from_numpy(sample.view(np.int64)).cuda()
    keys = torch.empty(N, dtype=torch.int64, device="cuda")
    st = ctx.rk_eval_range(0, N, 0, keys_dev=keys)
    assert st.evaluated == N and st.n_gt == N
    assert np.array_equal(keys[idx].cpu().numpy().view(np.uint64), want)
    assert st.key_min == int(keys.min().item()) and st.key_max == int(keys.max().item())


def test_policy_batch_and_public_api_vs_oracle(ctx):
    """C5-shaped batch under each policy (per-set stats vs the oracle's per-set
    sweep with Algorithm 1's candidate) and the public Sweeper report."""
    from paper_1511_07983_b200.sweep import Sweeper
    sets = W.c5_sets(24)
    for flags in (2, 4, 6):
        g = list(W.GTX580) + [flags]
        ctx.rk_set_gpu_params(g)
        res = ctx.rk_eval_batch(sets)
        want = O.sweep_sets(g, sets, threads=NCPU)
        for (st, ck), (ost, oidx, ock) in zip(res, want):
            assert st.as_tuple() == ost.as_tuple() and ck == ock
        gpu, ks = W.config("C3")
        rep = Sweeper(list(gpu) + [flags]).run(ks)
        cand = O.simulate(list(gpu) + [flags], ks, O.heuristic(gpu, ks)[0]).key
        ost, okeys = O.sweep(list(gpu) + [flags], ks, cand_key=cand, threads=NCPU, keys=True)
        assert (rep.best_key, rep.worst_key, rep.best_index, rep.worst_index, rep.n_lt, rep.n_eq, rep.n_gt) == \
            (ost.key_min, ost.key_max, ost.argmin, ost.argmax, ost.n_lt, ost.n_eq, ost.n_gt)
        assert rep.cand_key == cand
        assert rep.hist == O.histogram(okeys, ost.key_min, ost.key_max, 256)


def test_policy_unsupported_paths_fail_loudly(ctx):
    """Policies run on the per-order kernels only: S' > 32, branch and bound,
    compact keys and the fused histogram return RK_EUNSUPPORTED."""
    gpu, ks = W.config("C6")
    ctx.rk_set_gpu_params(list(gpu) + [rk.RK_FLAG_STRICT_RR])
    with pytest.raises(rk.RkError) as e:
        ctx.rk_set_kernels(ks)
    assert e.value.status == rk.RK_EUNSUPPORTED
    gpu, ks = W.config("C2")
    ctx.rk_set_gpu_params(list(gpu) + [rk.RK_FLAG_SKIP_AHEAD])
    ctx.rk_set_kernels(ks)
    assert ctx.rk_memo_info()[0] is False
    with pytest.raises(rk.RkError) as e:
        ctx.rk_best_order()
    assert e.value.status == rk.RK_EUNSUPPORTED
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    k32 = torch.empty(40320, dtype=torch.int32, device="cuda")
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    with pytest.raises(rk.RkError) as e:
        ctx.rk_eval_range32_async(0, 40320, None, rec, k32, 0, ovf)
    assert e.value.status == rk.RK_EUNSUPPORTED


def test_memo_hash_tables_race_audit(monkeypatch):
    """Race evidence for the lock-free memo hash tables (CAS claim, release
    publish, acquire probe; compute-sanitizer is not available on this pool):
    after every one of many rebuilds — C4 (the bench set) and random sets over
    the GPU shapes with memoisation forced — the device audit (rk_memo_audit)
    finds no BUSY slot, no lost publish, no duplicate state, no bad transition,
    per-level counts equal to the plan's, and the step's record and keys are
    bit-identical to the first build's (itself equal to the oracle: the C4
    golden test and test_memo_keys_equal_direct_keys)."""
    ctx = _direct_ctx(monkeypatch, "RK_FORCE_MEMO")
    try:
        cases = [W.config("C4"), W.config("C3"), W.config("C2")]
        for gi, gpu in enumerate(GPUS):
            for ks in W.random_small_sets(0xA0D1 + gi, 2, 8, 9, gpu=gpu):
                if all(W.feasible(gpu, k) for k in ks):
                    cases.append((gpu, ks))
        audited = 0
        for ci, (gpu, ks) in enumerate(cases):
            try:
                ctx.rk_set_gpu_params(gpu)
                ctx.rk_set_kernels(ks)
            except rk.RkError as e:
                assert e.status == rk.RK_EUNSUPPORTED
                continue
            if not ctx.rk_memo_info()[0]:
                continue
            N = math.factorial(len(ks))
            reps = 12 if ci == 0 else 4
            keys = torch.empty(N, dtype=torch.int64, device="cuda")
            cand = torch.zeros(1, dtype=torch.int64, device="cuda")
            rec = torch.zeros(8, dtype=torch.int64, device="cuda")
            first = None
            for r in range(reps):
                ctx.rk_sweep_pass1_async(0, N, cand, rec, keys)
                ctx.rk_sweep_pass2_async(0, N, cand, None, 0, None, keys, rec)
                bad = ctx.rk_memo_audit()
                assert bad[:7] == [0] * 7, (ci, r, bad)
                assert bad[7] > sum(ctx.rk_memo_info()[2][1:])  # levels 1..P + the level-(P+1) nodes
                h = (rec.cpu().clone(), torch.sum(keys * 7919 + 1).item(), keys[::9973].cpu())
                if first is None:
                    first = h
                else:
                    assert torch.equal(h[0], first[0]) and h[1] == first[1] and torch.equal(h[2], first[2])
            audited += 1
        assert audited >= 6
    finally:
        ctx.close()


def test_memo_compact_key_stream_c4_and_overflow(ctx):
    """rk_sweep_pass2_32_async (the bench's key stream with exact u32 offsets
    from the set's lower bound): on C4 every stored offset + base
    equals the u64 key of the same step, the record and histogram equal the
    oracle golden, 10^5 sampled keys equal the oracle's; on a set whose keys
    span >= 2^32 the overflow flag is raised."""
    g = _gold("c4_oracle.json")
    gpu, ks = W.config("C4")
    ctx.rk_set_gpu_params(gpu)
    ctx.rk_set_kernels(ks)
    N = math.factorial(12)
    base = ctx.rk_key_lower_bound()
    cand = torch.tensor([g["cand_key"]], dtype=torch.int64, device="cuda")
    rec = torch.zeros(8, dtype=torch.int64, device="cuda")
    hist = torch.zeros(256, dtype=torch.int64, device="cuda")
    k32 = torch.empty(N, dtype=torch.int32, device="cuda")
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.rk_sweep_pass1_async(0, N, cand, rec, None)
    ctx.rk_sweep_pass2_32_async(0, N, cand, rec, 256, hist, k32, base, ovf, rec)
    k64 = torch.empty(N, dtype=torch.int64, device="cuda")
    rec2 = torch.zeros(8, dtype=torch.int64, device="cuda")
    ctx.rk_sweep_pass1_async(0, N, cand, rec2, k64)
    ctx.rk_sweep_pass2_async(0, N, cand, rec2, 0, None, k64, rec2)
    torch.cuda.synchronize()
    assert int(ovf.item()) == 0
    st = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
    assert list(st.as_tuple()) == [g["stats"][f] for f in
                                   ("key_min", "key_max", "argmin", "argmax", "n_lt", "n_eq", "n_gt", "evaluated")]
    assert hist.cpu().tolist() == g["hist"] and torch.equal(rec, rec2)
    assert torch.equal((k32.to(torch.int64) & 0xFFFFFFFF) + base, k64)
    rng = np.random.default_rng(32)
    sample = rng.integers(0, N, 100000).astype(np.uint64)
    got = (k32[torch.from_numpy(sample.view(np.int64)).cuda()].to(torch.int64) & 0xFFFFFFFF).cpu().numpy() + base
    assert np.array_equal(got.astype(np.uint64), O.keys_of(gpu, ks, sample, threads=NCPU))
    # ragged sub-range (unaligned first, partial runs at both ends)
    f0, c0 = 1234567, 765433
    ovf.zero_()
    ctx.rk_sweep_pass1_async(f0, c0, cand, rec, None)
    ctx.rk_sweep_pass2_32_async(f0, c0, cand, rec, 0, None, k32, base, ovf, rec)
    torch.cuda.synchronize()
    assert int(ovf.item()) == 0
    assert torch.equal((k32[:c0].to(torch.int64) & 0xFFFFFFFF) + base, k64[f0:f0 + c0])
    # keys spanning >= 2^32 above the bound: the flag
    wide = None
    for ks2 in W.random_small_sets(0x91DE, 8, 7, 8):
        w = [(k[0], k[1], k[2], k[3], min(k[4] * 797, (1 << 32) - 1), min(k[5] * 787, (1 << 32) - 1)) for k in ks2]
        if W.key_bound(W.GTX580, w) < (1 << 62):
            wide = w
            break
    ctx.rk_set_kernels(wide)
    if ctx.rk_memo_info()[0]:
        n2 = math.factorial(len(wide))
        b2 = ctx.rk_key_lower_bound()
        ovf.zero_()
        ctx.rk_sweep_pass1_async(0, n2, cand, rec, None)
        ctx.rk_sweep_pass2_32_async(0, n2, cand, rec, 0, None, k32, b2, ovf, rec)
        torch.cuda.synchronize()
        st2 = rk.Stats.from_c(rk.rk_stats.from_buffer_copy(rec.cpu().numpy().tobytes()))
        assert int(ovf.item()) == (1 if st2.key_max - b2 >= (1 << 32) else 0)


@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_fig1_ranking_curve_and_median_gain_vs_oracle_golden(cfg):
    """Fig. 1's ranking curve as deciles of the sorted keys and
    the §6 median-sequence comparison: the public report's exact
    order statistics equal the oracle golden's (sorted full oracle run)."""
    from paper_1511_07983_b200.sweep import Sweeper
    g = _gold(f"{cfg.lower()}_oracle.json")
    gpu, ks = W.config(cfg)
    for compact in (False, True):
        rep = Sweeper(gpu, compact_keys=compact).run(ks, median=True, curve_points=11)
        assert rep.median_key == g["order_stats"][str(g["median_rank"])]
        assert [str(r) for r, _ in rep.ranking_curve] == [r for r in sorted(g["order_stats"], key=int)
                                                          if int(r) != g["median_rank"]]
        assert all(k == g["order_stats"][str(r)] for r, k in rep.ranking_curve)
        assert rep.gain_over_median_pct == 100.0 * (rep.median_key - g["cand_key"]) / g["cand_key"]


def test_strict_round_robin_on_the_memoised_and_bnb_paths(monkeypatch):
    """RK_FLAG_STRICT_RR keeps L4's prefix state, so it runs on the memoised
    step (forced on), the direct kernel and branch and bound: every key and
    statistic vs the oracle on C2, C3 and random sets over the GPU shapes,
    with and without the cursor-per-kernel reading; the optimum by branch and
    bound equals the full sweep's."""
    ctx = _direct_ctx(monkeypatch, "RK_FORCE_MEMO")
    try:
        cases = [W.config("C2"), W.config("C3")]
        for gi, gpu in enumerate(GPUS[:5]):
            for ks in W.random_small_sets(0x5A5A + gi, 3, 6, 8, gpu=gpu):
                if all(W.feasible(gpu, k) for k in ks):
                    cases.append((gpu, ks))
        memo_checked = 0
        for flags in (rk.RK_FLAG_STRICT_RR, rk.RK_FLAG_STRICT_RR | rk.RK_FLAG_CURSOR_PER_KERNEL):
            for gpu, ks in cases:
                g = list(gpu) + [flags]
                try:
                    ctx.rk_set_gpu_params(g)
                    ctx.rk_set_kernels(ks)
                except rk.RkError as e:
                    assert e.status == rk.RK_EUNSUPPORTED
                    continue
                memo_checked += ctx.rk_memo_info()[0]
                st = check_full_space(ctx, g, ks, bins=(32,))
                _, idx, key, _ = ctx.rk_best_order()
                assert (key, idx) == (st.key_min, st.argmin)
        assert memo_checked >= 8
    finally:
        ctx.close()


def test_memoised_batch_vs_oracle_and_direct(ctx, monkeypatch):
    """rk_eval_batch's memoised kernel (6 <= n <= 9 on S' <= 2: runs sharing an
    equal prefix state share one 120-key suffix row) equals the oracle's per-set
    sweep for n = 6..8 under every register-state reading, sets with repeated
    kernels (many equal states) included, and the direct batch kernel
    (RK_NO_MEMO=1) on 256 C5 sets; one launch per S' group (+ the candidate keys)."""
    direct = _direct_ctx(monkeypatch)
    try:
        for n in (6, 7, 8):
            sets = W.c5_sets(12, n=n)
            sets += [[s[0]] * 2 + list(s[2:]) for s in sets[:4]]  # two identical kernels
            sets += [[s[1]] * n for s in sets[:2]]                 # all identical
            for flags in (0, 1, 2, 3):
                g = list(W.GTX580) + [flags]
                ctx.rk_set_gpu_params(g)
                res = ctx.rk_eval_batch(sets)
                assert ctx.launches <= 3  # candidate keys + one launch per S' group
                want = O.sweep_sets(g, sets, threads=NCPU)
                for (st, ck), (ost, oidx, ock) in zip(res, want):
                    assert st.as_tuple() == ost.as_tuple() and ck == ock
        sets = W.c5_sets(256)
        for flags in (0, 2):
            g = list(W.GTX580) + [flags]
            ctx.rk_set_gpu_params(g)
            direct.rk_set_gpu_params(g)
            a = ctx.rk_eval_batch(sets)
            b = direct.rk_eval_batch(sets)
            assert direct.launches > ctx.launches
            assert [(s.as_tuple(), k) for s, k in a] == [(s.as_tuple(), k) for s, k in b]
            c = ctx.rk_eval_batch(np.array(sets, dtype=np.int64))  # (sets, n, 6) array input
            assert [(s.as_tuple(), k) for s, k in c] == [(s.as_tuple(), k) for s, k in a]
    finally:
        direct.close()


def test_memoised_batch_edge_cases(ctx):
    """The memoised batch kernel on one set, on given candidate indices (first,
    last and a middle order), and on n = 9 sets against the oracle directly."""
    F9 = math.factorial(9)
    ctx.rk_set_gpu_params(W.GTX580)
    sets = W.c5_sets(3)
    want = O.sweep_sets(list(W.GTX580), sets, threads=NCPU)
    one = ctx.rk_eval_batch(sets[:1])
    assert one[0][0].as_tuple() == want[0][0].as_tuple() and one[0][1] == want[0][2]
    for idx in ([0, F9 - 1, 12345], [F9 - 1, 0, F9 // 2]):
        res = ctx.rk_eval_batch(sets, cand_index=idx)
        for q, (st, ck) in enumerate(res):
            okey = O.simulate(list(W.GTX580), sets[q], O.unrank(idx[q], 9)).key
            ost = O.sweep(list(W.GTX580), sets[q], cand_key=okey, threads=NCPU)
            ost = ost[0] if isinstance(ost, tuple) else ost
            assert ck == okey and st.as_tuple() == ost.as_tuple()
