"""Property pins of the oracle: closed forms, invariants the paper states,
brute force on tiny inputs, and an independent trace checker of the
placement rules.
"""
import bisect
import itertools
import math
from collections import Counter
from fractions import Fraction

import pytest

import oracle as O
from paper_1511_07983_b200 import workloads as W

G = W.GTX580


def demand(k):
    return (k[2] * k[1], k[3], (k[1] + 31) // 32, 1)


def exact_lower_bound(gpu, ks):
    """T >= max(sum I, R_B * sum M), as den-scaled integers."""
    sI = sum(k[0] * k[4] for k in ks)
    sM = sum(k[0] * k[5] for k in ks)
    return max(gpu[6] * sI, gpu[5] * sM)


def check_trace(gpu, ks, order, trace, rounds):
    """Independent verifier of the placement rules on the oracle's trace."""
    S = gpu[0]
    caps = (gpu[1], gpu[2], gpu[3], gpu[4])
    blocks = [k for k in order for _ in range(ks[k][0])]
    assert len(blocks) == len(trace)
    used = [[0, 0, 0, 0] for _ in range(S)]
    cur_round, cursor = 0, 0
    placed = [[0] * len(ks)]

    def fits(s, d):
        return all(used[s][x] + d[x] <= caps[x] for x in range(4))

    for b, (k, (r, s)) in enumerate(zip(blocks, trace)):
        d = demand(ks[k])
        if r != cur_round:
            assert r == cur_round + 1
            # maximality: the block fits no SM of the closed round
            assert not any(fits(x, d) for x in range(S))
            used = [[0, 0, 0, 0] for _ in range(S)]
            cur_round, cursor = r, 0
            placed.append([0] * len(ks))
        # first fit scanning ring-wise from the cursor (reading L4)
        x = cursor
        while x != s:
            assert not fits(x, d), (b, x, s)
            x = (x + 1) % S
        assert fits(s, d)
        for q in range(4):
            used[s][q] += d[q]
        cursor = (s + 1) % S
        placed[r][k] += 1
    assert placed == rounds
    # conservation
    for i, k in enumerate(ks):
        assert sum(p[i] for p in rounds) == k[0]


def test_two_nsm_blocks_give_two_per_sm():
    # "if there are 2N_SM thread blocks in total, each SM will be assigned two"
    ks = [(16, 128, 16, 1024, 311, 100), (16, 64, 16, 2048, 1110, 100)]
    for order in ([0, 1], [1, 0]):
        r = O.simulate(G, ks, order, trace=True)
        assert len(r.rounds) == 1
        per_sm = [0] * 16
        for _, s in r.trace:
            per_sm[s] += 1
        assert per_sm == [2] * 16


def test_spec_place_blocks_partial_kernel_example():
    # A warps-footprint 24 then B warps 32 on N_warp_SM=48 -> A fully resident,
    # B partially placed (24 warp slots' worth), remainder in round 2.
    ks = [(16, 768, 1, 0, 10, 1), (32, 512, 1, 0, 10, 1)]  # A: 24 warps/blk; B: 16 warps/blk, 2 blk/SM
    r = O.simulate(G, ks, [0, 1])
    assert r.rounds == [[16, 16], [0, 16]]


@pytest.mark.parametrize("seed", range(40))
def test_total_blocks_le_nsm_single_round_closed_form(seed):
    # total blocks <= N_SM -> kernels share no SM, order irrelevant
    rng = W.SplitMix64(1000 + seed)
    n = 1 + rng.below(4)
    ks = []
    left = 16
    for i in range(n):
        t = 1 + rng.below(max(1, left - (n - i - 1)))
        left -= t
        tpb = rng.choice((64, 128, 256, 512, 1024))
        rn = rng.choice(W.RN_MEM + W.RN_CMP)
        c = 1 + rng.below(50)
        ks.append((t, tpb, rng.choice((16, 32)), rng.choice((0, 8192, 49152)), rn * c, 100 * c))
    want = exact_lower_bound(G, ks)  # one round: max(den*sum I, num*sum M)
    for order in itertools.permutations(range(n)):
        r = O.simulate(G, ks, list(order))
        assert len(r.rounds) == 1 and r.key == want


@pytest.mark.parametrize("classes", ["mem", "cmp"])
def test_same_side_theorem(classes):
    # all R_i on one side of R_B -> T = sum I (or R_B sum M) for every order
    sets = W.random_small_sets(0xB1 if classes == "mem" else 0xB2, 12, 3, 5, classes=classes)
    for ks in sets:
        sI = sum(k[0] * k[4] for k in ks)
        sM = sum(k[0] * k[5] for k in ks)
        want = G[6] * sI if classes == "cmp" else G[5] * sM
        s, keys = O.sweep(G, ks, keys=True)
        assert s.key_min == s.key_max == want


@pytest.mark.parametrize("seed", range(6))
def test_identical_kernels_differing_in_nblocks_are_order_invariant(seed):
    # identical kernels differing only in N_tblk -> order does not matter
    rng = W.SplitMix64(77 + seed)
    tpb = rng.choice((64, 128, 256, 512))
    rpt = rng.choice((16, 24, 32))
    shm = rng.choice((0, 4096, 12288, 24576))
    c = 1 + rng.below(40)
    rn = rng.choice(W.RN_MEM + W.RN_CMP)
    n = 5
    ks = [(rng.choice(W.GRID), tpb, rpt, shm, rn * c, 100 * c) for _ in range(n)]
    s, _ = O.sweep(G, ks)
    assert s.key_min == s.key_max


def _brute(gpu, ks, cand):
    keys = []
    for p in itertools.permutations(range(len(ks))):
        keys.append(O.simulate(gpu, ks, list(p)).key)
    kmin = min(keys)
    kmax = max(keys)
    return dict(key_min=kmin, key_max=kmax, argmin=keys.index(kmin), argmax=keys.index(kmax),
                n_lt=sum(k < cand for k in keys), n_eq=sum(k == cand for k in keys),
                n_gt=sum(k > cand for k in keys), evaluated=len(keys)), keys


@pytest.mark.parametrize("seed", range(8))
def test_sweep_stats_equal_brute_force_over_library_permutations(seed):
    sets = W.random_small_sets(0x5EED00 + seed, 3, 3, 6)
    for ks in sets:
        srt = sorted(O.simulate(G, ks, list(p)).key for p in itertools.permutations(range(len(ks))))
        cand = srt[len(srt) // 3]
        want, keys = _brute(G, ks, cand)
        s, skeys = O.sweep(G, ks, cand_key=cand, threads=3, keys=True)
        assert [int(k) for k in skeys] == keys
        for f, v in want.items():
            assert getattr(s, f) == v, f
        assert s.n_lt + s.n_eq + s.n_gt == math.factorial(len(ks))
        # lower bound and the naive double cross-check (O5, 1e-12)
        assert s.key_min >= exact_lower_bound(G, ks)
        assert s.max_rel_err <= 1e-12


@pytest.mark.parametrize("seed", range(6))
def test_placement_trace_rules_and_conservation(seed):
    sets = W.random_small_sets(0x7ACE + seed, 4, 2, 7)
    gpus = [G, (8, 65536, 102400, 64, 16, 7, 2), (3, 16384, 16384, 32, 4, 5, 1)]
    rng = W.SplitMix64(seed)
    for ks in sets:
        for gpu in gpus:
            if not all(W.feasible(gpu, k) for k in ks):
                continue
            for _ in range(3):
                order = list(range(len(ks)))
                for i in range(len(order) - 1, 0, -1):
                    j = rng.below(i + 1)
                    order[i], order[j] = order[j], order[i]
                r = O.simulate(gpu, ks, order, trace=True)
                check_trace(gpu, ks, order, r.trace, r.rounds)
                # round cost recomputed from the rounds with exact rationals
                RB = Fraction(gpu[5], gpu[6])
                T = sum(max(Fraction(sum(p[i] * ks[i][4] for i in range(len(ks)))),
                            RB * sum(p[i] * ks[i][5] for i in range(len(ks)))) for p in r.rounds)
                assert T * gpu[6] == r.key


def test_histogram_properties():
    gpu, ks = W.config("C2")
    s, keys = O.sweep(gpu, ks, keys=True, threads=4)
    for B in (1, 2, 7, 64, 256, 1000):
        h = O.histogram(keys, s.key_min, s.key_max, B)
        assert sum(h) == len(keys) == 40320
        assert h[0] >= 1 and h[-1] >= 1 if B > 1 else h == [40320]
        # bin b holds exactly the keys in [kmin + b*w, kmin + (b+1)*w), last bin closed:
        # locate each distinct key among the interval boundaries (bisect, library)
        w = Fraction(s.key_max - s.key_min, B)
        bounds = [s.key_min + b * w for b in range(1, B)]
        cnt = [0] * B
        for k, c in Counter(int(k) for k in keys).items():
            cnt[bisect.bisect_right(bounds, k)] += c
        assert cnt == h
    # all-equal keys -> bin 0
    assert O.histogram([5, 5, 5], 5, 5, 4) == [3, 0, 0, 0]


def test_ratio_identity_total_inst_over_total_mem():
    # SPEC:88 / PAPER:108: R_comb(a,b) = total inst / total mem units
    sets = W.random_small_sets(0xCAFE, 50, 2, 2)
    for ks in sets:
        _, _, rc = O.pair_score(G, ks, 0, 1)
        want = Fraction(ks[0][0] * ks[0][4] + ks[1][0] * ks[1][4], ks[0][0] * ks[0][5] + ks[1][0] * ks[1][5])
        assert abs(rc - float(want)) <= 1e-12 * float(want)
        assert min(ks[0][4] / ks[0][5], ks[1][4] / ks[1][5]) - 1e-12 <= rc <= max(
            ks[0][4] / ks[0][5], ks[1][4] / ks[1][5]) + 1e-12


def _footprint(gpu, k):
    b = -(-k[0] // gpu[0])
    d = demand(k)
    return (d[1] * b, d[0] * b, d[2] * b, b)  # H, G, W, Bk


@pytest.mark.parametrize("seed", range(10))
def test_heuristic_invariants(seed):
    sets = W.random_small_sets(0xA1 + seed, 10, 1, 9)
    for ks in sets:
        order, round_of = O.heuristic(G, ks)
        n = len(ks)
        assert sorted(order) == list(range(n))
        rounds = {}
        for k, r in zip(order, round_of):
            rounds.setdefault(r, []).append(k)
        assert sorted(rounds) == list(range(len(rounds)))
        for r, mem in rounds.items():
            H = [_footprint(G, ks[k])[0] for k in mem]
            assert H == sorted(H, reverse=True)
            if len(mem) > 1:  # SPEC:175 combined footprint within all four limits
                tot = [sum(_footprint(G, ks[k])[q] for k in mem) for q in range(4)]
                assert tot[0] <= G[2] and tot[1] <= G[1] and tot[2] <= G[3] and tot[3] <= G[4]
        # the first selected pair attains the max entry of the initial matrix
        if n >= 2:
            best = None
            for i in range(n):
                for j in range(i + 1, n):
                    f, sc, _ = O.pair_score(G, ks, i, j)
                    if f and (best is None or sc > best):
                        best = sc
            first = rounds[0]
            if best is not None:
                assert len(first) >= 2
                # the first two kernels chosen are a pair whose score equals the max
                found = any(O.pair_score(G, ks, min(a, b), max(a, b))[1] == best
                            for a in first for b in first if a != b)
                assert found


def test_heuristic_epbs6_pairs_opposite_types():
    # EpBs-6 (Table 2 row): 3 EP warps 4 R 3.11, 3 BS warps 12 R 11.1, shm 0
    # -> every round containing both types pairs an EP with a BS.
    ep = (16, 128, 16, 0, 311 * 40, 100 * 40)
    bs = (16, 384, 16, 0, 1110 * 40, 100 * 40)
    ks = [ep, ep, ep, bs, bs, bs]
    order, round_of = O.heuristic(G, ks)
    rounds = {}
    for k, r in zip(order, round_of):
        rounds.setdefault(r, []).append(k)
    for mem in rounds.values():
        types = {("EP" if k < 3 else "BS") for k in mem}
        assert types == {"EP", "BS"}


@pytest.mark.parametrize("seed", range(4))
def test_trace_rules_under_cursor_per_kernel_reading(seed):
    """The alternative-reading trace obeys first fit from SM 0 at every kernel."""
    sets = W.random_small_sets(0x7B1 + seed, 4, 2, 6)
    for ks in sets:
        gpu = list(G) + [1]
        order = list(range(len(ks)))[::-1]
        r = O.simulate(gpu, ks, order, trace=True)
        S = G[0]
        caps = (G[1], G[2], G[3], G[4])
        used = [[0, 0, 0, 0] for _ in range(S)]
        b, rnd = 0, 0
        for k in order:
            d = demand(ks[k])
            cursor = 0
            for _ in range(ks[k][0]):
                rr, s = r.trace[b]
                b += 1
                if rr != rnd:
                    rnd = rr
                    used = [[0, 0, 0, 0] for _ in range(S)]
                    cursor = 0
                x = cursor
                while x != s:
                    assert not all(used[x][q] + d[q] <= caps[q] for q in range(4))
                    x = (x + 1) % S
                for q in range(4):
                    used[s][q] += d[q]
                cursor = (s + 1) % S


READINGS = [1, 2, 3, 4, 5, 6, 7]  # f3 variants: cursor per kernel (1), strict RR (2), skip-ahead (4), combined


@pytest.mark.parametrize("flags", READINGS)
def test_reading_variants_keep_the_model_invariants(flags):
    """Properties every reading of L4/L5 must keep (the hand traces in
    readings_f3.json pin the rules themselves): block conservation,
    the lower bound max(sum I, R_B sum M) with the exact-rational
    re-score of the rounds, a single round when sum T <= N_SM
    (PAPER:70-71), order invariance of identical kernels and the
    same-side theorem; without skip-ahead, capacity safety of the trace."""
    gpus = [list(G) + [flags], [8, 65536, 102400, 64, 16, 7, 2, flags], [3, 16384, 16384, 32, 4, 5, 1, flags]]
    rng = W.SplitMix64(0xF3F3 + flags)
    for gpu in gpus:
        for ks in W.random_small_sets(0xA11 + flags, 4, 2, 6, gpu=gpu[:7]):
            if not all(W.feasible(gpu[:7], k) for k in ks):
                continue
            order = list(range(len(ks)))
            for i in range(len(order) - 1, 0, -1):
                j = rng.below(i + 1)
                order[i], order[j] = order[j], order[i]
            r = O.simulate(gpu, ks, order, trace=True)
            for i, k in enumerate(ks):
                assert sum(p[i] for p in r.rounds) == k[0]
            assert all(any(p) for p in r.rounds)
            RB = Fraction(gpu[5], gpu[6])
            T = sum(max(Fraction(sum(p[i] * ks[i][4] for i in range(len(ks)))),
                        RB * sum(p[i] * ks[i][5] for i in range(len(ks)))) for p in r.rounds)
            assert T * gpu[6] == r.key >= exact_lower_bound(gpu, ks)
            if not flags & 4:  # trace in launch order: replay the capacities per (round, SM)
                used = {}
                blocks = [k for k in order for _ in range(ks[k][0])]
                for k, (rr, s) in zip(blocks, r.trace):
                    u = used.setdefault((rr, s), [0, 0, 0, 0])
                    for q, dq in enumerate(demand(ks[k])):
                        u[q] += dq
                    assert all(u[q] <= gpu[1 + q] for q in range(4))
    # single round when the blocks do not exceed N_SM
    ks = [(3, 128, 16, 0, 311, 100), (5, 256, 32, 8192, 2400, 100), (8, 64, 20, 0, 50, 100)]
    for order in itertools.permutations(range(3)):
        r = O.simulate(list(G) + [flags], ks, list(order))
        assert len(r.rounds) == 1 and r.key == exact_lower_bound(G, ks)
    # identical kernels that differ only in N_tblk; same-side sets
    ks = [(g, 256, 24, 12288, 800 * 3, 100 * 3) for g in (16, 48, 24, 80, 32)]
    s, _ = O.sweep(list(G) + [flags], ks)
    assert s.key_min == s.key_max
    for cl in ("mem", "cmp"):
        for ks in W.random_small_sets(0xB3, 4, 3, 5, classes=cl):
            s, _ = O.sweep(list(G) + [flags], ks)
            want = G[6] * sum(k[0] * k[4] for k in ks) if cl == "cmp" else G[5] * sum(k[0] * k[5] for k in ks)
            assert s.key_min == s.key_max == want
