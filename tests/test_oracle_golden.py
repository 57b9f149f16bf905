"""Pins of the oracle against hand-derived goldens (tests/golden/*.json).

Each golden is derived by hand from the paper (PAPER:69-81 placement,
PAPER:110-198 Algorithm 1) and SPEC's round time; none of its
values comes from the oracle or the CUDA path.
"""
import itertools
import json
import os

import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _layers_to_rounds(spec: str, n: int, per_layer: int):
    rounds = []
    for grp in spec.strip("{}").split("}{"):
        p = [0] * n
        for c in grp.split(","):
            p[int(c)] += per_layer
        rounds.append(p)
    return rounds


W4 = _load("w4.json")


def test_w4_hand_list_of_24_orders_is_lexicographic_unrank():
    # the explicit hand-written list of the 24 orders (golden) == unrank(idx)
    for idx, ostr, _, _ in W4["orders"]:
        assert O.unrank(idx, 4) == [int(c) for c in ostr]
        assert O.rank([int(c) for c in ostr]) == idx


@pytest.mark.parametrize("row", W4["orders"], ids=lambda r: r[1])
def test_w4_every_order_time_and_rounds(row):
    idx, ostr, layers, T = row
    g, ks = W4["gpu"], W4["kernels"]
    r = O.simulate(g, ks, [int(c) for c in ostr])
    assert r.key == 100 * T  # K = den * T exactly
    assert r.rounds == _layers_to_rounds(layers, 4, W4["layer_blocks"])
    assert abs(r.t_naive - T) <= 1e-12 * T


def test_w4_sweep_stats_and_distribution():
    g, ks = W4["gpu"], W4["kernels"]
    st = W4["stats"]
    s, keys = O.sweep(g, ks, cand_key=100 * W4["heuristic"]["T"], keys=True)
    assert s.key_min == 100 * st["best"] and s.argmin == st["argmin"]
    assert s.key_max == 100 * st["worst"] and s.argmax == st["argmax"]
    dist = {}
    for k in keys:
        dist[str(int(k) // 100)] = dist.get(str(int(k) // 100), 0) + 1
    assert dist == st["distribution"]
    # percentile of the heuristic order (ties count for the candidate)
    assert 100.0 * (s.n_eq + s.n_gt) / 24 == W4["heuristic"]["percentile"]


@pytest.mark.parametrize("threads", [1, 2, 5, 24])
def test_w4_sweep_thread_split_is_identical(threads):
    g, ks = W4["gpu"], W4["kernels"]
    s1, _ = O.sweep(g, ks, cand_key=12966400, threads=1)
    st, _ = O.sweep(g, ks, cand_key=12966400, threads=threads)
    assert st.as_tuple() == s1.as_tuple()


def test_w4_histograms():
    g, ks = W4["gpu"], W4["kernels"]
    s, keys = O.sweep(g, ks, keys=True)
    assert O.histogram(keys, s.key_min, s.key_max, 4) == W4["hist4"]
    assert O.histogram(keys, s.key_min, s.key_max, 8) == W4["hist8"]


def test_w4_heuristic():
    g, ks = W4["gpu"], W4["kernels"]
    h = W4["heuristic"]
    order, round_of = O.heuristic(g, ks)
    assert order == h["order"]
    rounds = {}
    for k, r in zip(order, round_of):
        rounds.setdefault(r, []).append(k)
    assert [rounds[r] for r in sorted(rounds)] == h["rounds"]
    assert O.rank(order) == h["index"]
    assert O.simulate(g, ks, order).key == 100 * h["T"]
    for pair, want in h["pair_scores"].items():
        i, j = map(int, pair.split(","))
        feas, score, _ = O.pair_score(g, ks, i, j)
        if want is None:
            assert not feas
        else:
            assert feas and abs(score - want) < 5e-7
    worst = W4["stats"]["worst"]
    assert round(worst / h["T"], 4) == h["speedup_over_worst"]


def test_w2_cursor_pin():
    w = _load("w2_cursor.json")
    r = O.simulate(w["gpu"], w["kernels"], w["order"], trace=True)
    assert [list(t) for t in r.trace] == w["trace"]
    assert r.rounds == w["rounds"]
    assert r.key == w["T"] * w["gpu"][6]
    assert r.key != w["T_rejected_reading"]


def test_app_c1_one_block_per_sm_is_not_order_invariant():
    c = _load("counterexamples.json")["C1"]
    for order, T, rounds in c["cases"]:
        r = O.simulate(c["gpu"], c["kernels"], order)
        assert r.key == T and r.rounds == rounds


def test_app_c2_insertion_can_decrease_time():
    c = _load("counterexamples.json")["C2"]
    ks = c["kernels"]
    wo = c["without_X"]
    assert O.simulate(c["gpu"], [ks[i] for i in wo["kernels_idx"]], wo["order"]).key == wo["T"]
    wx = c["with_X_first"]
    assert O.simulate(c["gpu"], ks, wx["order"]).key == wx["T"]


SPEC_EX = _load("spec_examples.json")


def test_spec_score_same_side():
    e = SPEC_EX["score_same_side"]
    feas, score, _ = O.pair_score((16, 32768, 49152, 48, 8, 411, 100), e["kernels"], 0, 1)
    assert feas and round(score, 4) == e["score"]
    assert abs(score - (1 / 3 + 1 / 2 + 1 / 2)) < 1e-15


def test_spec_straddle_bonus_and_rcomb():
    e = SPEC_EX["straddle_bonus"]
    feas, score, rc = O.pair_score((16, 32768, 49152, 48, 8, 411, 100), e["kernels"], 0, 1)
    assert feas
    assert round(rc, 4) == e["r_comb"]
    slack = 1 + 24064 / 32768 + 36 / 48
    assert round(score - slack, 4) == e["bonus"]


def test_spec_fit_predicates():
    g = (16, 32768, 49152, 48, 8, 411, 100)
    e = SPEC_EX["infeasible_pair"]
    assert O.pair_score(g, e["kernels"], 0, 1)[0] is False
    e = SPEC_EX["boundary_fit"]
    assert O.pair_score(g, e["kernels"], 0, 1)[0] is True
    e = SPEC_EX["infeasible_kernel"]
    assert O.check_inputs(g, e["kernels"]) == O.OR_EINFEASIBLE


def test_input_validation_codes():
    g = (16, 32768, 49152, 48, 8, 411, 100)
    assert O.check_inputs(g, [(16, 0, 1, 0, 1, 1)]) == O.OR_EINVAL          # tpb >= 1
    assert O.check_inputs(g, [(16, 1025, 1, 0, 1, 1)]) == O.OR_EINVAL       # tpb <= 1024
    assert O.check_inputs(g, [(0, 32, 1, 0, 1, 1)]) == O.OR_EINVAL          # grid >= 1
    assert O.check_inputs(g, [(16, 32, 1, 0, 0, 1)]) == O.OR_EINVAL         # inst >= 1
    assert O.check_inputs(g, [(16, 32, 1, 0, 1, 0)]) == O.OR_EMISSINGRATIO
    assert O.check_inputs(g, [(16, 1024, 33, 0, 1, 1)]) == O.OR_EINFEASIBLE  # regs 33792 > 32768
    assert O.check_inputs((0, 1, 1, 1, 1, 1, 1), [(1, 32, 1, 0, 1, 1)]) == O.OR_EINVAL


def test_unrank_equals_library_permutation_enumeration():
    # itertools.permutations of a sorted list yields lexicographic order (library routine)
    for n in range(1, 9):
        for idx, p in enumerate(itertools.permutations(range(n))):
            if n >= 7 and idx % 7:  # sample the larger spaces
                continue
            assert O.unrank(idx, n) == list(p)
            assert O.rank(list(p)) == idx
    import math
    assert O.factorial(12) == math.factorial(12) == 479001600


def test_w2_alternative_cursor_reading():
    """the rejected reading of L4 (cursor restarts at SM 0 for
    every kernel) as a model flag; W2 gives T = 7 (hand trace, golden)."""
    w = _load("w2_cursor.json")
    gpu = list(w["gpu"]) + [1]
    r = O.simulate(gpu, w["kernels"], w["order"], trace=True)
    assert [list(t) for t in r.trace] == w["rejected_reading_trace"]
    assert r.rounds == w["rejected_reading_rounds"]
    assert r.key == w["T_rejected_reading"] * w["gpu"][6]


ALG1 = _load("alg1_branches.json")


@pytest.mark.parametrize("case", ALG1["cases"], ids=lambda c: c["name"])
def test_algorithm1_unspecified_branches_hand_golden(case):
    """Ties, no feasible pair, lone kernel,
    equal-shm insertion (reading L17) and the bonus clamp,
    each derived by hand in tests/golden/alg1_branches.json."""
    gpu, ks = ALG1["gpu"], case["kernels"]
    order, round_of = O.heuristic(gpu, ks)
    assert order == case["order"] and round_of == case["round_of"]
    for pair, want in case["pair_scores"].items():
        i, j = (int(x) for x in pair.split(","))
        feasible, score, _ = O.pair_score(gpu, ks, i, j)
        if want is None:
            assert not feasible
        else:
            assert feasible and abs(score - want) <= 1e-12


F3 = _load("readings_f3.json")


@pytest.mark.parametrize("case", F3["cases"], ids=lambda c: c["name"])
def test_model_reading_variants_hand_golden(case):
    """Strict round robin (L4 alt.) and skip-ahead (L5 alt.),
    alone and combined: rounds, dispatch trace and T derived by hand in
    tests/golden/readings_f3.json."""
    for flags, want in case["readings"].items():
        gpu = list(case["gpu"]) + [int(flags)]
        r = O.simulate(gpu, case["kernels"], case["order"], trace=True)
        assert r.rounds == want["rounds"], (flags, r.rounds)
        assert [list(t) for t in r.trace] == want["trace"], (flags, r.trace)
        assert r.key == want["T"] * case["gpu"][6] and r.t_naive == want["T"]


@pytest.mark.parametrize("threads", [1, 3])
def test_keys_of_explicit_indices_w4_hand_golden(threads):
    """or_keys_of (parity samples at full size) returns the hand-derived W4
    time of every index, in any index order and thread split."""
    g, ks = W4["gpu"], W4["kernels"]
    idx = [row[0] for row in W4["orders"]][::-1] + [5, 5, 23, 0]
    want = {row[0]: 100 * row[3] for row in W4["orders"]}
    got = O.keys_of(g, ks, idx, threads=threads)
    assert got.tolist() == [want[i] for i in idx]
    with pytest.raises(O.OracleError):
        O.keys_of(g, ks, [24])
