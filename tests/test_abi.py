"""C-ABI library: loads, exports every symbol include/rk.h declares, and its
host-side logic (validation, Lehmer rank/unrank, Algorithm 1) agrees with the
independent oracle.  No device compute here (runs on CPU)."""
import ctypes
import itertools
import os
import re

import pytest

import oracle as O
from paper_1511_07983_b200 import build as B
from paper_1511_07983_b200 import rk
from paper_1511_07983_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rk_[a-z0-9_]+)\s*\(", src)))


def test_header_declarations_match_binding_exports():
    assert declared_symbols() == sorted(rk.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(rk.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(L, name), name


def test_sm100a_cubin_embedded():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rk.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_rank_unrank_match_library_enumeration():
    for n in range(1, 8):
        for idx, p in enumerate(itertools.permutations(range(n))):
            assert rk.rk_unrank(idx, n) == list(p)
            assert rk.rk_rank(list(p)) == idx
    for idx in (0, 1, 12345678, 479001599):
        assert rk.rk_unrank(idx, 12) == O.unrank(idx, 12)
    with pytest.raises(rk.RkError):
        rk.rk_rank([0, 0, 1])
    with pytest.raises(rk.RkError):
        rk.rk_unrank(24, 4)


def test_host_only_ctx_refuses_compute():
    c = rk.Context(-1)
    c.rk_set_gpu_params(W.GTX580)
    c.rk_set_kernels(W.W4)
    with pytest.raises(rk.RkError) as e:
        c.rk_eval_range(0, 24)
    assert e.value.status == rk.RK_ENODEVICE
    with pytest.raises(rk.RkError) as e:
        c.rk_heuristic_order(with_key=True)
    assert e.value.status == rk.RK_ENODEVICE
    # the two-pass step, the optimum and the memo plan: no device, no evaluation
    for call in (lambda: c.rk_sweep_pass1_async(0, 24, None, None),
                 lambda: c.rk_sweep_pass2_async(0, 24, None, None, 4, None, None, None),
                 lambda: c.rk_sweep_pass2_32_async(0, 24, None, None, 4, None, None, 0, None, None),
                 lambda: c.rk_memo_audit(),
                 lambda: c.rk_best_order()):
        with pytest.raises(rk.RkError) as e:
            call()
        assert e.value.status == rk.RK_ENODEVICE
    assert c.rk_memo_info() == (False, 0, [])


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rk.RkError) as e:
        rk.Context(0)
    assert e.value.status == rk.RK_ENODEVICE


CASES = [
    ([(16, 0, 1, 0, 1, 1)], O.OR_EINVAL),
    ([(16, 1025, 1, 0, 1, 1)], O.OR_EINVAL),
    ([(0, 32, 1, 0, 1, 1)], O.OR_EINVAL),
    ([(16, 32, 1, 0, 0, 1)], O.OR_EINVAL),
    ([(16, 32, 1, 0, 1, 0)], O.OR_EMISSINGRATIO),
    ([(16, 1024, 33, 0, 1, 1)], O.OR_EINFEASIBLE),
    ([(16, 128, 20, 65536, 311, 100)], O.OR_EINFEASIBLE),
    ([(16, 128, 20, 0, 311, 100)] * 17, O.OR_ETOOMANY),
    ([(1 << 31, 32, 1, 0, 1 << 31, 1)], O.OR_EOVERFLOW),
]


@pytest.mark.parametrize("kernels,code", CASES)
def test_validation_codes_agree_with_oracle(kernels, code):
    c = rk.Context(-1)
    c.rk_set_gpu_params(W.GTX580)
    if code != O.OR_EOVERFLOW and code != O.OR_ETOOMANY:
        assert O.check_inputs(W.GTX580, kernels) == code
    with pytest.raises(rk.RkError) as e:
        c.rk_set_kernels(kernels)
    want = {O.OR_EINVAL: rk.RK_EINVAL, O.OR_EINFEASIBLE: rk.RK_EINFEASIBLE, O.OR_ETOOMANY: rk.RK_ETOOMANY,
            O.OR_EMISSINGRATIO: rk.RK_EMISSINGRATIO, O.OR_EOVERFLOW: rk.RK_EOVERFLOW}[code]
    assert e.value.status == want


def test_bad_gpu_params():
    c = rk.Context(-1)
    with pytest.raises(rk.RkError) as e:
        c.rk_set_gpu_params((0, 32768, 49152, 48, 8, 411, 100))
    assert e.value.status == rk.RK_EINVAL
    # 33 SMs: gcd(33, grids 32/16) = 1 -> 33 super-SMs: run-length state, accepted
    c.rk_set_gpu_params((33, 32768, 49152, 48, 8, 411, 100))
    c.rk_set_kernels(W.W4)
    # the B200 preset (148 SMs) is accepted; more than 65535 SMs is not
    c.rk_set_gpu_params(W.B200)
    c.rk_set_kernels(W.config("C6")[1])
    with pytest.raises(rk.RkError) as e:
        c.rk_set_gpu_params((65536, 32768, 49152, 48, 8, 411, 100))
    assert e.value.status == rk.RK_EUNSUPPORTED
    # 48 SMs with grids that are multiples of 16: reduced to 3 super-SMs, accepted
    c.rk_set_gpu_params((48, 32768, 49152, 48, 8, 411, 100))
    c.rk_set_kernels([(48, 128, 20, 0, 311, 100), (96, 256, 24, 0, 1110, 100)])
    c2 = rk.Context(-1)
    with pytest.raises(rk.RkError) as e:
        c2.rk_set_kernels(W.W4)
    assert e.value.status == rk.RK_ESTATE


def test_w4_heuristic_host():
    c = rk.Context(-1)
    c.rk_set_gpu_params(W.GTX580)
    c.rk_set_kernels(W.W4)
    order, round_of, idx, _ = c.rk_heuristic_order(with_key=False)
    assert order == [2, 1, 0, 3] and round_of == [0, 0, 1, 1] and idx == 14


@pytest.mark.parametrize("seed", range(20))
def test_heuristic_matches_oracle_algorithm1(seed):
    # product Algorithm 1 (rk_host.cpp) vs the oracle's independent implementation
    gpus = [W.GTX580, (8, 65536, 102400, 64, 16, 7, 2), (24, 32768, 49152, 48, 8, 311, 100)]
    sets = W.random_small_sets(0xA160 + seed, 25, 1, 12)
    c = rk.Context(-1)
    for i, ks in enumerate(sets):
        gpu = gpus[i % len(gpus)]
        if not all(W.feasible(gpu, k) for k in ks):
            continue
        c.rk_set_gpu_params(gpu)
        c.rk_set_kernels(ks)
        order, round_of, idx, _ = c.rk_heuristic_order(with_key=False)
        o2, r2 = O.heuristic(gpu, ks)
        assert (order, round_of) == (o2, r2)
        assert idx == O.rank(o2)


def test_heuristic_matches_oracle_on_configs():
    c = rk.Context(-1)
    for name in ("C1", "C2", "C3", "C4"):
        gpu, ks = W.config(name)
        c.rk_set_gpu_params(gpu)
        c.rk_set_kernels(ks)
        order, round_of, _, _ = c.rk_heuristic_order(with_key=False)
        assert (order, round_of) == O.heuristic(gpu, ks)
    sets = W.c5_sets(64)
    c.rk_set_gpu_params(W.GTX580)
    for ks in sets:
        c.rk_set_kernels(ks)
        assert c.rk_heuristic_order(with_key=False)[:2] == O.heuristic(W.GTX580, ks)


def test_heuristic_host_unspecified_branches_hand_golden():
    """rk_heuristic_order (host Algorithm 1) on the hand-derived branch goldens
    (tests/golden/alg1_branches.json: SPEC:182/184/187)."""
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "alg1_branches.json")))
    c = rk.Context(-1)
    c.rk_set_gpu_params(g["gpu"])
    for case in g["cases"]:
        c.rk_set_kernels(case["kernels"])
        order, round_of, idx, _ = c.rk_heuristic_order(with_key=False)
        assert (order, round_of) == (case["order"], case["round_of"]), case["name"]
        assert idx == rk.rk_rank(case["order"])


def test_model_reading_flags_validation_and_policy_limits():
    """rk_gpu_params.flags: the three f3 bits are accepted, any other bit is
    RK_EINVAL; strict RR / skip-ahead with more than 32 super-SMs is refused at
    rk_set_kernels (RK_EUNSUPPORTED) on host-only contexts too; Algorithm 1
    (host) is independent of the reading."""
    c = rk.Context(-1)
    for f in (1, 2, 3, 4, 5, 6, 7):
        c.rk_set_gpu_params(list(W.GTX580) + [f])
        c.rk_set_kernels(W.W4)
        assert c.rk_heuristic_order(with_key=False)[0] == [2, 1, 0, 3]
    with pytest.raises(rk.RkError) as e:
        c.rk_set_gpu_params(list(W.GTX580) + [8])
    assert e.value.status == rk.RK_EINVAL
    gpu, ks = W.config("C6")
    c.rk_set_gpu_params(list(gpu) + [rk.RK_FLAG_SKIP_AHEAD])
    with pytest.raises(rk.RkError) as e:
        c.rk_set_kernels(ks)
    assert e.value.status == rk.RK_EUNSUPPORTED
    c.rk_set_gpu_params(list(gpu) + [rk.RK_FLAG_CURSOR_PER_KERNEL])
    c.rk_set_kernels(ks)  # the cursor reading runs on every state (run-length included)
