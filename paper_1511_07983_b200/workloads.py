"""Seeded synthetic inputs shared by tests, bench and smoke — NO method arithmetic.

This module only *constructs* inputs (GPU presets and kernel profiles).  It
holds none of the model's arithmetic (no placement, no round scoring, no
Algorithm 1), so the product path and the oracle can both consume it without
sharing any computation (task rule ③).  The recipe is DESIGN.md §4.

A kernel is a 6-tuple ``(grid_blocks, threads_per_block, regs_per_thread,
shm_per_block, inst_per_block A_i, mem_per_block M_i)`` (Table 1,
PAPER:54-58); R_i = A_i / M_i.  A GPU is a 7-tuple ``(n_sm, regs_per_sm,
shm_per_sm, warps_per_sm, blocks_per_sm, rb_num, rb_den)`` with R_B =
rb_num / rb_den (Table 1).
"""
from __future__ import annotations

MASK64 = (1 << 64) - 1

#: GTX580 preset, PAPER:254 ("16 SMs, R_B=4.11, N_reg_SM=32K, N_warp_SM=48,
#: N_shm_SM=48K, N_blk_SM=8").  R_B = 411/100 exactly (reading L10).
GTX580 = (16, 32768, 49152, 48, 8, 411, 100)

#: B200 preset (not a paper configuration): 148 SMs, 64K
#: registers, 228 KB shared memory, 64 warps and 32 blocks per SM.  R_B follows
#: the paper's GTX580 figure, which is CUDA cores x clock / DRAM bandwidth
#: (512 x 1.544 GHz / 192.4 GB/s = 4.11): 148 x 128 x 1.965 GHz /
#: 8.0 TB/s = 4.65 (reading L24).
B200 = (148, 65536, 233472, 64, 32, 465, 100)

SEED_BASE = 0x0151107983000000


class SplitMix64:
    """splitmix64 (Steele, Lea, Flood 2014) — the seeded generator of DESIGN.md §4."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def below(self, n: int) -> int:
        return self.next() % n

    def choice(self, seq):
        return seq[self.below(len(seq))]

    def weighted(self, seq, weights):
        t = self.below(sum(weights))
        for v, w in zip(seq, weights):
            if t < w:
                return v
            t -= w
        raise AssertionError


def warps_of(tpb: int) -> int:
    return (tpb + 31) // 32


def key_bound(gpu, kernels) -> int:
    """Upper bound of any order's exact key: sum_i T_i*(den*A_i + num*M_i)."""
    return sum(k[0] * (gpu[6] * k[4] + gpu[5] * k[5]) for k in kernels)


def feasible(gpu, k) -> bool:
    """A single block fits a fresh SM."""
    return k[2] * k[1] <= gpu[1] and k[3] <= gpu[2] and warps_of(k[1]) <= gpu[3]


# ---- W4 (config C1 hand golden) --------------------------------
W4 = [
    (32, 128, 20, 16384, 311, 100),   # EP-like, memory-bound, R 3.11
    (32, 256, 24, 0, 1110, 100),      # BS-like, compute-bound, R 11.1
    (16, 128, 20, 32768, 622, 200),   # EP-like, memory-bound
    (32, 512, 16, 0, 2220, 200),      # BS-like, compute-bound
]

# ---- Generator G ("Rodinia/SDK-like") -------------------------------
TPB = (64, 128, 256, 512, 1024)
TPB_W = (1, 4, 4, 2, 1)
RPT = (16, 20, 24, 28, 32, 40, 48, 63)
SHM = (2048, 4096, 8192, 12288, 16384, 24576, 32768, 49152)
GRID = (16, 24, 32, 48, 64, 80, 96, 128)
RN_MEM = (50, 100, 150, 200, 311)
RN_CMP = (600, 800, 1110, 1600, 2400)


def _ratio_work(rng: SplitMix64, rn: int, tpb: int):
    c = (1 + rng.below(64)) * warps_of(tpb)
    return rn * c, 100 * c


def gen_g(rng: SplitMix64, n: int, gpu=GTX580):
    """Generator G: n kernels, classes alternate memory-/compute-bound."""
    while True:
        ks = []
        for i in range(n):
            while True:
                tpb = rng.weighted(TPB, TPB_W)
                rpt = rng.choice(RPT)
                shm = 0 if rng.below(10) < 4 else rng.choice(SHM)
                grid = rng.choice(GRID)
                rn = rng.choice(RN_MEM if i % 2 == 0 else RN_CMP)
                a, m = _ratio_work(rng, rn, tpb)
                k = (grid, tpb, rpt, shm, a, m)
                if feasible(gpu, k):
                    break
            ks.append(k)
        if key_bound(gpu, ks) < (1 << 63):
            return ks


GRID_B200 = (100, 128, 200, 256, 300, 444, 512, 600, 1000, 1024)
RPT_B200 = (16, 24, 32, 40, 48, 64, 96, 128, 168, 255)
SHM_B200 = (4096, 8192, 16384, 32768, 49152, 65536, 102400, 163840, 232448)


def gen_b200(rng: SplitMix64, n: int, gpu=B200):
    """Generator G scaled to the B200 preset: grids of 100-1024 blocks (so
    gcd(148, grids) is small and the reduced SM count stays > 32), up to 255
    registers/thread and 227 KB shared memory/block; classes alternate."""
    while True:
        ks = []
        for i in range(n):
            while True:
                tpb = rng.weighted(TPB, TPB_W)
                rpt = rng.choice(RPT_B200)
                shm = 0 if rng.below(10) < 4 else rng.choice(SHM_B200)
                grid = rng.choice(GRID_B200)
                rn = rng.choice(RN_MEM if i % 2 == 0 else RN_CMP)
                a, m = _ratio_work(rng, rn, tpb)
                k = (grid, tpb, rpt, shm, a, m)
                if feasible(gpu, k):
                    break
            ks.append(k)
        if key_bound(gpu, ks) < (1 << 63):
            return ks


def gen_c3(rng: SplitMix64, n: int = 10, gpu=GTX580):
    """C3: shm- and register-limited packing (1-3 blocks/SM by regs or shm)."""
    ks = []
    for i in range(n):
        while True:
            tpb = rng.choice((128, 256))
            rpt = rng.choice((32, 40, 48, 63))
            shm = rng.choice((12288, 16384, 24576, 32768))
            grid = rng.choice((16, 32, 48, 64))
            rn = rng.choice(RN_MEM if i % 2 == 0 else RN_CMP)
            a, m = _ratio_work(rng, rn, tpb)
            k = (grid, tpb, rpt, shm, a, m)
            if feasible(gpu, k):
                break
        ks.append(k)
    assert key_bound(gpu, ks) < (1 << 63)
    return ks


def gen_c2(rng: SplitMix64):
    """C2: EpBsEsSw-8 shape: 2 each of EP-, BS-, ES-, SW-like.

    EP and BS parameters follow Table 2 / PAPER:254 (R 3.11, 11.1); ES and SW are
    synthetic (not published)."""
    ks = []
    for _ in range(2):  # EP-like: R 3.11, tpb 128, regs 20, shm {0,16K}, grid {16,32}
        tpb = 128
        a, m = _ratio_work(rng, 311, tpb)
        ks.append((rng.choice((16, 32)), tpb, 20, rng.choice((0, 16384)), a, m))
    for _ in range(2):  # BS-like: R 11.1, tpb {128,256}, regs {16,24}, shm 0, grid {32,64}
        tpb = rng.choice((128, 256))
        a, m = _ratio_work(rng, 1110, tpb)
        ks.append((rng.choice((32, 64)), tpb, rng.choice((16, 24)), 0, a, m))
    for _ in range(2):  # ES-like: compute-bound R 24, tpb 256, regs 32, shm {0,4K}, grid {48,96}
        tpb = 256
        a, m = _ratio_work(rng, 2400, tpb)
        ks.append((rng.choice((48, 96)), tpb, 32, rng.choice((0, 4096)), a, m))
    for _ in range(2):  # SW-like: memory-bound R 1.5, tpb {64,128}, regs 28, shm {8K,24K}, grid {16,64}
        tpb = rng.choice((64, 128))
        a, m = _ratio_work(rng, 150, tpb)
        ks.append((rng.choice((16, 64)), tpb, 28, rng.choice((8192, 24576)), a, m))
    return ks


def config(name: str):
    """Return (gpu, kernels) for configs C1..C4 (BASELINE.json `configs`) and C6
    (the B200 preset)."""
    if name == "C1":
        return GTX580, list(W4)
    if name == "C2":
        return GTX580, gen_c2(SplitMix64(SEED_BASE + 2))
    if name == "C3":
        return GTX580, gen_c3(SplitMix64(SEED_BASE + 3))
    if name == "C4":
        return GTX580, gen_g(SplitMix64(SEED_BASE + 4), 12)
    if name == "C6":  # B200 preset (f3), same n as C4
        return B200, gen_b200(SplitMix64(SEED_BASE + 6), 12)
    raise KeyError(name)


def c1_random_sets(count: int = 64, n: int = 4):
    rng = SplitMix64(SEED_BASE + 1)
    return [gen_g(rng, n) for _ in range(count)]


def c5_sets(n_sets: int = 4096, n: int = 9):
    """C5: 4096 random 9-kernel sets, set s seeded SEED_BASE+5+s.  Alternating
    classes put kernels on both sides of R_B, so no set is degenerate (F1)."""
    return [gen_g(SplitMix64(SEED_BASE + 5 + s), n) for s in range(n_sets)]


def random_small_sets(seed: int, count: int, n_lo: int, n_hi: int, gpu=GTX580, classes: str = "mixed"):
    """Property-test inputs: count sets with n in [n_lo, n_hi].

    classes: "mixed" (alternating), "mem" (all R <= R_B), "cmp" (all R >= R_B)."""
    rng = SplitMix64(seed)
    out = []
    for _ in range(count):
        n = n_lo + rng.below(n_hi - n_lo + 1)
        ks = []
        for i in range(n):
            while True:
                tpb = rng.weighted(TPB, TPB_W)
                rpt = rng.choice(RPT)
                shm = 0 if rng.below(10) < 4 else rng.choice(SHM)
                grid = rng.choice(GRID)
                if classes == "mem":
                    rn = rng.choice(RN_MEM)
                elif classes == "cmp":
                    rn = rng.choice(RN_CMP)
                else:
                    rn = rng.choice(RN_MEM if i % 2 == 0 else RN_CMP)
                a, m = _ratio_work(rng, rn, tpb)
                k = (grid, tpb, rpt, shm, a, m)
                if feasible(gpu, k):
                    break
            ks.append(k)
        out.append(ks)
    return out
