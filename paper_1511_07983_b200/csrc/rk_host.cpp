/*
 * rk_host.cpp — host side of librk: the C ABI of include/rk.h, input
 * validation and device-table packing, Algorithm 1 (kept on the CPU because
 * it is sequential, BASELINE north_star), Lehmer rank/unrank, and the launch
 * orchestration of rk_kernels.cu.  Product path; shares nothing with oracle/.
 */
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "rk.h"
#include "rk_internal.h"

typedef unsigned __int128 u128;
constexpr uint32_t kSmemBinsHost = 32768; /* fused-histogram bins held in shared memory */

/* Device buffer that only grows (memo arenas are reused across kernel sets). */
struct Arena {
    void* p = nullptr;
    size_t cap = 0;
    /* ensure >= bytes; keep the first `keep` bytes of the contents */
    int reserve(size_t bytes, size_t keep = 0) {
        if (bytes <= cap) return 0;
        size_t want = std::max(bytes, cap + cap / 2);
        void* q = nullptr;
        int e = cudaMalloc(&q, want);
        if (e) return e;
        if (keep && p) e = cudaMemcpy(q, p, std::min(keep, cap), cudaMemcpyDeviceToDevice);
        cudaFree(p);
        p = q;
        cap = want;
        return e;
    }
    void release() {
        cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

/* Suffix-memoisation plan: per-level capacities found once per
 * kernel set (sizes only; every step rebuilds all tables).  Level j+1 holds at
 * most cnt[j] * (n - j) nodes; the planning build measures cnt[j+1] exactly. */
struct DpPlan {
    bool on = false;
    uint32_t P = 0;               /* run level: prefixes of P kernels, suffix rows of D = n - P kernels */
    uint32_t L = 0;               /* levels built: P + 1 (level P+1 feeds the 24-key rows of the suffix build) */
    uint32_t node_bytes = 0;
    std::vector<uint32_t> cnt;    /* distinct nodes per level 0..P (cnt[0] = 1) */
    std::vector<uint32_t> cap;    /* node capacity of level j (j >= 1) */
    std::vector<size_t> noff;     /* node byte offset of level j (j >= 1) */
    std::vector<size_t> toff;     /* hash-table slot offset of level j (j >= 1) */
    std::vector<uint32_t> tmask;  /* slots - 1 of level j */
    std::vector<size_t> xoff;     /* transition offset of level j (j < P): cnt[j] * n entries */
    std::vector<uint64_t> work;   /* launch work of level j: (nodes of level j) * n */
    /* the plan's own build (upper-bound layout) serves the first step after rk_set_kernels: that step
     * expands the range's prefixes over it instead of rebuilding the levels (then every step rebuilds) */
    bool reuse_ub = false, last_ub = false;
    std::vector<size_t> ub_noff, ub_xoff, ub_toff;
    std::vector<uint32_t> ub_cap, ub_tmask;
    size_t table_slots = 0;
    Arena nodes, tables, tid, dk, fst, counters; /* counters: P + 1 node counters, then the overflow flag */
    Arena code, dvc, dvp, nd, offs;              /* suffix rows: byte codes into sorted distinct (value, count) */
    Arena row24;                                 /* the (D-1)! = 24 suffix keys of every level-(P+1) node */
    Arena expand;                                /* the range's prefix expansion, levels 1..P-1 (level P recomputed) */
    Arena meta_u, meta_K;                        /* the range's run metadata for the key stream: node | wide, Kb */
    Arena rslot, rmult, rlist, rminrun;          /* the range's row multiset (distinct (node, K_closed), multiplicity, first run) */
    Arena rwlist, rwminrun;                      /* its weighted rows without a slot */
    Arena pslot, pmult, pminrun;                 /* the parent multiset (level P-1 prefixes) */
    uint32_t pmask = 0;
    uint32_t rmask = 0;                          /* its slots - 1 */
    bool runs_ok = false;                        /* meta_u/meta_K hold the range [runs_first, +runs_count) */
    uint64_t runs_first = 0, runs_count = 0;
    DPView view{};
};

struct rk_ctx {
    int device = -1;
    std::string err;
    bool has_params = false, has_kernels = false;
    rk_gpu_params gp{};
    std::vector<rk_kernel> ks;
    RkTables tab{};
    RkTables* tab_dev = nullptr;
    rk_stats* recs_dev = nullptr;     /* per-CTA records of rk_eval_kernel */
    uint32_t* counter_dev = nullptr;  /* last-CTA counter (self-resetting) */
    rk_stats* stats_dev = nullptr;    /* one record for the synchronous calls */
    uint64_t* u64_dev = nullptr;      /* small scratch (indices / keys) */
    void* batch_scratch = nullptr;    /* rk_eval_batch's memoised kernel: prefix states + rows per CTA */
    void* pin = nullptr;              /* rk_eval_batch's pinned upload staging (grow-only) */
    size_t pin_bytes = 0;
    size_t batch_scratch_bytes = 0;
    uint32_t max_ctas = 0;
    uint32_t sms = 0;                 /* SM count of `device` */
    uint32_t launches = 0;
    bool no_reduce = false; /* RK_NO_REDUCE=1: disable the symmetry reduction (testing) */
    bool force_runs = false; /* RK_FORCE_RUNS=1: run-length SM state for every S (testing) */
    bool no_memo = false;    /* RK_NO_MEMO=1: direct evaluation of every order (testing) */
    bool force_memo = false; /* RK_FORCE_MEMO=1: memoise even where it does not pay (testing) */
    bool no_coop = false;    /* RK_NO_COOP=1: one launch per level (no cooperative multi-level launch) */
    /* pass 2's counts/histogram: from the distinct rows (dedup, default) or every run.  Pass 1's run pass
     * (run metadata + the row multiset) runs beside the suffix-row build, pass 2's counts/histogram beside
     * the key stream, both on a high-priority side stream (RK_OVERLAP=0: all serial).  RK_ROW_DEDUP /
     * RK_OVERLAP = 0|1 force either (-1 = default) */
    int row_dedup = -1, overlap = -1;
    bool dedup_now = false;  /* the current range's counts/histogram come from the row multiset */
    uint32_t rows_ctas = 2;  /* RK_ROWS_CTAS: its CTAs per SM when overlapped */
    cudaStream_t side = nullptr;    /* pass 2's side stream (high priority) */
    cudaStream_t side1 = nullptr;   /* pass 1's side stream (the default priority: the suffix rows go first) */
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    DpPlan dp;
    /* optional per-phase device timing (rk_set_timing): event pairs recorded on
     * the launching stream around each phase, read back by rk_timing_read */
    bool timing = false;
    std::vector<cudaEvent_t> tev;  /* 2 per mark */
    std::vector<uint32_t> tphase;  /* phase of each mark */
    size_t tused = 0;
};

/* SM count that selects the kernel variant (the table keeps the real S) */
static uint32_t vS(const rk_ctx* c, uint32_t S) {
    if (c->gp.flags & RK_FLAG_SKIP_AHEAD) return S | RK_S_POLICY; /* per-order policy kernels */
    return c->force_runs ? 65535u : S;
}
/* skip-ahead: the state after a prefix carries pending blocks, so only the per-order policy kernels apply
 * (strict round robin keeps L4's prefix state and runs on every path, register state only) */
static bool policy(const rk_ctx* c) { return (c->gp.flags & RK_FLAG_SKIP_AHEAD) != 0; }

namespace {

rk_status fail(rk_ctx* c, rk_status s, const char* fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return s;
}

rk_status cuda_fail(rk_ctx* c, int e, const char* where) {
    return fail(c, RK_ECUDA, "%s: %s", where, cudaGetErrorString((cudaError_t)e));
}

struct DeviceGuard { /* keep the caller's current device */
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

uint64_t fact64(uint32_t m) {
    uint64_t f = 1;
    for (uint32_t i = 2; i <= m; i++) f *= i;
    return f;
}

/* ---------------- validation + device table packing ---------------------- */
struct Derived {
    uint64_t regs, shm, warps; /* per-block demand (O1 readings L6, L7) */
};

Derived derive(const rk_kernel& k) {
    Derived d;
    d.regs = (uint64_t)k.regs_per_thread * k.threads_per_block;
    d.shm = k.shm_bytes_per_block;
    d.warps = (k.threads_per_block + 31u) / 32u;
    return d;
}

rk_status check_params(rk_ctx* c, const rk_gpu_params& p) {
    if (!p.n_sm || !p.regs_per_sm || !p.shm_bytes_per_sm || !p.max_warps_per_sm || !p.max_blocks_per_sm ||
        !p.rb_num || !p.rb_den)
        return fail(c, RK_EINVAL, "gpu params must all be > 0 (SPEC:30-32)");
    if (p.flags & ~(RK_FLAG_CURSOR_PER_KERNEL | RK_FLAGS_POLICY)) return fail(c, RK_EINVAL, "unknown model flags");
    if (p.max_blocks_per_sm > 255) return fail(c, RK_EUNSUPPORTED, "max_blocks_per_sm > 255");
    if (p.max_warps_per_sm > 32767) return fail(c, RK_EUNSUPPORTED, "max_warps_per_sm > 32767");
    if (p.n_sm > 65535) return fail(c, RK_EUNSUPPORTED, "n_sm > 65535");
    return RK_OK;
}

/* Builds the device tables for one kernel set; validates everything. */
rk_status build_tables(rk_ctx* c, const rk_gpu_params& p, const rk_kernel* ks, uint32_t n, RkTables& t) {
    rk_status s = check_params(c, p);
    if (s) return s;
    if (n == 0) return fail(c, RK_EINVAL, "need at least one kernel");
    if (n > RK_MAX_N) return fail(c, RK_ETOOMANY, "n = %u > %d kernels", n, RK_MAX_N);
    u128 bound = 0;
    uint64_t gr = p.regs_per_sm, gs = p.shm_bytes_per_sm;
    std::vector<Derived> d(n);
    for (uint32_t i = 0; i < n; i++) {
        const rk_kernel& k = ks[i];
        if (k.grid_blocks < 1) return fail(c, RK_EINVAL, "kernel %u: grid_blocks must be >= 1 (SPEC:38)", i);
        if (k.threads_per_block < 1 || k.threads_per_block > 1024)
            return fail(c, RK_EINVAL, "kernel %u: threads_per_block must be in 1..1024 (SPEC:38)", i);
        if (k.inst_per_block < 1) return fail(c, RK_EINVAL, "kernel %u: inst_per_block must be >= 1 (SPEC:39)", i);
        if (k.mem_per_block < 1)
            return fail(c, RK_EMISSINGRATIO, "kernel %u: mem_per_block = 0, R_i undefined (SPEC:61,71)", i);
        d[i] = derive(k);
        if (d[i].regs > p.regs_per_sm || d[i].shm > p.shm_bytes_per_sm || d[i].warps > p.max_warps_per_sm)
            return fail(c, RK_EINFEASIBLE, "kernel %u: one block exceeds an SM limit (SPEC:46)", i);
        bound += (u128)k.grid_blocks * ((u128)p.rb_den * k.inst_per_block + (u128)p.rb_num * k.mem_per_block);
        gr = std::gcd(gr, d[i].regs);
        gs = std::gcd(gs, d[i].shm);
    }
    if (bound >= ((u128)1 << 63)) return fail(c, RK_EOVERFLOW, "exact key bound >= 2^63");
    /* symmetry reduction: g SMs behave as one super-SM */
    uint64_t gb = p.n_sm;
    uint64_t amax = 0;
    for (uint32_t i = 0; i < n; i++) {
        gb = std::gcd(gb, (uint64_t)ks[i].grid_blocks);
        amax = std::max<uint64_t>(amax, std::max(ks[i].inst_per_block, ks[i].mem_per_block));
    }
    while (gb > 1 && (u128)amax * gb * std::max(p.rb_num, p.rb_den) >= ((u128)1 << 63)) { /* keep den*A*g < 2^63 */
        uint64_t d = 2;
        while (gb % d) d++;
        gb /= d;
    }
    if (c && c->no_reduce) gb = 1;
    const uint32_t Sred = (uint32_t)(p.n_sm / gb);
    if ((p.flags & RK_FLAGS_POLICY) && Sred > RK_SMAX)
        return fail(c, RK_EUNSUPPORTED, "strict round robin / skip-ahead need a reduced SM count <= %u (got %u)",
                    (unsigned)RK_SMAX, Sred);
    /* Sred <= RK_SMAX: per-SM register state; larger: run-length state (SMAX = 0) */
    const uint64_t R = p.regs_per_sm / gr, Sh = p.shm_bytes_per_sm / gs;
    if (R > 32767 || Sh > 32767)
        return fail(c, RK_EUNSUPPORTED, "scaled regs %llu / shm %llu exceed the 15-bit packing", (unsigned long long)R,
                    (unsigned long long)Sh);
    std::memset(&t, 0, sizeof t);
    RkGTab& g = t.g;
    g.S = Sred;
    g.blkscale = (uint32_t)gb;
    g.num = p.rb_num;
    g.den = p.rb_den;
    g.freshA = (uint32_t)(2 * R + 1) | (uint32_t)(2 * Sh + 1) << 16;
    g.freshB = (uint32_t)(2 * p.max_warps_per_sm + 1) | (uint32_t)(2 * p.max_blocks_per_sm + 1) << 16;
    g.smagic = Sred > 1 ? (uint32_t)(((1ull << 32) + Sred - 1) / Sred) : 0u;
    /* binary search over t in [0, N_blk_SM - 1]: top bit = smallest power of two
     * with 2*tb >= N_blk_SM (0 when N_blk_SM == 1: t is always 0) */
    uint32_t tb = 0;
    if (p.max_blocks_per_sm > 1) {
        tb = 1;
        while (2 * tb < p.max_blocks_per_sm) tb *= 2;
    }
    g.tbits = tb;
    g.n = n;
    g.flags = p.flags;
    for (uint32_t i = 0; i <= RK_MAX_N; i++) g.fact[i] = fact64(i);
    const uint64_t caps[3] = {R, Sh, p.max_warps_per_sm};
    for (uint32_t i = 0; i < n; i++) {
        const uint64_t dem[3] = {d[i].regs / gr, d[i].shm / gs, d[i].warps};
        uint32_t mag[3], add[3];
        uint64_t C = p.max_blocks_per_sm;
        for (int r = 0; r < 3; r++) {
            if (dem[r] == 0) { /* numerator forced >= 2^30: quotient exceeds any cap */
                mag[r] = 0xFFFFFFFFu;
                add[r] = r == 0 ? 0x7FFF0000u : 0x7FFFu;
                continue;
            }
            C = std::min<uint64_t>(C, caps[r] / dem[r]);
            const uint64_t D = 2 * dem[r];
            const uint64_t m = ((1ull << 32) + D - 1) / D; /* ceil(2^32 / 2d) <= 2^31 */
            /* floor((2x+1)*m / 2^32) == floor(x/d) for all x <= cap: guaranteed when
             * (2cap+1)*e < 2^32 (e = m*2d - 2^32; the odd numerator keeps frac <=
             * (2d-1)/2d), otherwise checked exhaustively */
            const uint64_t e = m * D - (1ull << 32);
            if ((2 * caps[r] + 1) * e >= (1ull << 32))
                for (uint64_t x = 0; x <= caps[r]; x++)
                    if ((((2 * x + 1) * m) >> 32) != x / dem[r])
                        return fail(c, RK_EUNSUPPORTED, "kernel %u: no exact 32-bit magic for demand %llu", i,
                                    (unsigned long long)dem[r]);
            mag[r] = (uint32_t)m;
            add[r] = 0;
        }
        RkKTab& k = t.k[i];
        k.T = (uint32_t)(ks[i].grid_blocks / gb);
        k.mr = mag[0];
        k.ms = mag[1];
        k.mw = mag[2];
        k.zr = add[0];
        k.zs = add[1];
        k.dA = (uint32_t)(2 * dem[0]) | (uint32_t)(2 * dem[1]) << 16;
        k.dB = (uint32_t)(2 * dem[2]) | 2u << 16;
        const uint64_t Ared = (uint64_t)ks[i].inst_per_block * gb, Mred = (uint64_t)ks[i].mem_per_block * gb;
        k.cA = Ared * p.rb_den; /* < 2^63 by the key bound */
        k.cM = Mred * p.rb_num;
        k.C = (uint32_t)C;
        k.SC = (uint32_t)(C * Sred);
        k.scm = 0;
        if (k.SC >= 2) { /* floor(x/SC) = hi(x*scm) for x < T: verified bound x*e < 2^32 */
            const uint64_t m = ((1ull << 32) + k.SC - 1) / k.SC, e = m * k.SC - (1ull << 32);
            if ((uint64_t)k.T * e < (1ull << 32)) k.scm = (uint32_t)m;
        }
        const u128 ci = (u128)k.SC * k.cA, cm = (u128)k.SC * k.cM;
        const u128 fk = ci >= cm ? ci : cm;
        k.fullkey = fk >> 64 ? ~0ull : (uint64_t)fk; /* only used when T > SC, then bounded */
    }
    return RK_OK;
}

/* ------------------------- Algorithm 1 (host) ---------------------------- */
/* PAPER:110-198 with the readings of DESIGN.md §3 (L2 footprints, L16 ties /
 * infeasible / no-pair / odd n, L17 insertion, L18 inclusive straddle, L19).
 * Double arithmetic in the fixed order: shm, regs, warps slack, then bonus. */
struct Prof {
    uint64_t shm, regs, warps, blocks; /* per-SM footprint (reading L2) */
    double inst, ratio;
};

struct Alg1 {
    const rk_gpu_params& p;
    double RB;
    explicit Alg1(const rk_gpu_params& gp) : p(gp), RB((double)gp.rb_num / (double)gp.rb_den) {}

    Prof footprint(const rk_kernel& k) const {
        const uint64_t per_sm = (k.grid_blocks + p.n_sm - 1) / p.n_sm; /* ceil(N_tblk/N_SM) */
        const Derived d = derive(k);
        Prof f;
        f.shm = d.shm * per_sm;
        f.regs = d.regs * per_sm;
        f.warps = d.warps * per_sm;
        f.blocks = per_sm;
        f.inst = (double)k.grid_blocks * (double)k.inst_per_block;   /* N_inst_i */
        f.ratio = (double)k.inst_per_block / (double)k.mem_per_block; /* R_i */
        return f;
    }
    static Prof combine(const Prof& a, const Prof& b) { /* ProfileCombine */
        Prof c;
        c.shm = a.shm + b.shm;
        c.regs = a.regs + b.regs;
        c.warps = a.warps + b.warps;
        c.blocks = a.blocks + b.blocks;
        c.inst = a.inst + b.inst;
        c.ratio = (a.inst + b.inst) / (a.inst / a.ratio + b.inst / b.ratio);
        return c;
    }
    bool fits(const Prof& a, const Prof& b) const { /* PAPER:141 + slots */
        return a.shm + b.shm <= p.shm_bytes_per_sm && a.regs + b.regs <= p.regs_per_sm &&
               a.warps + b.warps <= p.max_warps_per_sm && a.blocks + b.blocks <= p.max_blocks_per_sm;
    }
    static double slack(uint64_t cap, uint64_t x, uint64_t y) {
        const double v = (double)((int64_t)cap - (int64_t)x - (int64_t)y) / (double)cap;
        return v > 0.0 ? v : 0.0;
    }
    double score(const Prof& a, const Prof& b) const { /* ScoreGen body */
        double s = 0.0;
        s += slack(p.shm_bytes_per_sm, a.shm, b.shm);
        s += slack(p.regs_per_sm, a.regs, b.regs);
        s += slack(p.max_warps_per_sm, a.warps, b.warps);
        const bool straddle = (a.ratio <= RB && RB <= b.ratio) || (b.ratio <= RB && RB <= a.ratio);
        if (straddle) {
            const double rc = (a.inst + b.inst) / (a.inst / a.ratio + b.inst / b.ratio);
            const double bonus = 1.0 - std::fabs(rc - RB) / RB;
            s += bonus > 0.0 ? bonus : 0.0;
        }
        return s;
    }

    void run(const rk_kernel* ks, uint32_t n, int32_t* order, int32_t* round_of) const {
        std::vector<Prof> f(n);
        for (uint32_t i = 0; i < n; i++) f[i] = footprint(ks[i]);
        std::vector<char> used(n, 0);
        uint32_t left = n, pos = 0;
        int32_t r = 0;
        auto emit = [&](const std::vector<uint32_t>& rd) {
            for (uint32_t x : rd) {
                order[pos] = (int32_t)x;
                if (round_of) round_of[pos] = r;
                pos++;
                used[x] = 1;
                left--;
            }
            r++;
        };
        while (left > 0) {
            if (left == 1) { /* lone kernel: singleton round */
                for (uint32_t i = 0; i < n; i++)
                    if (!used[i]) emit({i});
                break;
            }
            int ba = -1, bb = -1;
            double bs = 0.0;
            for (uint32_t a = 0; a < n; a++) {
                if (used[a]) continue;
                for (uint32_t b = a + 1; b < n; b++) {
                    if (used[b] || !fits(f[a], f[b])) continue;
                    const double sc = score(f[a], f[b]);
                    if (ba < 0 || sc > bs) {
                        ba = (int)a;
                        bb = (int)b;
                        bs = sc;
                    }
                }
            }
            if (ba < 0) { /* no feasible pair: singletons by decreasing shm, index order on ties */
                std::vector<uint32_t> rest;
                for (uint32_t i = 0; i < n; i++)
                    if (!used[i]) rest.push_back(i);
                std::stable_sort(rest.begin(), rest.end(),
                                 [&](uint32_t x, uint32_t y) { return f[x].shm > f[y].shm; });
                for (uint32_t x : rest) emit({x});
                break;
            }
            std::vector<uint32_t> rd;
            if (f[bb].shm > f[ba].shm) rd = {(uint32_t)bb, (uint32_t)ba};
            else rd = {(uint32_t)ba, (uint32_t)bb};
            used[ba] = used[bb] = 1; /* removed from K */
            Prof comb = combine(f[ba], f[bb]);
            for (;;) {
                int bc = -1;
                double cs = 0.0;
                for (uint32_t x = 0; x < n; x++) {
                    if (used[x] || !fits(comb, f[x])) continue;
                    const double sc = score(comb, f[x]);
                    if (bc < 0 || sc > cs) {
                        bc = (int)x;
                        cs = sc;
                    }
                }
                if (bc < 0) break;
                auto it = rd.begin();
                while (it != rd.end() && f[*it].shm >= f[bc].shm) ++it; /* stable decreasing shm */
                rd.insert(it, (uint32_t)bc);
                comb = combine(comb, f[bc]);
                used[bc] = 1;
            }
            for (uint32_t x : rd) used[x] = 0; /* emit() re-marks and counts them */
            emit(rd);
        }
    }
};

/* ----------------------- rank / unrank (Lehmer) --------------------------- */
rk_status do_rank(const int32_t* order, uint32_t n, uint64_t* idx) {
    if (n < 1 || n > 20) return RK_EINVAL;
    uint32_t seen = 0;
    uint64_t v = 0;
    for (uint32_t j = 0; j < n; j++) {
        const int32_t x = order[j];
        if (x < 0 || (uint32_t)x >= n || (seen >> x & 1u)) return RK_EINVAL;
        /* digit = number of unused values smaller than x */
        const uint32_t smaller_unused = (uint32_t)__builtin_popcount(~seen & ((1u << x) - 1u));
        v = v * (n - j) + smaller_unused;
        seen |= 1u << x;
    }
    *idx = v;
    return RK_OK;
}

rk_status do_unrank(uint64_t idx, uint32_t n, int32_t* out) {
    if (n < 1 || n > 20 || idx >= fact64(n)) return RK_EINVAL;
    uint32_t digits[20];
    for (uint32_t j = n; j-- > 0;) { /* factorial base, least significant first */
        const uint32_t base = n - j;
        digits[j] = (uint32_t)(idx % base);
        idx /= base;
    }
    uint32_t unused = (n == 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
    for (uint32_t j = 0; j < n; j++) {
        uint32_t m = unused;
        for (uint32_t q = 0; q < digits[j]; q++) m &= m - 1; /* drop the lowest set bits */
        const uint32_t x = (uint32_t)__builtin_ctz(m);
        out[j] = (int32_t)x;
        unused &= ~(1u << x);
    }
    return RK_OK;
}

rk_status need_device(rk_ctx* c) {
    if (!c) return RK_EINVAL;
    if (c->device < 0) return fail(c, RK_ENODEVICE, "host-only context: no device evaluation (no CPU fallback)");
    return RK_OK;
}

rk_status need_kernels(rk_ctx* c) {
    if (!c->has_params || !c->has_kernels) return fail(c, RK_ESTATE, "call rk_set_gpu_params and rk_set_kernels first");
    return RK_OK;
}

uint64_t space(const rk_ctx* c) { return fact64((uint32_t)c->ks.size()); }

/* phase timing: begin returns a mark (or -1 when off), end records its second event */
int tmark_begin(rk_ctx* c, uint32_t phase, void* stream) {
    if (!c->timing) return -1;
    if (c->tused == c->tphase.size()) {
        cudaEvent_t a = nullptr, b = nullptr;
        if (cudaEventCreate(&a) || cudaEventCreate(&b)) return -1;
        c->tev.push_back(a);
        c->tev.push_back(b);
        c->tphase.push_back(phase);
    }
    const size_t m = c->tused++;
    c->tphase[m] = phase;
    cudaEventRecord(c->tev[2 * m], (cudaStream_t)stream);
    return (int)m;
}
void tmark_end(rk_ctx* c, int m, void* stream) {
    if (m >= 0) cudaEventRecord(c->tev[2 * (size_t)m + 1], (cudaStream_t)stream);
}

void dp_free(DpPlan& d) {
    d.nodes.release();
    d.tables.release();
    d.tid.release();
    d.dk.release();
    d.fst.release();
    d.counters.release();
    for (Arena* a : {&d.code, &d.dvc, &d.dvp, &d.nd, &d.offs, &d.row24, &d.expand, &d.meta_u, &d.meta_K, &d.rslot, &d.rmult, &d.rlist, &d.rminrun, &d.rwlist, &d.rwminrun, &d.pslot, &d.pmult, &d.pminrun}) a->release();
    d.runs_ok = false;
    d.on = false;
}

uint32_t pow2_at_least(uint64_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

/* Enqueue levels j0..j1-1 of the plan's table build (level j reads level j's
 * nodes and count, writes level j+1). */
/* levels whose items (and expansion entries) stay under this go several to one cooperative launch */
constexpr uint64_t kCoopItems = 1u << 16;
int launch_level_run(rk_ctx* c, std::vector<RkLevel>& lv, void* stream) {
    /* consecutive small levels share one cooperative launch (<= 8), the others get one launch each */
    int e = 0;
    for (size_t i = 0; i < lv.size() && !e;) {
        size_t j = i + 1;
        auto small = [&](const RkLevel& l) { return l.work <= kCoopItems && (!l.ex || l.ex->cnt <= kCoopItems); };
        if (!c->no_coop && small(lv[i]))
            while (j < lv.size() && j - i < 8 && small(lv[j])) j++;
        e = rk_dp_levels(c->tab_dev, c->tab.g.S, lv.data() + i, (uint32_t)(j - i), stream, &c->launches);
        i = j;
    }
    return e;
}

int dp_levels(rk_ctx* c, uint32_t j0, uint32_t j1, void* stream, const std::vector<RkExpand>* ex = nullptr) {
    DpPlan& d = c->dp;
    const uint32_t n = c->tab.g.n;
    char* nodes = (char*)d.nodes.p;
    uint32_t* ctr = (uint32_t*)d.counters.p;
    std::vector<RkLevel> lv;
    for (uint32_t j = j0; j < j1; j++) {
        /* the launch of level j also expands the range's prefixes of level j-1 -> j */
        const RkExpand* x = (ex && j >= 1 && j < d.P && j - 1 < ex->size()) ? &(*ex)[j - 1] : nullptr;
        lv.push_back(RkLevel{j ? nodes + d.noff[j] : nullptr, j ? ctr + j : nullptr, nodes + d.noff[j + 1],
                             ctr + j + 1, d.cap[j + 1], (uint32_t*)d.tables.p + d.toff[j + 1], d.tmask[j + 1],
                             (uint32_t*)d.tid.p + d.xoff[j], (uint64_t*)d.dk.p + d.xoff[j], ctr + d.L + 1, x, n - j,
                             d.work[j] / n * (n - j)});
    }
    /* the leading levels small enough for one CTA (shared-memory dedup) go to one launch */
    size_t J = 0;
    const uint32_t im = (j0 == 0 && !c->no_coop) ? rk_dp_small_items_max(c->tab.g.S) : 0u;
    while (im && J < lv.size() && J < 4 && lv[J].work <= im) J++;
    int e = 0;
    if (J >= 2) {
        e = rk_dp_small_levels(c->tab_dev, c->tab.g.S, lv.data(), (uint32_t)J, im, stream, &c->launches);
        lv.erase(lv.begin(), lv.begin() + J);
    }
    if (!e) e = launch_level_run(c, lv, stream);
    return e;
}

/* Enqueue the level build of the current plan: clear, P levels (+ the given
 * prefix expansions, level j-1 -> j in level j's launch; the last one runs in
 * the run pass). */
int dp_build_levels(rk_ctx* c, void* stream, const std::vector<RkExpand>* ex = nullptr, uint32_t upto = ~0u) {
    DpPlan& d = c->dp;
    cudaStream_t st = (cudaStream_t)stream;
    int e = cudaMemsetAsync(d.tables.p, 0xFF, d.table_slots * 4, st);
    if (!e) e = cudaMemsetAsync(d.counters.p, 0, (d.L + 4) * 4, st); /* + the overflow flag, the row list counters */
    if (!e) e = dp_levels(c, 0, std::min(upto, d.L), stream, ex);
    return e;
}

/* Enqueue the suffix rows of the level-P nodes (after the levels): the 24-key
 * rows of the level-(P+1) nodes, then per level-P node its 120 keys gathered
 * through the level-P transitions and encoded. */
int dp_build_suffix(rk_ctx* c, void* stream) {
    DpPlan& d = c->dp;
    const std::vector<size_t>& noff = d.last_ub ? d.ub_noff : d.noff;
    int e = rk_dp_row24(c->tab_dev, c->tab.g.S, (char*)d.nodes.p + noff[d.L], (uint32_t*)d.counters.p + d.L,
                        (uint64_t*)d.row24.p, d.cnt[d.L], stream, &c->launches);
    if (!e)
        e = rk_dp_suffix(c->tab_dev, c->tab.g.S, (char*)d.nodes.p + noff[d.P], (uint32_t*)d.counters.p + d.P,
                         d.view.tid[d.P], d.view.dk[d.P], (const uint64_t*)d.row24.p, (uint8_t*)d.code.p, d.dvc.p,
                         d.dvp.p, (uint32_t*)d.nd.p, (uint64_t*)d.fst.p, (uint32_t*)d.offs.p, d.cnt[d.P], stream,
                         &c->launches);
    return e;
}

/* the ctx's side streams and their fork/join events: pass 2's counts/histogram at high priority (they
 * should slip in beside the HBM-bound key stream), pass 1's run pass at the default priority (the suffix
 * rows on the main stream are the longer chain); RK_SIDE_PRIO=0|1 puts both at default|high (testing) */
int ensure_side(rk_ctx* c) {
    if (c->side) return 0;
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const char* pr = getenv("RK_SIDE_PRIO");
    const int p2 = (pr && pr[0] == '0') ? lo : hi, p1 = (pr && pr[0] == '1') ? hi : lo;
    int e = cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, p2);
    if (!e) e = cudaStreamCreateWithPriority(&c->side1, cudaStreamNonBlocking, p1);
    if (!e) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    if (!e) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
    return e;
}

constexpr uint64_t kLimitEntries = 1ull << 26, kLimitBytes = 1ull << 31;

/* Level layout from per-level node counts (or upper bounds) m[0..P]: level j's
 * transitions m[j]*n, level j+1's capacity cap[j+1] and a hash table of
 * pow2(2*cap) slots.  Grow-only arenas (no copy unless keep_nodes: every
 * build rewrites them).
 * false = over the size limits (memoisation off). */
bool dp_layout(rk_ctx* c, const std::vector<uint64_t>& m, const std::vector<uint64_t>& cap, int& e,
               bool keep_nodes = false) {
    DpPlan& d = c->dp;
    const uint32_t n = c->tab.g.n;
    size_t nb = 0, ts = 0, xs = 0, tb = 0;
    for (uint32_t j = 0; j < d.L; j++) {
        const uint64_t work = m[j] * n, capn = cap[j + 1];
        const uint64_t slots = pow2_at_least(2 * capn);
        if (work > kLimitEntries || capn * d.node_bytes > kLimitBytes || slots > kLimitEntries) return false;
        d.work[j] = work;
        d.xoff[j] = xs;
        xs += work;
        d.noff[j + 1] = nb;
        d.cap[j + 1] = (uint32_t)capn;
        nb = (nb + capn * d.node_bytes + 255) & ~(size_t)255;
        d.toff[j + 1] = ts;
        d.tmask[j + 1] = (uint32_t)(slots - 1);
        ts += slots;
    }
    tb = nb + ts * 4 + xs * 12;
    if (tb > 3 * kLimitBytes) return false;
    d.table_slots = ts;
    e = d.nodes.reserve(nb, keep_nodes ? d.nodes.cap : 0); /* level-by-level: earlier levels stay */
    if (!e) e = d.tables.reserve(ts * 4);
    if (!e) e = d.tid.reserve(xs * 4);
    if (!e) e = d.dk.reserve(xs * 8);
    return true;
}

/* Find the exact per-level node counts.  Fast path: all P levels in one go with
 * upper-bound capacities (level j+1 holds at most min(n!/(n-j-1)!, 2^22)
 * distinct nodes) and ONE synchronous read of the counts; a capped level that
 * overflows (flag, probe guard) falls back to the level-by-level build whose
 * capacities come from the previous level's exact count.  Then the exact
 * layout the steps use.  Every rk_set_kernels re-plans (no cache), so the
 * first step on a new kernel set costs what a repeated one does plus this
 * plan.  Off (direct evaluation) for the run-length state, n < 6, the policy
 * readings, or when it would not pay. */
rk_status dp_plan(rk_ctx* c) {
    DpPlan& d = c->dp;
    d.on = false;
    d.runs_ok = false;
    const uint32_t n = c->tab.g.n, S = c->tab.g.S;
    if (c->device < 0 || c->no_memo || c->force_runs || policy(c) || n < RK_DP_D + 1)
        return RK_OK; /* S > 32: run-length nodes; policies: per-order kernels */
    d.P = n - RK_DP_D;
    d.L = d.P + 1;
    d.node_bytes = rk_dp_node_bytes(S);
    d.cnt.assign(d.L + 1, 0);
    d.cap.assign(d.L + 1, 0);
    d.noff.assign(d.L + 1, 0);
    d.toff.assign(d.L + 1, 0);
    d.tmask.assign(d.L + 1, 0);
    d.xoff.assign(d.L + 1, 0);
    d.work.assign(d.L + 1, 0);
    d.cnt[0] = 1;
    d.view = DPView{};
    int e = d.counters.reserve(64 * 4);
    bool counted = false;
    {   /* fast path: upper-bound capacities, one sync */
        std::vector<uint64_t> ub(d.L + 1, 1);
        for (uint32_t j = 0; j < d.L; j++) ub[j + 1] = std::min<uint64_t>(ub[j] * (n - j), 1ull << 22);
        if (!e && dp_layout(c, ub, ub, e) && !e) {
            e = cudaMemset(d.tables.p, 0xFF, d.table_slots * 4);
            if (!e) e = cudaMemset(d.counters.p, 0, 64 * 4);
            if (!e) e = dp_levels(c, 0, d.L, nullptr);
            std::vector<uint32_t> h(d.L + 2, 0); /* counts of levels 0..L, the overflow flag at L+1 */
            if (!e) e = cudaMemcpy(h.data(), d.counters.p, (d.L + 2) * 4, cudaMemcpyDeviceToHost);
            if (!e && !h[d.L + 1]) {
                counted = true;
                for (uint32_t j = 1; j <= d.L; j++) {
                    d.cnt[j] = h[j];
                    counted = counted && h[j] <= ub[j];
                }
                d.ub_noff = d.noff;
                d.ub_xoff = d.xoff;
                d.ub_toff = d.toff;
                d.ub_cap = d.cap;
                d.ub_tmask = d.tmask;
            }
        }
    }
    if (!e && !counted) { /* level by level, exact capacities */
        std::vector<uint64_t> m(d.L + 1, 0), cap(d.L + 1, 0);
        m[0] = 1;
        e = cudaMemset(d.counters.p, 0, 64 * 4);
        for (uint32_t j = 0; j < d.L && !e; j++) {
            cap[j + 1] = m[j] * (n - j);
            for (uint32_t q = j + 1; q <= d.L; q++) m[q] = q == j + 1 ? cap[j + 1] : 1;
            std::vector<uint64_t> cq(d.L + 1, 1);
            for (uint32_t q = 1; q <= j + 1; q++) cq[q] = cap[q];
            if (!dp_layout(c, m, cq, e, true) || e) return e ? cuda_fail(c, e, "memoisation plan") : RK_OK;
            e = cudaMemset((uint32_t*)d.tables.p + d.toff[j + 1], 0xFF, (d.tmask[j + 1] + 1ull) * 4);
            if (!e) e = dp_levels(c, j, j + 1, nullptr);
            uint32_t h[2] = {0, 0}; /* level j+1 count; the overflow flag lives at P+1 */
            if (!e) e = cudaMemcpy(&h[0], (uint32_t*)d.counters.p + j + 1, 4, cudaMemcpyDeviceToHost);
            if (!e) e = cudaMemcpy(&h[1], (uint32_t*)d.counters.p + d.L + 1, 4, cudaMemcpyDeviceToHost);
            if (e) break;
            if (h[0] > cap[j + 1] || h[1]) return RK_OK; /* cannot happen: capacity is an upper bound */
            m[j + 1] = d.cnt[j + 1] = h[0];
        }
    }
    if (e) {
        cudaGetLastError();
        return cuda_fail(c, e, "memoisation plan");
    }
    {   /* the exact layout of the steps: level j+1 capacity cnt[j] * (n - j) */
        std::vector<uint64_t> m(d.L + 1), cap(d.L + 1, 0);
        for (uint32_t j = 0; j <= d.L; j++) m[j] = d.cnt[j];
        for (uint32_t j = 0; j < d.L; j++) cap[j + 1] = (uint64_t)d.cnt[j] * (n - j);
        const void *np = d.nodes.p, *tp = d.tid.p, *kp = d.dk.p;
        if (!dp_layout(c, m, cap, e) || e) return e ? cuda_fail(c, e, "memoisation layout") : RK_OK;
        /* the upper-bound build is still intact unless an arena moved */
        d.reuse_ub = counted && np == d.nodes.p && tp == d.tid.p && kp == d.dk.p;
    }
    const uint64_t runs = fact64(n) / fact64(RK_DP_D), uP = d.cnt[d.P];
    const uint64_t DF = fact64(RK_DP_D);
    if (uP * DF * 8 > kLimitBytes) return RK_OK;
    if (uP * 4 > runs && !c->force_memo) return RK_OK; /* does not pay */
    e = d.code.reserve(uP * DF);
    if (!e) e = d.dvc.reserve(uP * DF * 16);
    if (!e) e = d.dvp.reserve(uP * DF * 8);
    if (!e) e = d.offs.reserve(uP * DF * 4);
    if (!e) e = d.nd.reserve(uP * 4);
    if (!e) e = d.fst.reserve(uP * 4 * 8);
    if (!e) e = d.row24.reserve((uint64_t)d.cnt[d.L] * 24 * 8 + 8);
    if (e) {
        cudaGetLastError();
        return cuda_fail(c, e, "memoisation buffers");
    }
    for (uint32_t j = 0; j < d.L; j++) {
        d.view.tid[j] = (const uint32_t*)d.tid.p + d.xoff[j];
        d.view.dk[j] = (const uint64_t*)d.dk.p + d.xoff[j];
    }
    d.view.code = (const uint8_t*)d.code.p;
    d.view.dvc = d.dvc.p;
    d.view.dvp = (const uint2*)d.dvp.p;
    d.view.offs = (const uint32_t*)d.offs.p;
    d.view.nd = (const uint32_t*)d.nd.p;
    d.view.fst = (const uint64_t*)d.fst.p;
    d.view.P = d.P;
    d.view.D = RK_DP_D;
    d.view.Dfact = (uint32_t)DF;
    d.on = true;
    return RK_OK;
}

/* the candidate key pointer, or a device zero (no candidate: every key counts as n_gt) */
const uint64_t* cand_or_zero(rk_ctx* c, const uint64_t* cand_dev, void* stream) {
    if (cand_dev) return cand_dev;
    cudaMemsetAsync(c->u64_dev + 9, 0, 8, (cudaStream_t)stream);
    return c->u64_dev + 9;
}

/* the range's row multiset buffers */
RkRows dp_rows(rk_ctx* c, uint64_t nrun) {
    DpPlan& d = c->dp;
    return RkRows{c->dedup_now ? d.rslot.p : nullptr, (uint32_t*)d.rmult.p, d.rmask, (uint32_t*)d.rlist.p,
                  (uint32_t*)d.counters.p + d.L + 2, nrun, (uint32_t*)d.rminrun.p, d.rwlist.p, (uint32_t*)d.rwminrun.p,
                  (uint32_t*)d.counters.p + d.L + 3};
}

/* Pass 1 of the memoised step: the levels rebuilt from scratch (the first
 * step after a plan runs over the plan's build) with the range's prefixes
 * expanded breadth-first (levels 1..P-1 when the range has <= 2^27 runs;
 * level P recomputed by the run pass); then, concurrently, level P+1, row24
 * and the suffix rows (main stream) and the run pass with the row multiset
 * (side stream: each run's (node, K_closed); parents and children multisets);
 * then the extremes from the distinct rows (the range's record: n_lt = n_eq =
 * 0, n_gt = evaluated = count).  RK_OVERLAP=0 keeps everything on the main
 * stream. */
int dp_pass1(rk_ctx* c, uint64_t first, uint64_t count, rk_stats* rec_dev, void* stream) {
    DpPlan& d = c->dp;
    d.runs_ok = false;
    /* the first step after the plan runs over the plan's build (upper-bound layout); later ones rebuild */
    const bool ub = d.reuse_ub;
    d.reuse_ub = false;
    d.last_ub = ub;
    for (uint32_t j = 0; j < d.L; j++) {
        d.view.tid[j] = (const uint32_t*)d.tid.p + (ub ? d.ub_xoff[j] : d.xoff[j]);
        d.view.dk[j] = (const uint64_t*)d.dk.p + (ub ? d.ub_xoff[j] : d.xoff[j]);
    }
    const uint32_t n = c->tab.g.n, P = d.P;
    const uint64_t DF = d.view.Dfact;
    const uint64_t rb = first / DF, re = count ? (first + count + DF - 1) / DF : rb;
    std::vector<RkExpand> ex;
    const uint64_t nrun = std::max<uint64_t>(re - rb, 1);
    cudaStream_t st = (cudaStream_t)stream;
    int e = d.meta_u.reserve(nrun * 4);
    if (!e) e = d.meta_K.reserve(nrun * 8);
    /* row multiset: ~8 runs per slot (C4: 217,659 distinct rows of 3,991,680 runs in 2^19 slots) */
    const uint64_t slots = std::min<uint64_t>(std::max<uint64_t>(pow2_at_least(nrun / 8), 4096), 1ull << 24); /* 16M slots: 13! has millions of distinct rows */
    d.rmask = (uint32_t)(slots - 1);
    if (!e) e = d.rslot.reserve(slots * 16);
    if (!e) e = d.rmult.reserve(slots * 4 * 8); /* 8 counters per slot */
    if (!e) e = d.rlist.reserve(nrun * 4);
    if (!e) e = d.rminrun.reserve(slots * 4);
    c->dedup_now = c->row_dedup != 0;
    const bool side = c->overlap != 0;
    if (!e && side) e = ensure_side(c);
    if (!e && re > rb && re - rb <= (1ull << 27)) {
        /* level j covers prefixes [a_j, b_j): span_j level-P prefixes under each */
        std::vector<uint64_t> a(P + 1), b(P + 1);
        uint64_t span = 1;
        for (int j = (int)P; j >= 0; j--) {
            a[j] = rb / span;
            b[j] = (re - 1) / span + 1;
            if (j > 0) span *= (n - (uint32_t)(j - 1));
        }
        std::vector<size_t> off(P + 1, 0);
        size_t tot = 0;
        for (uint32_t j = 1; j < P; j++) {
            off[j] = tot;
            tot += (b[j] - a[j]) * 16;
        }
        e = d.expand.reserve(std::max<size_t>(tot, 16));
        const void* prev = nullptr;
        for (uint32_t j = 0; j < P && !e; j++) {
            void* dst = j + 1 == P ? nullptr : (char*)d.expand.p + off[j + 1]; /* level P: not stored */
            ex.push_back(RkExpand{prev, a[j], dst, a[j + 1], b[j + 1] - a[j + 1], j, d.view.tid[j], d.view.dk[j]});
            prev = dst;
        }
    }
    /* the multiset from the stored level-(P-1) prefixes (parents, then children) when the range was expanded,
     * else run by run in the run pass */
    const bool hier = c->dedup_now && !ex.empty() && P >= 2;
    uint64_t pslots = 0;
    if (hier) {
        const uint64_t npar = ex.back().cnt ? (re - 1) / (n - P + 1) - ex.back().aj + 1 : 1;
        pslots = std::min<uint64_t>(std::max<uint64_t>(pow2_at_least(npar / 4), 4096), 1ull << 23);
        d.pmask = (uint32_t)(pslots - 1);
        if (!e) e = d.pslot.reserve(pslots * 16);
        if (!e) e = d.pmult.reserve(pslots * 32);
        if (!e) e = d.pminrun.reserve(pslots * 4);
        /* weighted rows without a slot: at most one per (parent slot, unused kernel) */
        if (!e) e = d.rwlist.reserve(pslots * (n - P + 1) * 16);
        if (!e) e = d.rwminrun.reserve(pslots * (n - P + 1) * 4);
    }
    const int m0 = tmark_begin(c, RK_PHASE_TABLES, stream);
    if (!e && hier) e = cudaMemsetAsync(d.pslot.p, 0, pslots * 16, st);
    if (!e && hier) e = cudaMemsetAsync(d.pmult.p, 0, pslots * 32, st);
    if (!e && hier) e = cudaMemsetAsync(d.pminrun.p, 0xFF, pslots * 4, st);
    if (!e && c->dedup_now) e = cudaMemsetAsync(d.rslot.p, 0, slots * 16, st);
    if (!e && c->dedup_now) e = cudaMemsetAsync(d.rmult.p, 0, slots * 32, st);
    if (!e && c->dedup_now) e = cudaMemsetAsync(d.rminrun.p, 0xFF, slots * 4, st);
    /* levels 0..P-1 (the run level's transitions and the range's expansions), then the run pass and the
     * multiset fork off beside the last level (P+1, for the suffix rows), row24 and the suffix rows */
    if (!e && !ub) e = dp_build_levels(c, stream, ex.empty() ? nullptr : &ex, P);
    if (!e && ub) { /* over the plan's levels: zero the list counters, expand the range's prefixes */
        e = cudaMemsetAsync((uint32_t*)d.counters.p + d.L + 2, 0, 8, st);
        std::vector<RkLevel> lv;
        for (uint32_t j = 1; j < P && j - 1 < ex.size(); j++)
            lv.push_back(RkLevel{nullptr, nullptr, nullptr, nullptr, 0, nullptr, 0, nullptr, nullptr,
                                 (uint32_t*)d.counters.p + d.L + 1, &ex[j - 1], 0, 0});
        if (!e) e = launch_level_run(c, lv, stream);
    }
    void* rs = side ? (void*)c->side1 : stream;
    if (!e && side) e = cudaEventRecord(c->ev_fork, st);
    if (!e && side) e = cudaStreamWaitEvent(c->side1, c->ev_fork, 0);
    if (!e && !side && !ub) e = dp_levels(c, P, d.L, stream, nullptr);
    const int mr = tmark_begin(c, RK_PHASE_RUNS, rs);
    RkRows runrows = dp_rows(c, re - rb);
    if (hier) runrows.slot = nullptr; /* the run pass writes the run metadata only */
    if (!e)
        e = rk_dp_runs(c->tab_dev, d.view, first, count, (uint32_t*)d.meta_u.p, (uint64_t*)d.meta_K.p, runrows,
                       ex.empty() ? nullptr : &ex.back(), rs, &c->launches);
    if (!e && hier) {
        const RkExpand& lx = ex.back();
        RkExpand parent_level = lx;
        parent_level.Rj = ex[P - 1].Rj; /* the stored level-(P-1) prefixes */
        const RkRows parents{d.pslot.p, (uint32_t*)d.pmult.p, d.pmask, nullptr, nullptr, 0, (uint32_t*)d.pminrun.p,
                             nullptr, nullptr, nullptr};
        e = rk_dp_multiset(n, first, count, &parent_level, parents, dp_rows(c, re - rb), rs, &c->launches);
    }
    tmark_end(c, mr, rs);
    if (!e && side) e = cudaEventRecord(c->ev_join, c->side1);
    if (!e && side && !ub) e = dp_levels(c, P, d.L, stream, nullptr);
    if (!e) e = dp_build_suffix(c, stream);
    tmark_end(c, m0, stream);
    if (!e && side) e = cudaStreamWaitEvent(st, c->ev_join, 0);
    const int m1 = tmark_begin(c, RK_PHASE_EXTREMES, stream);
    if (!e)
        e = rk_dp_ext(d.view, first, count, dp_rows(c, re - rb), (const uint32_t*)d.meta_u.p,
                      (const uint64_t*)d.meta_K.p, rec_dev, c->recs_dev, c->counter_dev, c->max_ctas, stream,
                      &c->launches);
    tmark_end(c, m1, stream);
    if (!e) {
        d.runs_ok = true;
        d.runs_first = first;
        d.runs_count = count;
    }
    return e;
}

/* Pass 2 over the range of the preceding pass 1: the key stream from its run
 * metadata (keys_dev), then the counts (into rec_dev) and the histogram
 * (hist_dev, bins <= rk_dp_max_fused_bins()) from the distinct rows (or every
 * run with the multiset off); with keys they run beside the key stream on the
 * ctx's high-priority side stream (RK_OVERLAP=0: after it). */
int dp_pass2(rk_ctx* c, uint64_t first, uint64_t count, const uint64_t* cand_dev, const rk_stats* range_dev,
             uint32_t bins, uint64_t* hist_dev, uint64_t* keys_dev, rk_stats* rec_dev, void* stream,
             uint32_t* keys32 = nullptr, uint64_t key_base = 0, uint32_t* ovf = nullptr) {
    DpPlan& d = c->dp;
    if (!(d.runs_ok && d.runs_first == first && d.runs_count == count)) return (int)cudaErrorNotReady;
    const uint32_t* mu = (const uint32_t*)d.meta_u.p;
    const uint64_t* mk = (const uint64_t*)d.meta_K.p;
    const uint64_t DF = d.view.Dfact;
    const uint64_t nrun = count ? (first + count + DF - 1) / DF - first / DF : 0;
    cudaStream_t st = (cudaStream_t)stream;
    const bool keys = (keys_dev || keys32) && count;
    const bool ov = keys && c->overlap != 0;
    int e = ov ? ensure_side(c) : 0;
    auto rows = [&](void* s, uint32_t cap) {
        const int m = tmark_begin(c, RK_PHASE_HIST, s);
        const int r = rk_dp_rows(c->tab_dev, d.view, first, count, cand_dev, range_dev, bins, hist_dev,
                                 dp_rows(c, nrun), mu, mk, rec_dev, cap, s, &c->launches);
        tmark_end(c, m, s);
        return r;
    };
    if (!e && ov) {
        e = cudaEventRecord(c->ev_fork, st);
        if (!e) e = cudaStreamWaitEvent(c->side, c->ev_fork, 0);
        if (!e) e = rows(c->side, c->rows_ctas * c->sms);
    }
    if (!e && keys) {
        const int m1 = tmark_begin(c, RK_PHASE_STREAM, stream);
        e = keys32 ? rk_dp_keys32(d.view, first, count, mu, mk, keys32, key_base, ovf, range_dev, stream, &c->launches)
                   : rk_dp_keys(d.view, first, count, mu, mk, keys_dev, stream, &c->launches);
        tmark_end(c, m1, stream);
    }
    if (!e && !ov) e = rows(stream, 0);
    if (!e && ov) {
        e = cudaEventRecord(c->ev_join, c->side);
        if (!e) e = cudaStreamWaitEvent(st, c->ev_join, 0);
    }
    return e;
}

/* memoised equivalent of rk_launch_eval (stats + optional keys, optional histogram) */
/* memoised stats (+ optional keys, optional histogram over a given range) of [first, first+count); ranges of
 * more than kChunkRuns runs go in chunks of whole runs (pass 1 + pass 2 each, records merged on the device),
 * so the per-run scratch (run metadata, multiset lists: ~36 B per run) stays bounded */
constexpr uint64_t kChunkRuns = 1ull << 26;
int dp_eval(rk_ctx* c, uint64_t first, uint64_t count, const uint64_t* cand_dev, rk_stats* stats_dev,
            uint64_t* keys_dev, const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, void* stream) {
    const uint64_t DF = c->dp.view.Dfact;
    const uint64_t nrun = count ? (first + count + DF - 1) / DF - first / DF : 0;
    if (nrun <= kChunkRuns) {
        int e = dp_pass1(c, first, count, stats_dev, stream);
        if (!e) e = dp_pass2(c, first, count, cand_dev, range_dev, bins, hist_dev, keys_dev, stats_dev, stream);
        return e;
    }
    /* chunk records at u64_dev[16..], the running merge at stats_dev (2-record merges) */
    rk_stats* part = reinterpret_cast<rk_stats*>(c->u64_dev + 16);
    int e = 0;
    for (uint64_t lo = first, end = first + count; lo < end && !e;) {
        const uint64_t hi = std::min(end, (lo / DF + kChunkRuns) * DF);
        rk_stats* out = lo == first ? stats_dev : part + 1;
        e = dp_pass1(c, lo, hi - lo, out, stream);
        if (!e)
            e = dp_pass2(c, lo, hi - lo, cand_dev, range_dev, bins, hist_dev, keys_dev ? keys_dev + (lo - first) : nullptr,
                         out, stream);
        if (!e && lo != first) { /* stats_dev <- merge(stats_dev, chunk) */
            e = cudaMemcpyAsync(part, stats_dev, sizeof(rk_stats), cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
            if (!e) e = rk_launch_merge(part, 2, stats_dev, stream, &c->launches);
        }
        lo = hi;
    }
    return e;
}

}  // namespace

/* ================================ C ABI ================================== */
extern "C" {

rk_status rk_create(rk_ctx** out, int cuda_device) {
    if (!out) return RK_EINVAL;
    rk_ctx* c = new rk_ctx();
    c->device = cuda_device;
    const char* nr = getenv("RK_NO_REDUCE");
    c->no_reduce = nr && nr[0] == '1';
    const char* fr = getenv("RK_FORCE_RUNS");
    c->force_runs = fr && fr[0] == '1';
    const char* nm = getenv("RK_NO_MEMO");
    c->no_memo = nm && nm[0] == '1';
    const char* nc = getenv("RK_NO_COOP");
    c->no_coop = nc && nc[0] == '1';
    const char* fm = getenv("RK_FORCE_MEMO");
    c->force_memo = fm && fm[0] == '1';
    const char* rd = getenv("RK_ROW_DEDUP");
    if (rd && (rd[0] == '0' || rd[0] == '1')) c->row_dedup = rd[0] - '0';
    const char* ovv = getenv("RK_OVERLAP");
    if (ovv && (ovv[0] == '0' || ovv[0] == '1')) c->overlap = ovv[0] - '0';
    const char* rc = getenv("RK_ROWS_CTAS");
    if (rc && atoi(rc) > 0) c->rows_ctas = (uint32_t)atoi(rc);
    if (cuda_device >= 0) {
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || cuda_device >= ndev) {
            delete c;
            return RK_ENODEVICE;
        }
        DeviceGuard dg(cuda_device);
        c->max_ctas = 0;
        for (uint32_t S : {1u, 2u, 3u, 4u, 5u, 8u, 9u, 16u, 17u, 32u, 33u})
            c->max_ctas = std::max(c->max_ctas, (uint32_t)rk_eval_max_ctas(S, cuda_device));
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
        c->sms = sms > 0 ? (uint32_t)sms : 148u;
        /* the batch calls' stream-ordered buffers stay in the device's default pool between calls */
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, cuda_device) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        /* per-CTA record slots: also for the memo extremes pass (8 CTAs per SM) */
        c->max_ctas = std::max<uint32_t>(c->max_ctas, (uint32_t)std::max(256, 8 * sms));
        bool ok = cudaMalloc(&c->tab_dev, sizeof(RkTables)) == cudaSuccess &&
                  cudaMalloc(&c->recs_dev, sizeof(rk_stats) * c->max_ctas * 2) == cudaSuccess &&
                  cudaMalloc(&c->counter_dev, sizeof(uint32_t)) == cudaSuccess &&
                  cudaMalloc(&c->stats_dev, sizeof(rk_stats)) == cudaSuccess &&
                  cudaMalloc(&c->u64_dev, sizeof(uint64_t) * 64) == cudaSuccess &&
                  cudaMemset(c->counter_dev, 0, sizeof(uint32_t)) == cudaSuccess &&
                  cudaDeviceSynchronize() == cudaSuccess;
        if (!ok) {
            rk_destroy(c);
            return RK_ECUDA;
        }
    }
    *out = c;
    return RK_OK;
}

void rk_destroy(rk_ctx* c) {
    if (!c) return;
    if (c->device >= 0) {
        DeviceGuard dg(c->device);
        dp_free(c->dp);
        cudaFree(c->tab_dev);
        cudaFree(c->recs_dev);
        cudaFree(c->counter_dev);
        cudaFree(c->stats_dev);
        cudaFree(c->u64_dev);
        cudaFree(c->batch_scratch);
        if (c->pin) cudaFreeHost(c->pin);
        for (cudaEvent_t ev : c->tev) cudaEventDestroy(ev);
        if (c->side) {
            cudaStreamDestroy(c->side);
            cudaStreamDestroy(c->side1);
            cudaEventDestroy(c->ev_fork);
            cudaEventDestroy(c->ev_join);
        }
    }
    delete c;
}

const char* rk_last_error(const rk_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

uint32_t rk_last_launch_count(const rk_ctx* c) { return c ? c->launches : 0; }

rk_status rk_set_gpu_params(rk_ctx* c, const rk_gpu_params* p) {
    if (!c || !p) return RK_EINVAL;
    rk_status s = check_params(c, *p);
    if (s) return s;
    c->gp = *p;
    c->has_params = true;
    c->has_kernels = false;
    return RK_OK;
}

rk_status rk_set_kernels(rk_ctx* c, const rk_kernel* k, uint32_t n) {
    if (!c || (!k && n)) return RK_EINVAL;
    if (!c->has_params) return fail(c, RK_ESTATE, "rk_set_gpu_params first");
    RkTables t;
    rk_status s = build_tables(c, c->gp, k, n, t);
    if (s) return s;
    if (c->device >= 0) {
        DeviceGuard dg(c->device);
        cudaError_t e = cudaMemcpy(c->tab_dev, &t, sizeof t, cudaMemcpyHostToDevice);
        if (e) return cuda_fail(c, e, "upload tables");
    }
    c->tab = t;
    c->ks.assign(k, k + n);
    c->has_kernels = true;
    if (c->device >= 0) {
        DeviceGuard dg(c->device);
        if ((s = dp_plan(c))) return s;
    }
    return RK_OK;
}

rk_status rk_eval_range_async(rk_ctx* c, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                              rk_stats* stats_dev, uint64_t* keys_dev, void* stream) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!stats_dev) return fail(c, RK_EINVAL, "stats_dev is required");
    if (first > space(c) || count > space(c) - first) return fail(c, RK_EINVAL, "range exceeds n!");
    DeviceGuard dg(c->device);
    c->launches = 0;
    if (c->dp.on) {
        const int e = dp_eval(c, first, count, cand_or_zero(c, cand_key_dev, stream), stats_dev, keys_dev, nullptr, 0,
                              nullptr, stream);
        return e ? cuda_fail(c, e, "memoised evaluation") : RK_OK;
    }
    int e = rk_launch_eval(c->tab_dev, c->tab.g.n, vS(c, c->tab.g.S), first, count, cand_key_dev, 0, stats_dev, keys_dev,
                           c->recs_dev, c->counter_dev, c->max_ctas, stream, &c->launches);
    return e ? cuda_fail(c, e, "rk_eval_kernel launch") : RK_OK;
}

rk_status rk_eval_range(rk_ctx* c, uint64_t first, uint64_t count, uint64_t candidate_key, rk_stats* out_host,
                        uint64_t* keys_dev, void* stream) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!out_host) return fail(c, RK_EINVAL, "out_host is required");
    if (first > space(c) || count > space(c) - first) return fail(c, RK_EINVAL, "range exceeds n!");
    DeviceGuard dg(c->device);
    c->launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (count == 0) {
        std::memset(out_host, 0, sizeof *out_host);
        return RK_OK;
    }
    int e;
    if (c->dp.on) {
        e = cudaMemcpyAsync(c->u64_dev + 8, &candidate_key, 8, cudaMemcpyHostToDevice, st);
        if (!e) e = dp_eval(c, first, count, c->u64_dev + 8, c->stats_dev, keys_dev, nullptr, 0, nullptr, stream);
    } else {
        e = rk_launch_eval(c->tab_dev, c->tab.g.n, vS(c, c->tab.g.S), first, count, nullptr, candidate_key,
                           c->stats_dev, keys_dev, c->recs_dev, c->counter_dev, c->max_ctas, stream, &c->launches);
    }
    if (e) return cuda_fail(c, e, "rk_eval_kernel launch");
    rk_stats h;
    e = cudaMemcpyAsync(&h, c->stats_dev, sizeof h, cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    if (e) return cuda_fail(c, e, "rk_eval_range");
    *out_host = h;
    return RK_OK;
}

rk_status rk_eval_index_async(rk_ctx* c, uint64_t index, uint64_t* key_dev, void* stream) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!key_dev) return fail(c, RK_EINVAL, "key_dev is required");
    if (index >= space(c)) return fail(c, RK_EINVAL, "index >= n!");
    DeviceGuard dg(c->device);
    c->launches = 0;
    int e = rk_launch_key_of_index(c->tab_dev, vS(c, c->tab.g.S), index, key_dev, stream, &c->launches);
    return e ? cuda_fail(c, e, "rk_eval_index_async") : RK_OK;
}

uint32_t rk_table_bytes(void) { return (uint32_t)sizeof(RkTables); }

rk_status rk_eval_range32_async(rk_ctx* c, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                                rk_stats* stats_dev, uint32_t* keys32_dev, uint64_t key_base, uint32_t* ovf_dev,
                                void* stream) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!stats_dev || !keys32_dev || !ovf_dev) return fail(c, RK_EINVAL, "stats_dev, keys32_dev, ovf_dev required");
    if (policy(c)) return fail(c, RK_EUNSUPPORTED, "compact keys under skip-ahead");
    if (first > space(c) || count > space(c) - first) return fail(c, RK_EINVAL, "range exceeds n!");
    DeviceGuard dg(c->device);
    c->launches = 0;
    int e = rk_launch_eval(c->tab_dev, c->tab.g.n, vS(c, c->tab.g.S), first, count, cand_key_dev, 0, stats_dev, nullptr,
                           c->recs_dev, c->counter_dev, c->max_ctas, stream, &c->launches, keys32_dev, key_base,
                           ovf_dev);
    return e ? cuda_fail(c, e, "rk_eval_kernel launch") : RK_OK;
}

rk_status rk_eval_range_hist_async(rk_ctx* c, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                                   rk_stats* stats_dev, const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev,
                                   void* stream) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!range_dev || !hist_dev || bins < 1 || bins > 32768) return fail(c, RK_EINVAL, "bad fused histogram args");
    if (policy(c)) return fail(c, RK_EUNSUPPORTED, "fused histogram under skip-ahead");
    if (first > space(c) || count > space(c) - first) return fail(c, RK_EINVAL, "range exceeds n!");
    DeviceGuard dg(c->device);
    c->launches = 0;
    rk_stats* out = stats_dev ? stats_dev : c->stats_dev;
    if (c->dp.on && bins <= rk_dp_max_fused_bins()) {
        const int e = dp_eval(c, first, count, cand_or_zero(c, cand_key_dev, stream), out, nullptr, range_dev, bins,
                              hist_dev, stream);
        return e ? cuda_fail(c, e, "memoised evaluation (fused histogram)") : RK_OK;
    }
    int e = rk_launch_eval(c->tab_dev, c->tab.g.n, vS(c, c->tab.g.S), first, count, cand_key_dev, 0, out, nullptr,
                           c->recs_dev, c->counter_dev, c->max_ctas, stream, &c->launches, nullptr, 0, nullptr,
                           range_dev, bins, hist_dev);
    return e ? cuda_fail(c, e, "rk_eval_kernel (fused histogram) launch") : RK_OK;
}

rk_status rk_sweep_pass1_async(rk_ctx* c, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                               rk_stats* rec_dev, uint64_t* keys_dev, void* stream) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!rec_dev || !cand_key_dev) return fail(c, RK_EINVAL, "rec_dev and cand_key_dev are required");
    if (first > space(c) || count > space(c) - first) return fail(c, RK_EINVAL, "range exceeds n!");
    DeviceGuard dg(c->device);
    c->launches = 0;
    int e;
    if (c->dp.on) {
        e = dp_pass1(c, first, count, rec_dev, stream);
    } else {
        const int m = tmark_begin(c, RK_PHASE_DIRECT, stream);
        e = rk_launch_eval(c->tab_dev, c->tab.g.n, vS(c, c->tab.g.S), first, count, cand_key_dev, 0, rec_dev, keys_dev,
                           c->recs_dev, c->counter_dev, c->max_ctas, stream, &c->launches);
        tmark_end(c, m, stream);
    }
    return e ? cuda_fail(c, e, "rk_sweep_pass1_async") : RK_OK;
}

rk_status rk_sweep_pass2_async(rk_ctx* c, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                               const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, uint64_t* keys_dev,
                               rk_stats* rec_dev, void* stream) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!rec_dev || !cand_key_dev) return fail(c, RK_EINVAL, "rec_dev and cand_key_dev are required");
    if (hist_dev && (!range_dev || bins < 1)) return fail(c, RK_EINVAL, "histogram needs range_dev and bins >= 1");
    if (first > space(c) || count > space(c) - first) return fail(c, RK_EINVAL, "range exceeds n!");
    DeviceGuard dg(c->device);
    c->launches = 0;
    int e = 0;
    if (c->dp.on) {
        const DpPlan& d = c->dp;
        if (!(d.runs_ok && d.runs_first == first && d.runs_count == count))
            return fail(c, RK_ESTATE, "pass 2 needs pass 1 over the same range first (it streams pass 1's run metadata)");
        const bool fused = hist_dev && bins <= rk_dp_max_fused_bins();
        if (hist_dev && !fused && !keys_dev) return fail(c, RK_EINVAL, "more than 32768 bins needs keys_dev");
        e = dp_pass2(c, first, count, cand_key_dev, range_dev, fused ? bins : 0, fused ? hist_dev : nullptr, keys_dev,
                     rec_dev, stream);
        if (!e && hist_dev && !fused)
            e = rk_launch_histogram(keys_dev, count, 0, 0, range_dev, bins, hist_dev, stream, &c->launches);
    } else if (hist_dev) {
        if (!keys_dev) return fail(c, RK_EINVAL, "keys_dev is required (direct evaluation)");
        const int m = tmark_begin(c, RK_PHASE_HIST, stream);
        e = rk_launch_histogram(keys_dev, count, 0, 0, range_dev, bins, hist_dev, stream, &c->launches);
        tmark_end(c, m, stream);
    }
    return e ? cuda_fail(c, e, "rk_sweep_pass2_async") : RK_OK;
}

rk_status rk_sweep_pass2_32_async(rk_ctx* c, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                                  const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, uint32_t* keys32_dev,
                                  uint64_t key_base, uint32_t* ovf_dev, rk_stats* rec_dev, void* stream) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!rec_dev || !cand_key_dev || !keys32_dev || !ovf_dev || !range_dev)
        return fail(c, RK_EINVAL, "rec_dev, cand_key_dev, range_dev, keys32_dev and ovf_dev are required");
    if (hist_dev && (!range_dev || bins < 1 || bins > rk_dp_max_fused_bins()))
        return fail(c, RK_EINVAL, "histogram needs range_dev and 1 <= bins <= 32768");
    if (first > space(c) || count > space(c) - first) return fail(c, RK_EINVAL, "range exceeds n!");
    if (!c->dp.on) return fail(c, RK_EUNSUPPORTED, "compact pass 2 needs memoisation (use rk_eval_range32_async)");
    DeviceGuard dg(c->device);
    c->launches = 0;
    const DpPlan& d = c->dp;
    if (!(d.runs_ok && d.runs_first == first && d.runs_count == count))
        return fail(c, RK_ESTATE, "pass 2 needs pass 1 over the same range first (it streams pass 1's run metadata)");
    const int e = dp_pass2(c, first, count, cand_key_dev, range_dev, hist_dev ? bins : 0, hist_dev, nullptr, rec_dev,
                           stream, keys32_dev, key_base, ovf_dev);
    return e ? cuda_fail(c, e, "rk_sweep_pass2_32_async") : RK_OK;
}

rk_status rk_set_timing(rk_ctx* c, int on) {
    rk_status s = need_device(c);
    if (s) return s;
    c->timing = on != 0;
    c->tused = 0;
    return RK_OK;
}

rk_status rk_timing_read(rk_ctx* c, double* ms_sum, uint32_t* counts, uint32_t n_phases) {
    rk_status s = need_device(c);
    if (s) return s;
    if (!ms_sum || !counts) return fail(c, RK_EINVAL, "ms_sum and counts are required");
    DeviceGuard dg(c->device);
    for (uint32_t p = 0; p < n_phases; p++) {
        ms_sum[p] = 0.0;
        counts[p] = 0;
    }
    for (size_t m = 0; m < c->tused; m++) {
        const uint32_t p = c->tphase[m];
        if (p >= n_phases) continue;
        cudaError_t e = cudaEventSynchronize(c->tev[2 * m + 1]);
        float ms = 0.f;
        if (!e) e = cudaEventElapsedTime(&ms, c->tev[2 * m], c->tev[2 * m + 1]);
        if (e) return cuda_fail(c, e, "rk_timing_read");
        ms_sum[p] += ms;
        counts[p]++;
    }
    c->tused = 0;
    return RK_OK;
}

rk_status rk_memo_info(rk_ctx* c, uint32_t* on_out, uint32_t* levels_out, uint32_t* nodes_out, uint32_t max_levels) {
    if (!c || !on_out) return RK_EINVAL;
    *on_out = c->dp.on ? 1u : 0u;
    if (levels_out) *levels_out = c->dp.on ? c->dp.P : 0u;
    if (nodes_out && c->dp.on)
        for (uint32_t j = 0; j <= c->dp.P && j < max_levels; j++) nodes_out[j] = c->dp.cnt[j];
    return RK_OK;
}

rk_status rk_memo_audit(rk_ctx* c, uint64_t* out) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!out) return fail(c, RK_EINVAL, "out is required");
    DpPlan& d = c->dp;
    if (!d.on || !d.runs_ok) return fail(c, RK_ESTATE, "memo audit needs memoisation on and a pass 1 first");
    DeviceGuard dg(c->device);
    unsigned long long* bad = nullptr;
    std::vector<unsigned long long> h(6 * d.L, 0);
    std::vector<uint32_t> cnt(d.L + 1, 0);
    int e = cudaMalloc(&bad, sizeof(unsigned long long) * 6 * d.L);
    if (!e) e = cudaMemset(bad, 0, sizeof(unsigned long long) * 6 * d.L);
    const char* nodes = (const char*)d.nodes.p;
    const bool ub = d.last_ub; /* the tables of the last pass 1: the plan's build, or the step's rebuild */
    const std::vector<size_t>& noff = ub ? d.ub_noff : d.noff;
    const std::vector<size_t>& toff = ub ? d.ub_toff : d.toff;
    const std::vector<uint32_t>& cap = ub ? d.ub_cap : d.cap;
    const std::vector<uint32_t>& tmask = ub ? d.ub_tmask : d.tmask;
    for (uint32_t j = 1; j <= d.L && !e; j++)
        e = rk_dp_audit(c->tab.g.S, nodes + noff[j], (const uint32_t*)d.counters.p + j, cap[j],
                        (const uint32_t*)d.tables.p + toff[j], tmask[j], d.view.tid[j - 1],
                        (uint64_t)d.cnt[j - 1] * c->tab.g.n, j > 1 ? nodes + noff[j - 1] : nullptr, c->tab.g.n,
                        bad + 6 * (j - 1), nullptr);
    if (!e) e = cudaMemcpy(h.data(), bad, sizeof(unsigned long long) * 6 * d.L, cudaMemcpyDeviceToHost);
    if (!e) e = cudaMemcpy(cnt.data(), d.counters.p, 4 * (d.L + 1), cudaMemcpyDeviceToHost);
    cudaFree(bad);
    if (e) return cuda_fail(c, e, "rk_memo_audit");
    for (int q = 0; q < 8; q++) out[q] = 0;
    for (uint32_t j = 1; j <= d.L; j++) {
        for (int q = 0; q < 5; q++) out[q] += h[6 * (j - 1) + q];
        out[5] += h[6 * (j - 1) + 5] != cnt[j];   /* published slots != count */
        out[6] += cnt[j] != d.cnt[j];             /* count != the plan's (deterministic) count */
        out[7] += cnt[j];
    }
    return RK_OK;
}

rk_status rk_key_lower_bound(rk_ctx* c, uint64_t* lb_out) {
    if (!c || !lb_out) return RK_EINVAL;
    rk_status s = need_kernels(c);
    if (s) return s;
    u128 sI = 0, sM = 0;
    for (const rk_kernel& k : c->ks) {
        sI += (u128)k.grid_blocks * k.inst_per_block;
        sM += (u128)k.grid_blocks * k.mem_per_block;
    }
    const u128 a = sI * c->gp.rb_den, b = sM * c->gp.rb_num;
    *lb_out = (uint64_t)(a >= b ? a : b); /* < 2^63 by the key bound */
    return RK_OK;
}

rk_status rk_histogram32_async(rk_ctx* c, const uint32_t* keys32_dev, uint64_t count, uint64_t key_base,
                               const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, void* stream) {
    rk_status s = need_device(c);
    if (s) return s;
    if (bins < 1 || bins > 65536 || !hist_dev || !range_dev || (count && !keys32_dev))
        return fail(c, RK_EINVAL, "bad histogram args");
    DeviceGuard dg(c->device);
    c->launches = 0;
    if (count == 0) return RK_OK;
    int e = rk_launch_histogram32(keys32_dev, count, key_base, range_dev, bins, hist_dev, stream, &c->launches);
    return e ? cuda_fail(c, e, "histogram32 launch") : RK_OK;
}

rk_status rk_merge_stats_async(rk_ctx* c, const rk_stats* in_dev, uint32_t n_records, rk_stats* out_dev,
                               void* stream) {
    rk_status s = need_device(c);
    if (s) return s;
    if (!in_dev || !out_dev || n_records == 0) return fail(c, RK_EINVAL, "bad merge arguments");
    DeviceGuard dg(c->device);
    c->launches = 0;
    int e = rk_launch_merge(in_dev, n_records, out_dev, stream, &c->launches);
    return e ? cuda_fail(c, e, "merge launch") : RK_OK;
}

static rk_status hist_common(rk_ctx* c, const uint64_t* keys_dev, uint64_t count, uint64_t kmin, uint64_t kmax,
                             const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, void* stream) {
    rk_status s = need_device(c);
    if (s) return s;
    if (bins < 1 || bins > 65536 || !hist_dev || (count && !keys_dev)) return fail(c, RK_EINVAL, "bad histogram args");
    if (!range_dev && kmax < kmin) return fail(c, RK_EINVAL, "kmax < kmin");
    DeviceGuard dg(c->device);
    c->launches = 0;
    if (count == 0) return RK_OK;
    int e = rk_launch_histogram(keys_dev, count, kmin, kmax, range_dev, bins, hist_dev, stream, &c->launches);
    return e ? cuda_fail(c, e, "histogram launch") : RK_OK;
}

rk_status rk_histogram(rk_ctx* c, const uint64_t* keys_dev, uint64_t count, uint64_t kmin, uint64_t kmax,
                       uint32_t bins, uint64_t* hist_dev, void* stream) {
    return hist_common(c, keys_dev, count, kmin, kmax, nullptr, bins, hist_dev, stream);
}

rk_status rk_histogram_async(rk_ctx* c, const uint64_t* keys_dev, uint64_t count, const rk_stats* range_dev,
                             uint32_t bins, uint64_t* hist_dev, void* stream) {
    if (!range_dev) return fail(c, RK_EINVAL, "range_dev is required");
    return hist_common(c, keys_dev, count, 0, 0, range_dev, bins, hist_dev, stream);
}

rk_status rk_range_histogram(rk_ctx* c, const uint64_t* keys_dev, uint64_t count, uint64_t lo, uint64_t span,
                             uint32_t bins, uint64_t* hist_dev, void* stream) {
    rk_status s = need_device(c);
    if (s) return s;
    if (span == 0 || bins < 1 || bins > 65536 || !hist_dev || (count && !keys_dev))
        return fail(c, RK_EINVAL, "bad range histogram args");
    DeviceGuard dg(c->device);
    c->launches = 0;
    if (count == 0) return RK_OK;
    int e = rk_launch_range_histogram(keys_dev, count, lo, span, bins, hist_dev, stream, &c->launches);
    return e ? cuda_fail(c, e, "range histogram launch") : RK_OK;
}

static rk_status select_common(rk_ctx* c, const void* keys_dev, bool k32, uint64_t key_base, uint64_t count,
                               uint64_t kmin, uint64_t kmax, const uint64_t* ranks, uint32_t m, uint64_t* keys_out,
                               void* stream) {
    rk_status s = need_device(c);
    if (s) return s;
    if (!keys_dev || !ranks || !keys_out || kmax < kmin) return fail(c, RK_EINVAL, "bad select args");
    for (uint32_t j = 0; j < m; j++)
        if (ranks[j] >= count) return fail(c, RK_EINVAL, "rank %llu >= count", (unsigned long long)ranks[j]);
    DeviceGuard dg(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (kmax - kmin == ~0ull) return fail(c, RK_EINVAL, "key range must be < 2^64 - 1");
    constexpr uint32_t B = 16384;
    uint64_t* hd = nullptr;
    int e = cudaMalloc(&hd, sizeof(uint64_t) * B);
    std::vector<uint64_t> h(B);
    uint32_t launches = 0;
    std::vector<uint64_t> out(m);
    for (uint32_t j = 0; j < m && !e; j++) {
        uint64_t lo = kmin, span = kmax - kmin + 1, r = ranks[j];
        for (;;) {
            const uint32_t bins = span <= B ? (uint32_t)span : B;
            e = cudaMemsetAsync(hd, 0, sizeof(uint64_t) * bins, st);
            if (!e)
                e = k32 ? rk_launch_range_histogram32((const uint32_t*)keys_dev, count, key_base, lo, span, bins, hd,
                                                      stream, &launches)
                        : rk_launch_range_histogram((const uint64_t*)keys_dev, count, lo, span, bins, hd, stream,
                                                    &launches);
            if (!e) e = cudaMemcpyAsync(h.data(), hd, sizeof(uint64_t) * bins, cudaMemcpyDeviceToHost, st);
            if (!e) e = cudaStreamSynchronize(st);
            if (e) break;
            uint64_t cum = 0;
            uint32_t b = 0;
            for (; b < bins; b++) {
                if (r < cum + h[b]) break;
                cum += h[b];
            }
            if (b == bins) { /* keys outside [kmin, kmax]: caller error */
                e = -1;
                break;
            }
            r -= cum;
            if (bins == span) { /* unit bins: exact */
                out[j] = lo + b;
                break;
            }
            /* bin b = keys with x in [ceil(b*span/bins), ceil((b+1)*span/bins)) */
            const u128 a0 = ((u128)b * span + bins - 1) / bins, a1 = ((u128)(b + 1) * span + bins - 1) / bins;
            lo += (uint64_t)a0;
            span = (uint64_t)(a1 - a0);
        }
    }
    cudaFree(hd);
    c->launches = launches;
    if (e == -1) return fail(c, RK_EINVAL, "keys outside [kmin, kmax]");
    if (e) return cuda_fail(c, e, "rk_select_keys");
    std::memcpy(keys_out, out.data(), sizeof(uint64_t) * m);
    return RK_OK;
}

rk_status rk_select_keys(rk_ctx* c, const uint64_t* keys_dev, uint64_t count, uint64_t kmin, uint64_t kmax,
                         const uint64_t* ranks, uint32_t m, uint64_t* keys_out, void* stream) {
    return select_common(c, keys_dev, false, 0, count, kmin, kmax, ranks, m, keys_out, stream);
}

rk_status rk_select_keys32(rk_ctx* c, const uint32_t* keys32_dev, uint64_t key_base, uint64_t count, uint64_t kmin,
                           uint64_t kmax, const uint64_t* ranks, uint32_t m, uint64_t* keys_out, void* stream) {
    return select_common(c, keys32_dev, true, key_base, count, kmin, kmax, ranks, m, keys_out, stream);
}

rk_status rk_range_histogram32(rk_ctx* c, const uint32_t* keys32_dev, uint64_t key_base, uint64_t count, uint64_t lo,
                               uint64_t span, uint32_t bins, uint64_t* hist_dev, void* stream) {
    rk_status s = need_device(c);
    if (s) return s;
    if (span == 0 || bins < 1 || bins > 65536 || !hist_dev || (count && !keys32_dev))
        return fail(c, RK_EINVAL, "bad range histogram args");
    DeviceGuard dg(c->device);
    c->launches = 0;
    if (count == 0) return RK_OK;
    int e = rk_launch_range_histogram32(keys32_dev, count, key_base, lo, span, bins, hist_dev, stream, &c->launches);
    return e ? cuda_fail(c, e, "range histogram32 launch") : RK_OK;
}

/* key of one index on the device (synchronous) */
static rk_status key_of_index(rk_ctx* c, uint64_t idx, uint64_t* key, void* stream) {
    DeviceGuard dg(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    int e = cudaMemcpyAsync(c->u64_dev, &idx, sizeof idx, cudaMemcpyHostToDevice, st);
    if (!e) e = rk_launch_keys_of_same(c->tab_dev, vS(c, c->tab.g.S), c->u64_dev, 1, c->u64_dev + 1, stream, &c->launches);
    uint64_t h = 0;
    if (!e) e = cudaMemcpyAsync(&h, c->u64_dev + 1, sizeof h, cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    if (e) return cuda_fail(c, e, "key_of_index");
    *key = h;
    return RK_OK;
}

rk_status rk_heuristic_order(rk_ctx* c, int32_t* order_out, int32_t* round_of_out, uint64_t* index_out,
                             uint64_t* key_out) {
    if (!c || !order_out) return RK_EINVAL;
    rk_status s = need_kernels(c);
    if (s) return s;
    if (key_out && (s = need_device(c))) return s;
    const uint32_t n = (uint32_t)c->ks.size();
    std::vector<int32_t> order(n), rounds(n);
    Alg1(c->gp).run(c->ks.data(), n, order.data(), rounds.data());
    uint64_t idx = 0;
    do_rank(order.data(), n, &idx);
    c->launches = 0;
    if (key_out) {
        uint64_t k = 0;
        if ((s = key_of_index(c, idx, &k, nullptr))) return s;
        *key_out = k;
    }
    std::memcpy(order_out, order.data(), n * sizeof(int32_t));
    if (round_of_out) std::memcpy(round_of_out, rounds.data(), n * sizeof(int32_t));
    if (index_out) *index_out = idx;
    return RK_OK;
}

/* Validate and pack the tables of n_sets sets (rk_set_kernels' checks) on up to
 * 16 host threads; the lowest failing set's error is reported. */
static rk_status build_tables_batch(rk_ctx* c, const rk_kernel* sets, uint32_t n, uint32_t n_sets, RkTables* tabs) {
    const uint32_t hw = std::max(1u, std::thread::hardware_concurrency());
    const uint32_t nt = std::max(1u, std::min({16u, hw, n_sets / 256u}));
    std::vector<rk_status> st(nt, RK_OK);
    std::vector<uint32_t> bad(nt, 0xFFFFFFFFu);
    std::vector<std::string> msg(nt);
    auto work = [&](uint32_t w) {
        rk_ctx local; /* fail() writes the message here */
        local.no_reduce = c->no_reduce;
        RkTables tmp;
        const uint32_t a = (uint32_t)((uint64_t)n_sets * w / nt), b = (uint32_t)((uint64_t)n_sets * (w + 1) / nt);
        for (uint32_t q = a; q < b; q++) {
            const rk_status s = build_tables(&local, c->gp, sets + (size_t)q * n, n, tabs ? tabs[q] : tmp);
            if (s) {
                st[w] = s;
                bad[w] = q;
                msg[w] = local.err;
                return;
            }
        }
    };
    if (nt == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (uint32_t w = 0; w < nt; w++) th.emplace_back(work, w);
        for (auto& t : th) t.join();
    }
    for (uint32_t w = 0; w < nt; w++)
        if (st[w]) {
            c->err = "set " + std::to_string(bad[w]) + ": " + msg[w];
            return st[w];
        }
    return RK_OK;
}

/* Algorithm 1 on device for sets already validated */
static rk_status heuristic_batch_dev(rk_ctx* c, const rk_kernel* sets, uint32_t n, uint32_t n_sets,
                                     int32_t* orders_out, uint64_t* index_out, void* stream) {
    DeviceGuard dg(c->device);
    c->launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    rk_kernel* sets_dev = nullptr;
    int32_t* ord_dev = nullptr;
    uint64_t* idx_dev = nullptr;
    int e = cudaMallocAsync((void**)&sets_dev, sizeof(rk_kernel) * (size_t)n * n_sets, st);
    if (!e) e = cudaMallocAsync((void**)&ord_dev, sizeof(int32_t) * (size_t)n * n_sets, st);
    if (!e) e = cudaMallocAsync((void**)&idx_dev, sizeof(uint64_t) * n_sets, st);
    if (!e) e = cudaMemcpyAsync(sets_dev, sets, sizeof(rk_kernel) * (size_t)n * n_sets, cudaMemcpyHostToDevice, st);
    if (!e) e = rk_launch_heuristic(sets_dev, n, n_sets, &c->gp, ord_dev, idx_dev, stream, &c->launches);
    if (!e) e = cudaMemcpyAsync(index_out, idx_dev, sizeof(uint64_t) * n_sets, cudaMemcpyDeviceToHost, st);
    if (!e && orders_out)
        e = cudaMemcpyAsync(orders_out, ord_dev, sizeof(int32_t) * (size_t)n * n_sets, cudaMemcpyDeviceToHost, st);
    if (sets_dev) cudaFreeAsync(sets_dev, st);
    if (ord_dev) cudaFreeAsync(ord_dev, st);
    if (idx_dev) cudaFreeAsync(idx_dev, st);
    if (!e) e = cudaStreamSynchronize(st);
    return e ? cuda_fail(c, e, "rk_heuristic_batch") : RK_OK;
}

rk_status rk_heuristic_batch(rk_ctx* c, const rk_kernel* sets, uint32_t n, uint32_t n_sets, int32_t* orders_out,
                             uint64_t* index_out, void* stream) {
    rk_status s = need_device(c);
    if (s) return s;
    if (!c->has_params) return fail(c, RK_ESTATE, "rk_set_gpu_params first");
    if (!sets || !index_out || n_sets == 0) return fail(c, RK_EINVAL, "bad heuristic batch arguments");
    if (n == 0 || n > RK_MAX_N) return fail(c, n ? RK_ETOOMANY : RK_EINVAL, "n out of range");
    if ((s = build_tables_batch(c, sets, n, n_sets, nullptr))) return s; /* same validation as rk_set_kernels */
    return heuristic_batch_dev(c, sets, n, n_sets, orders_out, index_out, stream);
}

rk_status rk_percentile(rk_ctx* c, const int32_t* order, uint64_t first, uint64_t count, uint64_t* n_ge_out,
                        uint64_t* key_out) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    if (!order || !n_ge_out) return fail(c, RK_EINVAL, "null argument");
    uint64_t idx;
    if (do_rank(order, (uint32_t)c->ks.size(), &idx)) return fail(c, RK_EINVAL, "order is not a permutation");
    uint64_t key;
    if ((s = key_of_index(c, idx, &key, nullptr))) return s;
    uint32_t l0 = c->launches;
    rk_stats st;
    if ((s = rk_eval_range(c, first, count, key, &st, nullptr, nullptr))) return s;
    c->launches += l0;
    *n_ge_out = st.n_eq + st.n_gt;
    if (key_out) *key_out = key;
    return RK_OK;
}

rk_status rk_eval_batch(rk_ctx* c, const rk_kernel* sets, uint32_t n, uint32_t n_sets, const uint64_t* cand_index,
                        rk_stats* out_host, uint64_t* cand_key_out, void* stream) {
    rk_status s = need_device(c);
    if (s) return s;
    if (!c->has_params) return fail(c, RK_ESTATE, "rk_set_gpu_params first");
    if (!sets || !out_host || n_sets == 0) return fail(c, RK_EINVAL, "bad batch arguments");
    if (n == 0 || n > RK_MAX_N) return fail(c, n ? RK_ETOOMANY : RK_EINVAL, "n out of range");
    /* RK_BATCH_TRACE=1: host-side phase times of this call on stderr (profiling aid) */
    static const bool trace = [] { const char* v = getenv("RK_BATCH_TRACE"); return v && v[0] == '1'; }();
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t0 = now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        const auto t1 = now();
        fprintf(stderr, "rk_eval_batch %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    };
    std::unique_ptr<RkTables[]> tabs(new RkTables[n_sets]); /* every entry written by build_tables */
    std::vector<uint64_t> idx(n_sets);
    if ((s = build_tables_batch(c, sets, n, n_sets, tabs.get()))) return s;
    mark("tables");
    if (cand_index)
        for (uint32_t q = 0; q < n_sets; q++) {
            if (cand_index[q] >= fact64(n)) return fail(c, RK_EINVAL, "set %u: candidate index >= n!", q);
            idx[q] = cand_index[q];
        }
    if (!cand_index && (s = heuristic_batch_dev(c, sets, n, n_sets, nullptr, idx.data(), stream))) return s;
    mark("heuristic");
    /* group the sets by reduced SM count so every launch runs a compile-time variant */
    std::vector<uint32_t> perm(n_sets), Sv(n_sets);
    for (uint32_t q = 0; q < n_sets; q++) {
        perm[q] = q;
        Sv[q] = tabs[q].g.S;
    }
    std::stable_sort(perm.begin(), perm.end(), [&](uint32_t a, uint32_t b) { return Sv[a] < Sv[b]; });
    /* the sorted tables and candidate indices go up from a pinned staging buffer kept by the ctx
     * (grow-only; every call ends with a stream synchronize, so no copy is in flight on reuse) */
    const size_t pin_need = (sizeof(RkTables) + sizeof(uint64_t)) * (size_t)n_sets;
    if (pin_need > c->pin_bytes) {
        if (c->pin) cudaFreeHost(c->pin);
        c->pin = nullptr;
        c->pin_bytes = 0;
        if (cudaMallocHost(&c->pin, pin_need) != cudaSuccess) return fail(c, RK_ECUDA, "pinned staging");
        c->pin_bytes = pin_need;
    }
    RkTables* ptabs = reinterpret_cast<RkTables*>(c->pin);
    uint64_t* pidx = reinterpret_cast<uint64_t*>(ptabs + n_sets);
    for (uint32_t q = 0; q < n_sets; q++) {
        std::memcpy(&ptabs[q], &tabs[perm[q]], sizeof(RkTables));
        pidx[q] = idx[perm[q]];
    }
    mark("sort");
    DeviceGuard dg(c->device);
    c->launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t max_chunks = 0;
    for (uint32_t q = 0; q < n_sets; q++)
        max_chunks = std::max(max_chunks, (uint32_t)rk_batch_chunks_per_set(n, vS(c, ptabs[q].g.S)));
    RkTables* tabs_dev = nullptr;
    uint64_t *idx_dev = nullptr, *keys_dev = nullptr;
    rk_stats *recs = nullptr, *out_dev = nullptr;
    int e = cudaMallocAsync((void**)&tabs_dev, sizeof(RkTables) * n_sets, st);
    if (!e) e = cudaMallocAsync((void**)&idx_dev, sizeof(uint64_t) * n_sets, st);
    if (!e) e = cudaMallocAsync((void**)&keys_dev, sizeof(uint64_t) * n_sets, st);
    if (!e) e = cudaMallocAsync((void**)&recs, sizeof(rk_stats) * (size_t)n_sets * max_chunks, st);
    if (!e) e = cudaMallocAsync((void**)&out_dev, sizeof(rk_stats) * n_sets, st);
    if (!e) e = cudaMemcpyAsync(tabs_dev, ptabs, sizeof(RkTables) * n_sets, cudaMemcpyHostToDevice, st);
    if (!e) e = cudaMemcpyAsync(idx_dev, pidx, sizeof(uint64_t) * n_sets, cudaMemcpyHostToDevice, st);
    uint32_t smax_k = 0;
    for (uint32_t q = 0; q < n_sets; q++) smax_k = std::max(smax_k, vS(c, ptabs[q].g.S));
    if (!e) e = rk_launch_keys_of(tabs_dev, n, smax_k, idx_dev, n_sets, keys_dev, stream, &c->launches);
    mark("upload");
    /* groups on S' <= 2 run the memoised batch kernel (RK_NO_MEMO=1: the direct one) */
    auto memo_group = [&](uint32_t S) { return !c->no_memo && !(S & RK_S_POLICY) && rk_batch_memo_ok(n, S); };
    size_t memo_bytes = 0;
    for (uint32_t a = 0; a < n_sets;) {
        uint32_t b = a;
        while (b < n_sets && ptabs[b].g.S == ptabs[a].g.S) b++;
        const uint32_t S = vS(c, ptabs[a].g.S);
        if (memo_group(S))
            memo_bytes = std::max(memo_bytes, rk_batch_memo_scratch(n, S, rk_batch_memo_grid(S, b - a)));
        a = b;
    }
    if (!e && memo_bytes > c->batch_scratch_bytes) { /* grow-only, kept by the context */
        cudaFree(c->batch_scratch);
        c->batch_scratch = nullptr;
        c->batch_scratch_bytes = 0;
        e = cudaMalloc(&c->batch_scratch, memo_bytes);
        if (!e) c->batch_scratch_bytes = memo_bytes;
    }
    for (uint32_t a = 0; a < n_sets && !e;) {
        uint32_t b = a;
        while (b < n_sets && ptabs[b].g.S == ptabs[a].g.S) b++;
        const uint32_t S = vS(c, ptabs[a].g.S), chunks = (uint32_t)rk_batch_chunks_per_set(n, S);
        if (memo_group(S))
            e = rk_launch_batch_memo(tabs_dev + a, n, S, b - a, keys_dev + a, out_dev + a, c->batch_scratch,
                                     (uint32_t)rk_batch_memo_grid(S, b - a), stream, &c->launches);
        else
            e = rk_launch_batch(tabs_dev + a, n, S | 0x80000000u, b - a, keys_dev + a, out_dev + a, recs, chunks,
                                stream, &c->launches);
        a = b;
    }
    mark("launch");
    std::vector<uint64_t> keys(n_sets);
    std::vector<rk_stats> pout(n_sets);
    if (!e) e = cudaMemcpyAsync(pout.data(), out_dev, sizeof(rk_stats) * n_sets, cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaMemcpyAsync(keys.data(), keys_dev, sizeof(uint64_t) * n_sets, cudaMemcpyDeviceToHost, st);
    for (void* p : {(void*)tabs_dev, (void*)idx_dev, (void*)keys_dev, (void*)recs, (void*)out_dev})
        if (p) cudaFreeAsync(p, st);
    if (!e) e = cudaStreamSynchronize(st);
    mark("device+d2h");
    if (e) return cuda_fail(c, e, "rk_eval_batch");
    for (uint32_t q = 0; q < n_sets; q++) {
        out_host[perm[q]] = pout[q];
        if (cand_key_out) cand_key_out[perm[q]] = keys[q];
    }
    return RK_OK;
}

rk_status rk_simulate_order(rk_ctx* c, const int32_t* order, uint32_t* rounds_out, uint32_t max_rounds,
                            uint32_t* n_rounds_out, uint64_t* key_out) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    const uint32_t n = (uint32_t)c->ks.size();
    uint64_t idx;
    if (!order || do_rank(order, n, &idx)) return fail(c, RK_EINVAL, "order is not a permutation");
    if (max_rounds == 0 || !rounds_out) return fail(c, RK_EINVAL, "rounds_out / max_rounds");
    DeviceGuard dg(c->device);
    c->launches = 0;
    int32_t* order_dev = nullptr;
    uint32_t* rounds_dev = nullptr;
    uint32_t* nr_dev = nullptr;
    uint64_t* key_dev = nullptr;
    int e = cudaMalloc(&order_dev, n * sizeof(int32_t));
    if (!e) e = cudaMalloc(&rounds_dev, (size_t)max_rounds * n * sizeof(uint32_t));
    if (!e) e = cudaMalloc(&nr_dev, sizeof(uint32_t));
    if (!e) e = cudaMalloc(&key_dev, sizeof(uint64_t));
    if (!e) e = cudaMemcpy(order_dev, order, n * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (!e) e = rk_launch_simulate(c->tab_dev, n, vS(c, c->tab.g.S), order_dev, rounds_dev, max_rounds, nr_dev, key_dev,
                                   nullptr, &c->launches);
    uint32_t nr = 0;
    uint64_t key = 0;
    std::vector<uint32_t> rounds((size_t)max_rounds * n);
    if (!e) e = cudaMemcpy(rounds.data(), rounds_dev, rounds.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost);
    if (!e) e = cudaMemcpy(&nr, nr_dev, sizeof nr, cudaMemcpyDeviceToHost);
    if (!e) e = cudaMemcpy(&key, key_dev, sizeof key, cudaMemcpyDeviceToHost);
    cudaFree(order_dev);
    cudaFree(rounds_dev);
    cudaFree(nr_dev);
    cudaFree(key_dev);
    if (e) return cuda_fail(c, e, "rk_simulate_order");
    std::memcpy(rounds_out, rounds.data(), rounds.size() * sizeof(uint32_t));
    if (n_rounds_out) *n_rounds_out = nr;
    if (key_out) *key_out = key;
    if (nr > max_rounds) return fail(c, RK_EINVAL, "order has %u rounds > max_rounds %u", nr, max_rounds);
    return RK_OK;
}

rk_status rk_best_order(rk_ctx* c, uint64_t seed_index, int32_t* order_out, uint64_t* index_out, uint64_t* key_out,
                        uint64_t* nodes_out, void* stream) {
    rk_status s = need_device(c);
    if (s || (s = need_kernels(c))) return s;
    const uint32_t n = c->tab.g.n;
    if (seed_index != UINT64_MAX && seed_index >= space(c)) return fail(c, RK_EINVAL, "seed_index >= n!");
    if (policy(c)) return fail(c, RK_EUNSUPPORTED, "branch and bound under skip-ahead");
    DeviceGuard dg(c->device);
    c->launches = 0;
    uint64_t seed = ~0ull;
    if (seed_index != UINT64_MAX && (s = key_of_index(c, seed_index, &seed, stream))) return s;
    /* prefix depth P: enough units for dynamic balance (8 per thread), P <= n-1 */
    const uint64_t threads = (uint64_t)rk_bnb_ctas() * 128;
    uint32_t P = 0;
    uint64_t units = 1;
    while (P + 1 < n && units < 8 * threads) units *= (n - P++);
    const int ctas = rk_bnb_ctas();
    struct {
        unsigned long long best, nodes;
        unsigned int next_unit, done;
        unsigned long long key, index;
    } h{seed, 0, 0, 0, 0, 0};
    static_assert(sizeof h == 40, "BnbGlobal layout");
    void* gb = nullptr;
    unsigned long long* recs = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    int e = cudaMalloc(&gb, sizeof h);
    if (!e) e = cudaMalloc(&recs, sizeof(unsigned long long) * 2 * ctas);
    if (!e) e = cudaMemcpyAsync(gb, &h, sizeof h, cudaMemcpyHostToDevice, st);
    if (!e) e = rk_launch_bnb(c->tab_dev, vS(c, c->tab.g.S), P, units, gb, recs, stream, &c->launches);
    if (!e) e = cudaMemcpyAsync(&h, gb, sizeof h, cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    cudaFree(gb);
    cudaFree(recs);
    if (e) return cuda_fail(c, e, "rk_best_order");
    if (h.index >= space(c)) return fail(c, RK_EINVAL, "rk_best_order: no order found (internal)");
    if (order_out) do_unrank(h.index, n, order_out);
    if (index_out) *index_out = h.index;
    if (key_out) *key_out = h.key;
    if (nodes_out) *nodes_out = h.nodes;
    return RK_OK;
}

rk_status rk_rank(const int32_t* order, uint32_t n, uint64_t* idx_out) {
    if (!order || !idx_out) return RK_EINVAL;
    return do_rank(order, n, idx_out);
}

rk_status rk_unrank(uint64_t idx, uint32_t n, int32_t* order_out) {
    if (!order_out) return RK_EINVAL;
    return do_unrank(idx, n, order_out);
}

} /* extern "C" */
