/*
 * rk_kernels.cu — sm_100a kernels of the exhaustive launch-order evaluation
 * (arXiv 1511.07983).  Product path; shares nothing with oracle/.
 *
 * One thread evaluates a "run": the 3! = 6 consecutive lexicographic indices
 * that share an (n-3)-prefix (prefix sharing).  It unranks the
 * prefix (Lehmer code, PAPER:254 / SPEC:292), places the prefix kernels once,
 * places each of the 3 level-(n-2) kernels, and for each of the 6 leaves places
 * the level-(n-1) kernel fused with the evaluation of the last kernel (the
 * leaf's SM state is never materialised).
 *
 * Placement of one kernel is the closed-form "water-fill" equivalent of the
 * paper's block-by-block round-robin dispatch:
 * per SM the capacity c_s = min over the four limits of
 * floor(free/demand); blocks go round-robin over the SMs with remaining
 * capacity starting at the cursor, so after t passes SM s holds min(c_s, t);
 * the pass holding the last block comes from a binary search on t (16x2 SIMD
 * mins over SM pairs), the last block's SM from a select on the ring-rotated
 * eligibility mask.  A block that fits nowhere closes the execution round
 * (PAPER:79-81); rounds are scored exactly as K += max(den*I_r, num*M_r)
 * (reading L1).
 *
 * SM state lives in registers (2 packed u32 per SM, fully unrolled over
 * SMAX; FULL = compile-time S == SMAX), kernel tables in shared memory,
 * reductions via warp shuffles then shared memory then a last-CTA merge.
 */
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rk_internal.h"

namespace cg = cooperative_groups;
namespace {

#ifndef RK_EVAL_THREADS
#define RK_EVAL_THREADS 256
#endif
constexpr int kThreads = RK_EVAL_THREADS;
/* branch-free overflow handling up to this many (super-)SMs (measured) */
#ifndef RK_BF_MAX
#define RK_BF_MAX 32
#endif

/* Round key max(den*I_r, num*M_r) = den * max(I_r, R_B*M_r): the
 * state accumulates the scaled sums den*I_r and num*M_r directly (per-kernel
 * den*A_i and num*M_i precomputed), so closing a round is one 64-bit max. */
__device__ __forceinline__ uint64_t round_key(uint64_t dI, uint64_t nM, uint32_t, uint32_t) {
    return dI >= nM ? dI : nM;
}

constexpr uint32_t kSmemBins = 32768; /* 128 KB of u32 bins per CTA */

struct BinCalc {
    uint64_t kmin, D, inv;
    uint32_t bins, m32, kmin32, D32;
    bool fast;   /* D*bins < 2^63: 64-bit products suffice */
    bool fast32; /* bins < D < 2^32: 32-bit offset, 32-bit magic, one exact correction */
    /* Fig. 1 bins over [kmin, kmax] (last bin closed) */
    __device__ __forceinline__ void init(uint64_t lo, uint64_t hi, uint32_t nb) { init_span(lo, hi - lo, nb); }
    /* floor((K - lo) * nb / span) */
    __device__ __forceinline__ void init_span(uint64_t lo, uint64_t span, uint32_t nb) {
        kmin = lo;
        D = span;
        bins = nb;
        fast = D != 0 && D < (1ull << 63) / nb;
        inv = D ? (~0ull) / D : 0;
        fast32 = D > nb && D < (1ull << 32); /* m32 < 2^32 needs D > bins */
        kmin32 = (uint32_t)kmin;
        D32 = (uint32_t)D;
        m32 = fast32 ? (uint32_t)(((uint64_t)nb << 32) / D) : 0u;
    }
    __device__ __forceinline__ uint32_t operator()(uint64_t K) const {
        if (fast32) {
            /* x = K - kmin < 2^32 (keys lie in [kmin, kmax]); q0 = hi(x*m32) with
             * m32 = floor(2^32*bins/D) is floor(x*bins/D) or one less */
            const uint32_t x = (uint32_t)K - kmin32;
            uint32_t q = __umulhi(x, m32);
            const uint64_t p = (uint64_t)x * bins;
            q += ((uint64_t)(q + 1u) * D32 <= p) ? 1u : 0u;
            return min(q, bins - 1u);
        }
        if (D == 0) return 0;
        const uint64_t x = K <= kmin ? 0ull : (K - kmin >= D ? D : K - kmin);
        uint64_t q;
        if (fast) {
            const uint64_t p = x * (uint64_t)bins;
            q = __umul64hi(p, inv); /* <= floor(p/D), at most 2 below */
            while ((q + 1) * D <= p) q++;
        } else { /* exact 128-bit: b*D <= x*bins < (b+1)*D */
            const uint64_t plo = x * (uint64_t)bins, phi = __umul64hi(x, (uint64_t)bins);
            q = (uint64_t)((double)x * ((double)bins / (double)D));
            if (q > bins) q = bins;
            for (;;) {
                const uint64_t qlo = q * D, qhi = __umul64hi(q, D);
                if (q > 0 && (qhi > phi || (qhi == phi && qlo > plo))) q--;
                else break;
            }
            for (;;) {
                const uint64_t b1 = q + 1, qlo = b1 * D, qhi = __umul64hi(b1, D);
                if (qhi < phi || (qhi == phi && qlo <= plo)) q++;
                else break;
            }
        }
        return q > bins - 1 ? bins - 1 : (uint32_t)q;
    }
};

/* shared-memory u32 bin += c (c <= 2^20); a bin that reaches 2^31 is drained
 * into its u64 global bin (exchange, then add), so no shared bin ever wraps
 * however many keys one CTA bins */
__device__ __forceinline__ void sh_bin_add(uint32_t* shist, uint64_t* hist, uint32_t b, uint32_t c) {
    const uint32_t old = atomicAdd(&shist[b], c);
    if (old >= 0x80000000u - c) {
        const uint32_t x = atomicExch(&shist[b], 0u);
        atomicAdd((unsigned long long*)&hist[b], (unsigned long long)x);
    }
}

template <int SMAX>
struct St {
    uint32_t fa[SMAX], fb[SMAX];
    uint32_t cur;
    uint64_t I, M, K; /* open round's den*I_r and num*M_r; closed rounds' key */
};

/* SMAX == 0: run-length SM state for any (super-)SM count S > 32 (e.g. the
 * 148-SM B200 preset).  Within a round every SM's words are
 * fixed by how many blocks of each placed kernel it holds; one water-fill
 * changes that count uniformly except at the cursor and the new cursor, so
 * run boundaries are a subset of {0} U {cursor after each placement of the
 * round}: at most 1 + 16 runs (+1 transient). */
constexpr int RK_RUNS = RK_MAX_N + 2;
template <>
struct St<0> {
    uint32_t fa[RK_RUNS], fb[RK_RUNS], st[RK_RUNS]; /* run j = SMs [st[j], st[j+1]) (st[nr] := S) */
    uint32_t nr, cur;
    uint64_t I, M, K;
};

/* number of SMs: compile-time when FULL */
template <int SMAX, bool FULL>
__device__ __forceinline__ uint32_t nsm(const RkGTab& g) {
    if constexpr (FULL) return (uint32_t)SMAX;
    else return g.S;
}
template <int SMAX, bool FULL>
__device__ __forceinline__ bool live_sm(int i, const RkGTab& g) {
    if constexpr (FULL) return true;
    else return (uint32_t)i < g.S;
}

struct NoRec {
    __device__ __forceinline__ void add(uint32_t, uint32_t) {}
    __device__ __forceinline__ void close() {}
    __device__ __forceinline__ void full(uint32_t, uint32_t, uint32_t) {}
};

/* Records the round partition p[r][i] for rk_simulate_order. */
struct Rec {
    uint32_t* rounds;
    uint32_t max_rounds, n, r, scale; /* scale: SMs per super-SM */
    __device__ void add(uint32_t k, uint32_t cnt) {
        if (r < max_rounds) rounds[r * n + k] += cnt * scale;
    }
    __device__ void close() { r++; }
    __device__ void full(uint32_t k, uint32_t nfull, uint32_t sc) {
        for (uint32_t q = 0; q < nfull; q++) {
            add(k, sc);
            close();
        }
    }
};

template <int SMAX, bool FULL>
__device__ __forceinline__ void st_fresh(St<SMAX>& s, const RkGTab& g) {
    if constexpr (SMAX == 0) {
        s.nr = 1;
        s.st[0] = 0;
        s.fa[0] = g.freshA;
        s.fb[0] = g.freshB;
        s.cur = 0;
        s.I = s.M = s.K = 0;
        return;
    } else {
#pragma unroll
    for (int i = 0; i < SMAX; i++) {
        s.fa[i] = live_sm<SMAX, FULL>(i, g) ? g.freshA : 0u;
        s.fb[i] = live_sm<SMAX, FULL>(i, g) ? g.freshB : 0u;
    }
    s.cur = 0;
    s.I = s.M = s.K = 0;
    }
}

/* Capacity of one SM for kernel k: min(floor(regs/dr), floor(shm/ds),
 * floor(warps/dw), slots) — the four limits of PAPER:76-78, inclusive <=
 * (reading L8).  Fields are stored as 2x+1, so floor(x/d) = floor((2x+1)/(2d))
 * = IMAD.HI with a host-verified magic; a zero demand adds 0xFFFF instead. */
struct CapK {
    uint32_t mr, ms, mw, zr, zs;
};
__device__ __forceinline__ CapK capk(const RkKTab& k) { return CapK{k.mr, k.ms, k.mw, k.zr, k.zs}; }
__device__ __forceinline__ uint32_t cap1(uint32_t fa, uint32_t fb, const CapK& k) {
    /* zero demand: the numerator gets bits >= 2^30 (LOP3 OR / funnel shift, no
     * extra instruction) and the magic 0xFFFFFFFF keeps it >> any cap */
    const uint32_t qr = __umulhi((fa & 0xFFFFu) | k.zr, k.mr);
    const uint32_t qs = __umulhi(__funnelshift_r(fa, k.zs, 16), k.ms);
    const uint32_t qw = __umulhi(fb & 0xFFFFu, k.mw); /* warps demand >= 1 */
    return min(__vimin3_u32(qr, qs, qw), fb >> 17);
}

/* complete single-kernel rounds among x = n - 1 leftover blocks: floor(x / SC) */
__device__ __forceinline__ uint32_t full_rounds(uint32_t x, const RkKTab& k) {
    uint32_t q = __umulhi(x, k.scm); /* exact for x < T (host-verified) */
    if (k.scm == 0) q = k.SC == 1 ? x : x / k.SC; /* SC == 1 or an unverifiable bound */
    return q;
}

/* Ring rotation of an S-bit mask (S <= 32). */
template <int SMAX, bool FULL>
__device__ __forceinline__ uint32_t rotr_s(uint32_t m, uint32_t r, uint32_t S) {
    if constexpr (FULL && SMAX == 1) {
        return m;
    } else if constexpr (FULL && SMAX <= 16) {
        return ((m | (m << SMAX)) >> r) & ((1u << SMAX) - 1u);
    } else {
        const uint64_t mm = (uint64_t)m | ((uint64_t)m << S);
        const uint32_t full = (S >= 32) ? 0xFFFFFFFFu : ((1u << S) - 1u);
        return (uint32_t)(mm >> r) & full;
    }
}

/* 0-based position of the r-th (1-based) set bit of m (r <= popc(m)). */
template <int SMAX>
__device__ __forceinline__ uint32_t select_bit(uint32_t m, uint32_t r) {
    uint32_t p = 0;
#pragma unroll
    for (int w = SMAX / 2; w >= 1; w >>= 1) {
        const uint32_t lowc = __popc(m & ((1u << w) - 1u));
        if (lowc < r) {
            r -= lowc;
            m >>= w;
            p += (uint32_t)w;
        }
    }
    return p;
}

/* Outcome of placing kernel k into an SM state (everything but the per-SM words). */
struct Placed {
    uint32_t cur;
    uint64_t I, M, K;
};

/* Water-fill of n blocks (1 <= n <= sum c) with capacities c[] on the SM
 * words (bfa, bfb) from cursor cur: after tlo passes every SM holds
 * min(c_s, tlo); pass tlo+1 gives one more block to the first r SMs with
 * c_s > tlo in ring order.  Emits the new words via upd; returns the cursor. */
template <int SMAX, bool FULL, class U>
__device__ __forceinline__ uint32_t water_fill(uint32_t n, const uint32_t (&c)[SMAX], const uint32_t (&bfa)[SMAX],
                                               const uint32_t (&bfb)[SMAX], uint32_t cur, const RkKTab& k,
                                               const RkGTab& g, U& upd) {
    const uint32_t S = nsm<SMAX, FULL>(g);
    /* tlo = max{t : f(t) < n}, f(t) = sum_s min(c_s, t); SM pairs in 16x2 SIMD */
    constexpr int NP = SMAX / 2;
    uint32_t cp[NP > 0 ? NP : 1];
#pragma unroll
    for (int j = 0; j < NP; j++) cp[j] = __byte_perm(c[2 * j], c[2 * j + 1], 0x5410);
    uint32_t tlo, flo;
    if constexpr (FULL && SMAX == 1) {
        tlo = n - 1u; /* f(t) = min(c, t) < n  <=>  t < n (n <= c) */
        flo = tlo;
    } else if constexpr (FULL && SMAX == 2) {
        /* f(t) = 2t up to the smaller cap lo, then lo + t (n <= lo + hi) */
        const uint32_t lo = min(c[0], c[1]);
        const bool even = n <= 2u * lo;
        tlo = even ? (n - 1u) >> 1 : n - 1u - lo;
        flo = even ? 2u * tlo : n - 1u;
    } else {
        tlo = 0;
        flo = 0;
        for (uint32_t b = g.tbits; b; b >>= 1) {
            const uint32_t tt = tlo + b;
            uint32_t f;
            if constexpr (NP > 0) {
                const uint32_t t2 = tt * 0x10001u;
                uint32_t s2 = 0;
#pragma unroll
                for (int j = 0; j < NP; j++) s2 += __vminu2(cp[j], t2);
                f = (s2 & 0xFFFFu) + (s2 >> 16);
            } else {
                f = min(c[0], tt);
            }
            if (f < n) {
                tlo = tt;
                flo = f;
            }
        }
    }
    const uint32_t r = n - flo; /* >= 1 blocks of pass tlo+1, to SMs with c_s > tlo in ring order */
    if constexpr (FULL && SMAX == 1) {
        upd(0, bfa[0] - n * k.dA, bfb[0] - n * k.dB); /* one SM takes all n (n <= c) */
        return 0u;
    } else if constexpr (FULL && SMAX == 2) {
        /* ring order from the cursor: SM a = cur, then SM b.  r == 2: both get
         * pass tlo+1 (both eligible), the last lands on b, cursor stays;
         * r == 1: the first eligible of (a, b) gets it, cursor = the other. */
        const uint32_t a = cur, ca = a ? c[1] : c[0], cb = a ? c[0] : c[1];
        const bool ea = ca > tlo, two = r == 2u;
        const uint32_t xa = min(ca, tlo) + ((two || ea) ? 1u : 0u);
        const uint32_t xb = min(cb, tlo) + ((two || !ea) ? 1u : 0u);
        const uint32_t x0 = a ? xb : xa, x1 = a ? xa : xb;
        upd(0, bfa[0] - x0 * k.dA, bfb[0] - x0 * k.dB);
        upd(1, bfa[1] - x1 * k.dA, bfb[1] - x1 * k.dB);
        return (two || !ea) ? a : 1u - a;
    }
    uint32_t E;
    if constexpr (NP > 0 && SMAX <= 16) {
        /* E = {s : c_s > tlo}: per pair min(c, tlo+1) - min(c, tlo) is 0/1 in each half */
        const uint32_t lo2 = tlo * 0x10001u, hi2 = lo2 + 0x10001u;
        uint32_t acc = 0;
#pragma unroll
        for (int j = 0; j < NP; j++) acc += (__vminu2(cp[j], hi2) - __vminu2(cp[j], lo2)) << (2 * j);
        E = (acc & 0x5555u) | ((acc >> 15) & 0xAAAAu);
    } else {
        E = 0;
#pragma unroll
        for (int i = 0; i < SMAX; i++) E |= (c[i] > tlo ? 1u : 0u) << i;
    }
    const uint32_t Er = rotr_s<SMAX, FULL>(E, cur, S);
    const uint32_t p = select_bit<SMAX>(Er, r);
    const uint32_t Xr = Er & ((2u << p) - 1u); /* first r eligible SMs from the cursor */
    const uint32_t X = rotr_s<SMAX, FULL>(Xr, S - cur, S);
    const uint32_t nc = cur + p + 1u;
#pragma unroll
    for (int i = 0; i < SMAX; i++) {
        const uint32_t x = min(c[i], tlo) + ((X >> i) & 1u);
        upd(i, bfa[i] - x * k.dA, bfb[i] - x * k.dB);
    }
    return nc >= S ? nc - S : nc; /* cursor = SM of the last block + 1 */
}

/* Dispatch all T_k blocks of kernel k on state `in`; the new
 * per-SM words are handed to upd(i, fa, fb) so callers either store them
 * (a new state) or consume them on the fly (the fused last level). */
/* ST = false: a variant compiled without the strict round-robin reading (the
 * direct kernels branch once per launch on the flag) */
template <int SMAX, bool FULL, class R, class U, bool ST = true>
__device__ __forceinline__ Placed place_core(const St<SMAX>& in, const RkKTab& k, uint32_t kid, const RkGTab& g,
                                             R& rec, U& upd) {
    const CapK ck = capk(k);
    uint32_t c[SMAX];
    uint32_t F = 0;
#pragma unroll
    for (int i = 0; i < SMAX; i++) {
        c[i] = cap1(in.fa[i], in.fb[i], ck);
        F += c[i];
    }
    if (ST && (g.flags & RK_FLAG_STRICT_RR)) {
        /* L4 read literally: block b goes to SM (cur + b) mod S, so the round holds
         * m = min_s ((s - cur) mod S + c_s S) of them (m <= F: SM s receives
         * ceil((m - d_s) / S) <= c_s).  Up to m blocks that round robin never meets
         * a full SM, so the water-fill below places them identically; beyond m the
         * round closes and the rest is the same fresh-round fill — strict RR is the
         * default dispatch with F := m. */
        const uint32_t S = nsm<SMAX, FULL>(g);
        const uint32_t cur = (g.flags & RK_FLAG_CURSOR_PER_KERNEL) ? 0u : in.cur;
        uint32_t m = 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < SMAX; i++) {
            const uint32_t d = (uint32_t)i >= cur ? (uint32_t)i - cur : (uint32_t)i + S - cur;
            if (live_sm<SMAX, FULL>(i, g)) m = min(m, d + c[i] * S);
        }
        F = min(F, m);
        /* the new cursor, for consumers that need it before the words (StrictCapUpd) */
        const uint32_t n = k.T;
        const uint32_t nr = n > F ? n - F - full_rounds(n - F - 1u, k) * k.SC : cur + n;
        upd.set_cursor(nr % S);
    }
    uint32_t n = k.T;
    Placed o;
    const bool ovf = n > F;
    /* n > F: every SM takes its c_s and the next block fits nowhere, so the round
     * closes; complete single-kernel rounds follow; the rest opens a
     * fresh round (all SMs fresh, cursor 0) — the same water-fill on fresh inputs. */
    const uint32_t nfull = full_rounds(ovf ? n - F - 1u : 0u, k);
    if (ovf) {
        rec.add(kid, F);
        rec.close();
        rec.full(kid, nfull, k.SC);
    }
    if constexpr (SMAX <= RK_BF_MAX) {
        /* branch-free: lanes disagree on ovf often; the fresh round is the same
         * water-fill on fresh words, so select the inputs instead of branching */
        const uint64_t kc = in.K + round_key(in.I + (uint64_t)F * k.cA, in.M + (uint64_t)F * k.cM, g.num, g.den) +
                            (uint64_t)nfull * k.fullkey;
        n = ovf ? n - F - nfull * k.SC : n;
        o.K = ovf ? kc : in.K;
        uint32_t bfa[SMAX], bfb[SMAX];
#pragma unroll
        for (int i = 0; i < SMAX; i++) {
            const bool live = live_sm<SMAX, FULL>(i, g);
            bfa[i] = ovf ? (live ? g.freshA : 0u) : in.fa[i];
            bfb[i] = ovf ? (live ? g.freshB : 0u) : in.fb[i];
            c[i] = ovf ? (live ? k.C : 0u) : c[i];
        }
        o.cur = water_fill<SMAX, FULL>(n, c, bfa, bfb, (ovf || (g.flags & RK_FLAG_CURSOR_PER_KERNEL)) ? 0u : in.cur,
                                           k, g, upd);
        o.I = (ovf ? 0ull : in.I) + (uint64_t)n * k.cA;
        o.M = (ovf ? 0ull : in.M) + (uint64_t)n * k.cM;
    } else {
        if (ovf) {
            o.K = in.K + round_key(in.I + (uint64_t)F * k.cA, in.M + (uint64_t)F * k.cM, g.num, g.den) +
                  (uint64_t)nfull * k.fullkey;
            n -= F + nfull * k.SC;
            uint32_t q, r;
            if constexpr (FULL) {
                q = n / (uint32_t)SMAX; /* power of two: a shift */
                r = n % (uint32_t)SMAX;
            } else {
                q = n / g.S;
                r = n - q * g.S;
            }
#pragma unroll
            for (int i = 0; i < SMAX; i++) {
                const uint32_t x = q + ((uint32_t)i < r ? 1u : 0u);
                if (live_sm<SMAX, FULL>(i, g)) upd(i, g.freshA - x * k.dA, g.freshB - x * k.dB);
                else upd(i, 0u, 0u);
            }
            o.cur = r;
            o.I = (uint64_t)n * k.cA;
            o.M = (uint64_t)n * k.cM;
        } else {
            o.cur = water_fill<SMAX, FULL>(n, c, in.fa, in.fb, (g.flags & RK_FLAG_CURSOR_PER_KERNEL) ? 0u : in.cur,
                                           k, g, upd);
            o.I = in.I + (uint64_t)n * k.cA;
            o.M = in.M + (uint64_t)n * k.cM;
            o.K = in.K;
        }
    }
    rec.add(kid, n);
    return o;
}

template <int SMAX>
struct StoreUpd {
    St<SMAX>& out;
    __device__ __forceinline__ void set_cursor(uint32_t) {}
    __device__ __forceinline__ void operator()(int i, uint32_t a, uint32_t b) {
        out.fa[i] = a;
        out.fb[i] = b;
    }
};

struct CapSumUpd { /* consume the new words: capacity sum for the next kernel */
    CapK k;
    uint32_t F;
    __device__ __forceinline__ void set_cursor(uint32_t) {}
    __device__ __forceinline__ void operator()(int, uint32_t a, uint32_t b) { F += cap1(a, b, k); }
};

/* strict round robin (RK_FLAG_STRICT_RR): the next kernel's blocks go to SM (cur + b) mod S, so the
 * first that cannot be placed is b = min_s ((s - cur) mod S + c_s S); consumes the new words once the
 * placing kernel has set the new cursor (0 for the cursor-per-kernel reading) */
struct StrictCapUpd {
    CapK k;
    uint32_t S, cur, m;
    bool perk;
    __device__ __forceinline__ void set_cursor(uint32_t c) { cur = perk ? 0u : c; }
    __device__ __forceinline__ void operator()(int i, uint32_t a, uint32_t b) {
        if ((uint32_t)i >= S) return;
        const uint32_t d = (uint32_t)i >= cur ? (uint32_t)i - cur : (uint32_t)i + S - cur;
        m = min(m, d + cap1(a, b, k) * S);
    }
};

struct CapBothUpd { /* CapSumUpd and StrictCapUpd in one pass */
    CapK k;
    uint32_t F, S, cur, m;
    bool perk;
    __device__ __forceinline__ void set_cursor(uint32_t c) { cur = perk ? 0u : c; }
    __device__ __forceinline__ void operator()(int i, uint32_t a, uint32_t b) {
        const uint32_t c = cap1(a, b, k);
        F += c;
        const uint32_t d = (uint32_t)i >= cur ? (uint32_t)i - cur : (uint32_t)i + S - cur;
        if ((uint32_t)i < S) m = min(m, d + c * S);
    }
};

/* ---- run-length state (SMAX == 0): the same dispatch rules (PAPER:69-81,
 * readings L4/L5) as place_core, on runs of identical SMs ---- */
__device__ __forceinline__ uint32_t rle_end(const St<0>& s, uint32_t j, uint32_t S) {
    return j + 1 < s.nr ? s.st[j + 1] : S;
}

/* total capacity sum_s c_s of the state for kernel k */
__device__ __forceinline__ uint32_t rle_capsum(const St<0>& s, const CapK& ck, uint32_t S) {
    uint32_t F = 0;
    for (uint32_t j = 0; j < s.nr; j++) F += (rle_end(s, j, S) - s.st[j]) * cap1(s.fa[j], s.fb[j], ck);
    return F;
}

template <class R>
__device__ void rle_place(const St<0>& in, St<0>& out, const RkKTab& k, uint32_t kid, const RkGTab& g, R& rec) {
    const CapK ck = capk(k);
    const uint32_t S = g.S;
    uint32_t c[RK_RUNS];
    uint32_t F = 0;
    for (uint32_t j = 0; j < in.nr; j++) {
        c[j] = cap1(in.fa[j], in.fb[j], ck);
        F += (rle_end(in, j, S) - in.st[j]) * c[j];
    }
    uint32_t n = k.T;
    if (n > F) { /* round closes; full rounds; fresh round from SM 0 */
        rec.add(kid, F);
        rec.close();
        const uint32_t nfull = full_rounds(n - F - 1u, k);
        rec.full(kid, nfull, k.SC);
        const uint64_t K = in.K + round_key(in.I + (uint64_t)F * k.cA, in.M + (uint64_t)F * k.cM, g.num, g.den) +
                           (uint64_t)nfull * k.fullkey;
        n -= F + nfull * k.SC;
        const uint32_t q = n / S, r = n - q * S;
        out.st[0] = 0;
        out.fa[0] = g.freshA - (q + (r ? 1u : 0u)) * k.dA;
        out.fb[0] = g.freshB - (q + (r ? 1u : 0u)) * k.dB;
        out.nr = 1;
        if (r) {
            out.st[1] = r;
            out.fa[1] = g.freshA - q * k.dA;
            out.fb[1] = g.freshB - q * k.dB;
            out.nr = 2;
        }
        out.cur = r;
        out.K = K;
        out.I = (uint64_t)n * k.cA;
        out.M = (uint64_t)n * k.cM;
        rec.add(kid, n);
        return;
    }
    const uint32_t cur = (g.flags & RK_FLAG_CURSOR_PER_KERNEL) ? 0u : in.cur;
    /* tlo = max{t : f(t) < n}, f(t) = sum_runs len * min(c, t) */
    uint32_t tlo = 0, flo = 0;
    for (uint32_t b = g.tbits; b; b >>= 1) {
        const uint32_t tt = tlo + b;
        uint32_t f = 0;
        for (uint32_t j = 0; j < in.nr; j++) f += (rle_end(in, j, S) - in.st[j]) * min(c[j], tt);
        if (f < n) {
            tlo = tt;
            flo = f;
        }
    }
    /* pass tlo+1: one more block to the first r eligible (c > tlo) SMs in ring
     * order from the cursor; nc = the SM after the r-th one */
    uint32_t need = n - flo;
    uint32_t jc = 0;
    for (uint32_t j = 1; j < in.nr; j++)
        if (in.st[j] <= cur) jc = j;
    uint32_t nc = cur;
    for (uint32_t step = 0; step <= in.nr; step++) {
        const uint32_t j = (jc + step) % in.nr;
        const uint32_t lo = step == 0 ? cur : in.st[j];
        const uint32_t hi = step == in.nr ? cur : rle_end(in, j, S);
        if (c[j] > tlo && hi > lo) {
            if (need <= hi - lo) {
                nc = lo + need;
                break;
            }
            need -= hi - lo;
        }
    }
    if (nc >= S) nc -= S;
    const uint32_t L = nc > cur ? nc - cur : nc + S - cur; /* ring interval [cur, cur+L) got pass tlo+1 */
    St<0> o;
    o.nr = 0;
    for (uint32_t j = 0; j < in.nr; j++) {
        const uint32_t lo = in.st[j], hi = rle_end(in, j, S);
        uint32_t cut1 = (cur > lo && cur < hi) ? cur : hi, cut2 = (nc > lo && nc < hi) ? nc : hi;
        if (cut2 < cut1) {
            const uint32_t x = cut1;
            cut1 = cut2;
            cut2 = x;
        }
        const uint32_t base = min(c[j], tlo), elig = c[j] > tlo ? 1u : 0u;
        const uint32_t ps[3] = {lo, cut1, cut2};
        for (int q = 0; q < 3; q++) {
            const uint32_t pstart = ps[q];
            if (pstart >= hi || (q > 0 && pstart == ps[q - 1])) continue;
            const uint32_t d = pstart >= cur ? pstart - cur : pstart + S - cur;
            const uint32_t x = base + ((d < L) ? elig : 0u);
            const uint32_t a = in.fa[j] - x * k.dA, b = in.fb[j] - x * k.dB;
            if (o.nr && o.fa[o.nr - 1] == a && o.fb[o.nr - 1] == b) continue; /* merge equal neighbours */
            if (o.nr < (uint32_t)RK_RUNS) {
                o.st[o.nr] = pstart;
                o.fa[o.nr] = a;
                o.fb[o.nr] = b;
                o.nr++;
            }
        }
    }
    o.cur = nc;
    o.I = in.I + (uint64_t)n * k.cA;
    o.M = in.M + (uint64_t)n * k.cM;
    o.K = in.K;
    rec.add(kid, n);
    out = o;
}

template <int SMAX, bool FULL, bool ST = true, class R>
__device__ __forceinline__ void place(const St<SMAX>& in, St<SMAX>& out, const RkKTab& k, uint32_t kid,
                                      const RkGTab& g, R& rec) {
    if constexpr (SMAX == 0) {
        rle_place(in, out, k, kid, g, rec);
        return;
    } else {
    StoreUpd<SMAX> u{out};
    const Placed o = place_core<SMAX, FULL, R, StoreUpd<SMAX>, ST>(in, k, kid, g, rec, u);
    out.cur = o.cur;
    out.I = o.I;
    out.M = o.M;
    out.K = o.K;
    }
}

/* The last kernel of an order: only its split into the open round and fresh
 * rounds matters (F = its total capacity on the final state). */
template <class R>
__device__ __forceinline__ uint64_t finish_key(uint32_t F, uint64_t I, uint64_t M, uint64_t K, const RkKTab& k,
                                               uint32_t kid, const RkGTab& g, R& rec) {
    uint32_t n = k.T;
    if (n <= F) {
        rec.add(kid, n);
        rec.close();
        return K + round_key(I + (uint64_t)n * k.cA, M + (uint64_t)n * k.cM, g.num, g.den);
    }
    rec.add(kid, F);
    rec.close();
    K += round_key(I + (uint64_t)F * k.cA, M + (uint64_t)F * k.cM, g.num, g.den);
    n -= F;
    const uint32_t nfull = full_rounds(n - 1u, k);
    K += (uint64_t)nfull * k.fullkey;
    rec.full(kid, nfull, k.SC);
    n -= nfull * k.SC;
    rec.add(kid, n);
    rec.close();
    return K + round_key((uint64_t)n * k.cA, (uint64_t)n * k.cM, g.num, g.den);
}

template <int SMAX, bool ST = true, class R>
__device__ __forceinline__ uint64_t finish(const St<SMAX>& s, const RkKTab& k, uint32_t kid, const RkGTab& g,
                                           R& rec) {
    const CapK ck = capk(k);
    uint32_t F = 0;
    if constexpr (SMAX == 0) {
        F = rle_capsum(s, ck, g.S);
    } else if (ST && (g.flags & RK_FLAG_STRICT_RR)) { /* the first block that does not fit on its SM */
        StrictCapUpd u{ck, g.S, 0u, 0xFFFFFFFFu, (g.flags & RK_FLAG_CURSOR_PER_KERNEL) != 0};
        u.set_cursor(s.cur);
#pragma unroll
        for (int i = 0; i < SMAX; i++) u(i, s.fa[i], s.fb[i]);
        F = u.m;
    } else {
#pragma unroll
        for (int i = 0; i < SMAX; i++) F += cap1(s.fa[i], s.fb[i], ck);
    }
    return finish_key(F, s.I, s.M, s.K, k, kid, g, rec);
}

/* place kb on `in`, then evaluate the last kernel kc — leaf of the suffix tree */
template <int SMAX, bool FULL, bool ST = true>
__device__ __forceinline__ uint64_t place_finish(const St<SMAX>& in, const RkKTab& kb, uint32_t kbid,
                                                 const RkKTab& kc, uint32_t kcid, const RkGTab& g) {
    NoRec nr;
    if constexpr (SMAX == 0) {
        St<0> s1;
        rle_place(in, s1, kb, kbid, g, nr);
        return finish<0>(s1, kc, kcid, g, nr);
    } else {
        if constexpr (!ST) {
            CapSumUpd u{capk(kc), 0u};
            const Placed o = place_core<SMAX, FULL, NoRec, CapSumUpd, false>(in, kb, kbid, g, nr, u);
            return finish_key(u.F, o.I, o.M, o.K, kc, kcid, g, nr);
        }
        /* one placement, both fits of kc: the capacity sum and, for strict round
         * robin, the first block that fails from kb's new cursor (set before the words) */
        CapBothUpd u{capk(kc), 0u, nsm<SMAX, FULL>(g), 0u, 0xFFFFFFFFu, (g.flags & RK_FLAG_CURSOR_PER_KERNEL) != 0};
        const Placed o = place_core<SMAX, FULL>(in, kb, kbid, g, nr, u);
        return finish_key((g.flags & RK_FLAG_STRICT_RR) ? u.m : u.F, o.I, o.M, o.K, kc, kcid, g, nr);
    }
}

/* Nibble list of unused kernels, ascending: remove and return entry d. */
__device__ __forceinline__ uint32_t take_nibble(uint64_t& L, uint32_t d) {
    const uint32_t sh = 4u * d;
    const uint32_t v = (uint32_t)(L >> sh) & 15u;
    const uint64_t low = L & ((1ull << sh) - 1ull);
    const uint64_t high = sh + 4u >= 64u ? 0ull : (L >> (sh + 4u)) << sh;
    L = low | high;
    return v;
}
__device__ __forceinline__ uint64_t identity_list(uint32_t n) {
    uint64_t L = 0;
    for (uint32_t i = 0; i < n; i++) L |= (uint64_t)i << (4u * i);
    return L;
}

/* Key of one lexicographic index, from scratch (candidate, samples, n < 3). */
template <int SMAX, bool FULL, class R>
__device__ uint64_t eval_index(const RkTables& t, uint64_t idx, R& rec) {
    const RkGTab& g = t.g;
    const uint32_t n = g.n;
    St<SMAX> s;
    st_fresh<SMAX, FULL>(s, g);
    uint64_t L = identity_list(n);
    uint64_t rem = idx;
    for (uint32_t j = 0; j + 1 < n; j++) {
        const uint64_t f = g.fact[n - 1 - j];
        const uint32_t d = (uint32_t)(rem / f);
        rem -= (uint64_t)d * f;
        const uint32_t k = take_nibble(L, d);
        St<SMAX> s2;
        place<SMAX, FULL>(s, s2, t.k[k], k, g, rec);
        s = s2;
    }
    const uint32_t k = (uint32_t)L & 15u;
    return finish<SMAX>(s, t.k[k], k, g, rec);
}

struct TStats {
    uint64_t kmin, kmax, amin, amax;
    uint32_t nlt, neq, cnt; /* per thread (< 2^32 orders per thread) */
    __device__ __forceinline__ void init() {
        kmin = ~0ull;
        kmax = 0;
        amin = amax = ~0ull;
        nlt = neq = cnt = 0;
    }
    /* updated per run by Leaf::end_run (reading L12: smallest index on ties) */
};

/* Records may carry counts without evaluated orders (a lane that counted a
 * row of another lane's run): counts always add, extremes come only from
 * records with evaluated > 0. */
__device__ __forceinline__ void merge_into(rk_stats& a, const rk_stats& b) {
    if (b.evaluated == 0) {
        a.n_lt += b.n_lt;
        a.n_eq += b.n_eq;
        a.n_gt += b.n_gt;
        return;
    }
    if (a.evaluated == 0) {
        const uint64_t lt = a.n_lt, eq = a.n_eq, gt = a.n_gt;
        a = b;
        a.n_lt += lt;
        a.n_eq += eq;
        a.n_gt += gt;
        return;
    }
    if (b.key_min < a.key_min || (b.key_min == a.key_min && b.argmin < a.argmin)) {
        a.key_min = b.key_min;
        a.argmin = b.argmin;
    }
    if (b.key_max > a.key_max || (b.key_max == a.key_max && b.argmax < a.argmax)) {
        a.key_max = b.key_max;
        a.argmax = b.argmax;
    }
    a.n_lt += b.n_lt;
    a.n_eq += b.n_eq;
    a.n_gt += b.n_gt;
    a.evaluated += b.evaluated;
}

__device__ __forceinline__ rk_stats to_rec(const TStats& t) {
    rk_stats r;
    r.key_min = t.kmin;
    r.key_max = t.kmax;
    r.argmin = t.amin;
    r.argmax = t.amax;
    r.n_lt = t.nlt;
    r.n_eq = t.neq;
    r.n_gt = (uint64_t)(t.cnt - t.nlt - t.neq);
    r.evaluated = t.cnt;
    return r;
}

__device__ __forceinline__ rk_stats shfl_rec(const rk_stats& a, int off) {
    rk_stats b;
    b.key_min = __shfl_xor_sync(0xFFFFFFFFu, a.key_min, off);
    b.key_max = __shfl_xor_sync(0xFFFFFFFFu, a.key_max, off);
    b.argmin = __shfl_xor_sync(0xFFFFFFFFu, a.argmin, off);
    b.argmax = __shfl_xor_sync(0xFFFFFFFFu, a.argmax, off);
    b.n_lt = __shfl_xor_sync(0xFFFFFFFFu, a.n_lt, off);
    b.n_eq = __shfl_xor_sync(0xFFFFFFFFu, a.n_eq, off);
    b.n_gt = __shfl_xor_sync(0xFFFFFFFFu, a.n_gt, off);
    b.evaluated = __shfl_xor_sync(0xFFFFFFFFu, a.evaluated, off);
    return b;
}

/* warp shuffle -> shared memory -> one record per CTA (all threads must call) */
__device__ rk_stats block_reduce(rk_stats v) {
    __shared__ rk_stats warp_recs[32];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        rk_stats o = shfl_rec(v, off);
        merge_into(v, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) warp_recs[wid] = v;
    __syncthreads();
    rk_stats r{};
    r.evaluated = 0;
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        if (lane < nw) r = warp_recs[lane];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            rk_stats o = shfl_rec(r, off);
            merge_into(r, o);
        }
    }
    return r; /* valid in warp 0 */
}

/* Per-CTA record, then the last CTA to finish merges all records (no extra
 * launch; the counter resets itself). */
__device__ void commit(const rk_stats& cta, rk_stats* recs, uint32_t* counter, rk_stats* out) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        recs[blockIdx.x] = cta;
        __threadfence();
        uint32_t prev = atomicAdd(counter, 1u);
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    rk_stats v{};
    v.evaluated = 0;
    for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
        const rk_stats* q = recs + i; /* written by other CTAs: read through L2 */
        rk_stats o;
        o.key_min = __ldcg(&q->key_min);
        o.key_max = __ldcg(&q->key_max);
        o.argmin = __ldcg(&q->argmin);
        o.argmax = __ldcg(&q->argmax);
        o.n_lt = __ldcg(&q->n_lt);
        o.n_eq = __ldcg(&q->n_eq);
        o.n_gt = __ldcg(&q->n_gt);
        o.evaluated = __ldcg(&q->evaluated);
        merge_into(v, o);
    }
    rk_stats r = block_reduce(v);
    if (threadIdx.x == 0) {
        *out = r;
        *counter = 0;
    }
}


/* Suffix-tree depth per SM-count variant: placements are cheap for few
 * (super-)SMs, so share longer prefixes (DESIGN.md §5 "prefix sharing"). */
#ifndef RK_DEPTH_LARGE
#define RK_DEPTH_LARGE 3
#endif
#ifndef RK_DEPTH_SMALL
#define RK_DEPTH_SMALL 5
#endif
template <int SMAX>
struct Depth {
    static constexpr int value = SMAX == 0 ? RK_DEPTH_LARGE : (SMAX <= 2 ? RK_DEPTH_SMALL : (SMAX <= 8 ? 4 : RK_DEPTH_LARGE));
};
__host__ __device__ constexpr uint32_t cfact(int m) { return m <= 1 ? 1u : (uint32_t)m * cfact(m - 1); }

/* One evaluated order.  Leaves are visited run by run; inside a run by a u32
 * offset (the run's first index run0 is u64).  Per-run extremes and counts are
 * folded into the thread's TStats at the run's end (offsets increase inside a
 * run and runs increase per thread, so strict compares keep the smallest index
 * on ties).  EXTRA adds the compact-key and fused-histogram outputs. */
template <bool EXTRA>
struct Leaf {
    TStats& ts;
    uint64_t* keys;   /* u64 keys (nullable) */
    uint32_t* keys32; /* EXTRA: compact u32 offsets K - base (ovf set if one does not fit) */
    uint64_t base;
    uint32_t ovf;
    uint64_t lo, hi, first;
    uint64_t cand;
    uint32_t* shist; /* EXTRA: fused Fig. 1 binning (second pass without stored keys) */
    uint64_t* ghist; /* its u64 global bins (drained into when a shared bin nears 2^31) */
    BinCalc bc;
    uint32_t hcur, hrun;
    /* per run */
    uint64_t run0;
    uint32_t olo, ohi;
    uint64_t* kout;
    uint32_t* kout32;
    uint64_t rmin, rmax;
    uint32_t omin, omax, rlt, req;
    bool pair_ok; /* kout 16-byte aligned for pair stores */

    __device__ __forceinline__ void begin_run(uint64_t r0, uint32_t R) {
        run0 = r0;
        olo = lo > r0 ? (uint32_t)(lo - r0) : 0u;
        ohi = hi < r0 + R ? (uint32_t)(hi - r0) : R;
        kout = keys ? keys + (r0 - first) : nullptr;
        pair_ok = (reinterpret_cast<uintptr_t>(kout) & 15u) == 0;
        if (EXTRA) kout32 = keys32 ? keys32 + (r0 - first) : nullptr;
        rmin = ~0ull;
        rmax = 0;
        omin = omax = 0;
        rlt = req = 0;
    }
    __device__ __forceinline__ void operator()(uint32_t off, uint64_t K) {
        if (off >= olo && off < ohi) {
            if (K < rmin) { rmin = K; omin = off; }
            if (K > rmax) { rmax = K; omax = off; } /* K >= 1 > 0 */
            rlt += (K < cand) ? 1u : 0u;
            req += (K == cand) ? 1u : 0u;
            if (kout) kout[off] = K;
            if constexpr (EXTRA) {
                if (kout32) {
                    const uint64_t x = K - base;
                    ovf |= (x >> 32) != 0 ? 1u : 0u;
                    kout32[off] = (uint32_t)x;
                }
                if (shist) {
                    const uint32_t b = bc(K);
                    if (b == hcur && hrun < (1u << 20)) {
                        hrun++;
                    } else {
                        if (hrun) sh_bin_add(shist, ghist, hcur, hrun);
                        hcur = b;
                        hrun = 1;
                    }
                }
            }
        }
    }
    /* the two leaves of a depth-2 node: offsets off, off+1 (off even) */
    __device__ __forceinline__ void pair(uint32_t off, uint64_t K0, uint64_t K1) {
        if (!EXTRA && kout && off >= olo && off + 1u < ohi && pair_ok) {
            /* both in range: statistics, then one 16-byte store (fuller sectors) */
            const uint32_t o1 = off + 1u;
            if (K0 < rmin) { rmin = K0; omin = off; }
            if (K1 < rmin) { rmin = K1; omin = o1; }
            if (K0 > rmax) { rmax = K0; omax = off; }
            if (K1 > rmax) { rmax = K1; omax = o1; }
            rlt += ((K0 < cand) ? 1u : 0u) + ((K1 < cand) ? 1u : 0u);
            req += ((K0 == cand) ? 1u : 0u) + ((K1 == cand) ? 1u : 0u);
            *reinterpret_cast<ulonglong2*>(kout + off) = make_ulonglong2(K0, K1);
            return;
        }
        (*this)(off, K0);
        (*this)(off + 1u, K1);
    }
    __device__ __forceinline__ void end_run() {
        if (ohi <= olo) return;
        if (rmin < ts.kmin) { ts.kmin = rmin; ts.amin = run0 + omin; }
        if (rmax > ts.kmax) { ts.kmax = rmax; ts.amax = run0 + omax; }
        ts.nlt += rlt;
        ts.neq += req;
        ts.cnt += ohi - olo;
    }
    __device__ __forceinline__ void flush() {
        if constexpr (EXTRA)
            if (shist && hrun) sh_bin_add(shist, ghist, hcur, hrun);
        hrun = 0;
    }
};

/* The D kernels left after a prefix are the low D nibbles of `rem` (ascending);
 * visit their D! orders in lexicographic order, leaf offsets off .. off+D!-1. */
template <int SMAX, bool FULL, int D, class LF, bool ST = true>
__device__ __forceinline__ void dfs(const RkTables& t, const St<SMAX>& s, uint32_t rem, uint32_t off, LF& leaf) {
    if constexpr (D == 2) {
        const uint32_t x = rem & 15u, y = (rem >> 4) & 15u;
        const uint64_t K0 = place_finish<SMAX, FULL, ST>(s, t.k[x], x, t.k[y], y, t.g);
        const uint64_t K1 = place_finish<SMAX, FULL, ST>(s, t.k[y], y, t.k[x], x, t.g);
        leaf.pair(off, K0, K1);
    } else {
        NoRec nr;
#pragma unroll 1
        for (uint32_t a = 0; a < (uint32_t)D; a++) {
            const uint32_t sh = 4u * a;
            const uint32_t ka = (rem >> sh) & 15u;
            const uint32_t rest = (rem & ((1u << sh) - 1u)) | ((rem >> (sh + 4u)) << sh);
            St<SMAX> s1;
            place<SMAX, FULL, ST>(s, s1, t.k[ka], ka, t.g, nr);
            dfs<SMAX, FULL, D - 1, LF, ST>(t, s1, rest, off + a * cfact(D - 1), leaf);
        }
    }
}

/* A run = the D! consecutive indices sharing an (n-D)-prefix. */
template <int SMAX, bool FULL, int D, class LF, bool ST = true>
__device__ __forceinline__ void eval_run(const RkTables& t, uint64_t run, LF& leaf) {
    const RkGTab& g = t.g;
    const uint32_t n = g.n;
    NoRec nr;
    const uint64_t idx0 = run * cfact(D);
    leaf.begin_run(idx0, cfact(D));
    St<SMAX> s0;
    st_fresh<SMAX, FULL>(s0, g);
    uint64_t L = identity_list(n);
    uint64_t rem = idx0;
    for (uint32_t j = 0; j + D < n; j++) { /* shared (n-D)-prefix */
        const uint64_t f = g.fact[n - 1 - j];
        uint32_t d;
        if (rem < (1ull << 32) && f < (1ull << 32)) { /* 32-bit division when it fits (n <= 12) */
            d = (uint32_t)rem / (uint32_t)f;
        } else {
            d = (uint32_t)(rem / f);
        }
        rem -= (uint64_t)d * f;
        const uint32_t k = take_nibble(L, d);
        place<SMAX, FULL, ST>(s0, s0, t.k[k], k, g, nr);
    }
    dfs<SMAX, FULL, D, LF, ST>(t, s0, (uint32_t)L, 0u, leaf);
    leaf.end_run();
}

/* All runs of [lo, hi) handled by this thread (stride over the grid). */
template <int SMAX, bool FULL, int D, class LF, bool ST = true>
__device__ __forceinline__ void eval_runs(const RkTables& t, uint64_t lo, uint64_t hi, uint32_t tid, uint32_t nth,
                                          LF& leaf) {
    constexpr uint64_t R = cfact(D);
    const uint64_t rb = lo / R, re = (hi + R - 1u) / R;
    for (uint64_t run = rb + tid; run < re; run += nth) eval_run<SMAX, FULL, D, LF, ST>(t, run, leaf);
}

/* n-dependent depth: D = min(n, Depth<SMAX>); n == 1 evaluates the single order. */
template <int SMAX, bool FULL, class LF, bool ST = true>
__device__ __forceinline__ void eval_space(const RkTables& t, uint64_t lo, uint64_t hi, uint32_t tid, uint32_t nth,
                                           LF& leaf) {
    constexpr int DM = Depth<SMAX>::value;
    const uint32_t n = t.g.n;
    if (n >= (uint32_t)DM) eval_runs<SMAX, FULL, DM, LF, ST>(t, lo, hi, tid, nth, leaf);
    else if (DM > 4 && n == 4) eval_runs<SMAX, FULL, (DM > 4 ? 4 : 2)>(t, lo, hi, tid, nth, leaf);
    else if (DM > 3 && n == 3) eval_runs<SMAX, FULL, (DM > 3 ? 3 : 2)>(t, lo, hi, tid, nth, leaf);
    else if (n == 2) eval_runs<SMAX, FULL, 2, LF, ST>(t, lo, hi, tid, nth, leaf);
    else if (tid == 0 && lo < hi) {
        NoRec nr;
        leaf.begin_run(0ull, 1u);
        leaf(0u, eval_index<SMAX, FULL>(t, 0, nr));
        leaf.end_run();
    }
}

__device__ __forceinline__ void load_tables(RkTables& sm, const RkTables* src) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(&sm);
    for (uint32_t i = threadIdx.x; i < sizeof(RkTables) / 4; i += blockDim.x) d[i] = s[i];
    __syncthreads();
}

/* CTAs per SM the register allocator must allow: few (super-)SMs keep the
 * state small, so trade registers for occupancy (measured). */
template <int SMAX>
struct MinBlocks {
#ifdef RK_EVAL_MIN_BLOCKS
    static constexpr int value = RK_EVAL_MIN_BLOCKS;
#else
    static constexpr int value = (SMAX >= 1 && SMAX <= 4) ? 2 : 1;
#endif
};

template <int SMAX, bool FULL, bool EXTRA, bool ST>
__device__ __forceinline__ void eval_body(const RkTables* __restrict__ tab, uint64_t first, uint64_t count,
                                          const uint64_t* cand_dev, uint64_t cand_imm, rk_stats* out, uint64_t* keys,
                                          rk_stats* recs, uint32_t* counter, uint32_t* keys32, uint64_t key_base,
                                          uint32_t* ovf_dev, const rk_stats* hist_range, uint32_t bins,
                                          uint64_t* hist) {
    __shared__ RkTables t;
    extern __shared__ uint32_t shist[];
    if (EXTRA && hist)
        for (uint32_t i = threadIdx.x; i < bins; i += blockDim.x) shist[i] = 0;
    load_tables(t, tab); /* (includes the barrier) */
    const uint64_t cand = cand_dev ? *cand_dev : cand_imm;
    const uint64_t lo = first, hi = first + count;
    TStats ts;
    ts.init();
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    Leaf<EXTRA> leaf{ts, keys, keys32, key_base, 0u, lo, hi, first, cand, (EXTRA && hist) ? shist : nullptr, hist};
    leaf.hcur = 0xFFFFFFFFu;
    leaf.hrun = 0;
    if (EXTRA && hist) leaf.bc.init(hist_range->key_min, hist_range->key_max, bins);
    eval_space<SMAX, FULL, Leaf<EXTRA>, ST>(t, lo, hi, gtid, nth, leaf);
    if constexpr (EXTRA) {
        leaf.flush();
        if (leaf.ovf) atomicOr(ovf_dev, 1u);
        if (hist) {
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < bins; i += blockDim.x)
                if (shist[i]) atomicAdd((unsigned long long*)&hist[i], (unsigned long long)shist[i]);
        }
    }
    const rk_stats r = block_reduce(to_rec(ts));
    commit(r, recs, counter, out);
}

/* the hot path: statistics + optional u64 keys */
template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kThreads, MinBlocks<SMAX>::value)
    rk_eval_kernel(const RkTables* __restrict__ tab, uint64_t first, uint64_t count, const uint64_t* cand_dev,
                   uint64_t cand_imm, rk_stats* out, uint64_t* keys, rk_stats* recs, uint32_t* counter,
                   uint32_t* keys32, uint64_t key_base, uint32_t* ovf_dev, const rk_stats* hist_range,
                   uint32_t bins, uint64_t* hist) {
    if (tab->g.flags & RK_FLAG_STRICT_RR) /* uniform: the strict-capable copy only when the reading is on */
        eval_body<SMAX, FULL, false, true>(tab, first, count, cand_dev, cand_imm, out, keys, recs, counter, nullptr, 0,
                                           nullptr, nullptr, 0, nullptr);
    else
        eval_body<SMAX, FULL, false, false>(tab, first, count, cand_dev, cand_imm, out, keys, recs, counter, nullptr, 0,
                                            nullptr, nullptr, 0, nullptr);
}

/* + compact keys / fused histogram */
template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kThreads, MinBlocks<SMAX>::value)
    rk_eval_x_kernel(const RkTables* __restrict__ tab, uint64_t first, uint64_t count, const uint64_t* cand_dev,
                     uint64_t cand_imm, rk_stats* out, uint64_t* keys, rk_stats* recs, uint32_t* counter,
                     uint32_t* keys32, uint64_t key_base, uint32_t* ovf_dev, const rk_stats* hist_range,
                     uint32_t bins, uint64_t* hist) {
    if (tab->g.flags & RK_FLAG_STRICT_RR)
        eval_body<SMAX, FULL, true, true>(tab, first, count, cand_dev, cand_imm, out, keys, recs, counter, keys32,
                                          key_base, ovf_dev, hist_range, bins, hist);
    else
        eval_body<SMAX, FULL, true, false>(tab, first, count, cand_dev, cand_imm, out, keys, recs, counter, keys32,
                                           key_base, ovf_dev, hist_range, bins, hist);
}

/* C5 batch: blockIdx.y = set, blockIdx.x = chunk of that set's runs.  All sets
 * of one launch share the variant (max super-SM count over the batch). */
template <int SMAX, bool FULL, bool ST>
__device__ __forceinline__ void batch_body(const RkTables* __restrict__ tabs, const uint64_t* __restrict__ cand_keys,
                                           rk_stats* recs) {
    __shared__ RkTables t;
    const uint32_t set = blockIdx.y;
    load_tables(t, tabs + set);
    const uint64_t cand = cand_keys[set];
    const uint32_t n = t.g.n;
    const uint64_t total = t.g.fact[n];
    TStats ts;
    ts.init();
    /* chunk c of the set's index space, aligned to the run size */
    const uint64_t R = cfact(n < (uint32_t)Depth<SMAX>::value ? (int)n : Depth<SMAX>::value);
    const uint64_t runs = (total + R - 1) / R;
    const uint64_t per = (runs + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = min(total, (uint64_t)blockIdx.x * per * R), hi = min(total, lo + per * R);
    Leaf<false> leaf{ts, nullptr, nullptr, 0ull, 0u, lo, hi, 0ull, cand, nullptr};
    eval_space<SMAX, FULL, Leaf<false>, ST>(t, lo, hi, threadIdx.x, blockDim.x, leaf);
    const rk_stats r = block_reduce(to_rec(ts));
    if (threadIdx.x == 0) recs[set * gridDim.x + blockIdx.x] = r;
}

template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kThreads, MinBlocks<SMAX>::value)
    rk_batch_kernel(const RkTables* __restrict__ tabs, const uint64_t* __restrict__ cand_keys, rk_stats* recs) {
    if (tabs[blockIdx.y].g.flags & RK_FLAG_STRICT_RR) batch_body<SMAX, FULL, true>(tabs, cand_keys, recs);
    else batch_body<SMAX, FULL, false>(tabs, cand_keys, recs);
}

/* C5 batch with suffix memoisation: one CTA per set, persistent over the sets.
 * K only accumulates closed rounds (the order's key is
 * the sum of its rounds' keys), so the key of an order is K_prefix + g(state
 * after its (n-5)-prefix with K = 0, remaining kernels): runs whose prefix
 * states agree on the per-SM words, cursor, open round (I, M) and remaining
 * set share one 120-key suffix row.  (A) prefix state of every run; (B) exact
 * dedup in a shared-memory hash table (fingerprint, then full compare against
 * the representative); (C) the rows of the distinct states, each split five
 * ways at its first suffix position; (D) each row's extremes; (E) per run:
 * extremes from its row's, counts against the candidate from its row's range
 * (whole-row scan only where the range straddles the candidate); smallest
 * index on ties, as the direct kernels. */
constexpr int kMemoD = 5;                /* rows of 5! = 120 keys */
constexpr uint32_t kMemoRow = 120;
constexpr uint32_t kMemoRunsMax = 4096;  /* n <= 9: 9!/120 = 3024 runs */
constexpr uint32_t kMemoHT = 4096;       /* slots: fingerprint (44 b) | representative run (20 b) */
constexpr size_t kMemoSmem = kMemoHT * 8 + kMemoRunsMax * 8 + 3 * kMemoRunsMax * 2;

template <int SMAX>
struct MemoRun {
    St<SMAX> s;
    uint32_t L; /* remaining kernels, ascending nibbles */
};

template <int SMAX>
__device__ __forceinline__ uint64_t memo_fp(const St<SMAX>& s, uint32_t L) {
    uint64_t h = ((uint64_t)L << 32 | s.cur) * 0x9E3779B97F4A7C15ull;
    h = (h ^ (h >> 31) ^ s.I) * 0xBF58476D1CE4E5B9ull;
    h = (h ^ (h >> 29) ^ s.M) * 0x94D049BB133111EBull;
#pragma unroll
    for (int i = 0; i < SMAX; i++) h = (h ^ (h >> 32) ^ ((uint64_t)s.fa[i] << 32 | s.fb[i])) * 0x9E3779B97F4A7C15ull;
    return (h ^ (h >> 30)) >> 20;
}

template <int SMAX>
__device__ __forceinline__ bool memo_eq(const MemoRun<SMAX>& a, const MemoRun<SMAX>& b) {
    bool e = a.L == b.L && a.s.cur == b.s.cur && a.s.I == b.s.I && a.s.M == b.s.M;
#pragma unroll
    for (int i = 0; i < SMAX; i++) e = e && a.s.fa[i] == b.s.fa[i] && a.s.fb[i] == b.s.fb[i];
    return e;
}

struct MemoRowStat {
    uint64_t mn, mx;
    uint32_t a; /* offset of the first minimum | offset of the first maximum << 8 */
};

/* stores a part of a row and its extremes (leaves arrive in increasing offset) */
struct RowLeaf {
    uint64_t* row;
    uint64_t mn, mx;
    uint32_t an, ax;
    __device__ __forceinline__ void operator()(uint32_t off, uint64_t K) {
        row[off] = K;
        if (K < mn) { mn = K; an = off; }
        if (K > mx) { mx = K; ax = off; }
    }
    __device__ __forceinline__ void pair(uint32_t off, uint64_t K0, uint64_t K1) {
        (*this)(off, K0);
        (*this)(off + 1u, K1);
    }
};

template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kThreads, MinBlocks<SMAX>::value)
    rk_batch_memo_kernel(const RkTables* __restrict__ tabs, const uint64_t* __restrict__ cand_keys, uint32_t n_sets,
                         uint32_t stride, MemoRun<SMAX>* __restrict__ scratch_runs,
                         uint64_t* __restrict__ scratch_rows, MemoRowStat* __restrict__ scratch_rst,
                         rk_stats* __restrict__ out) {
    __shared__ RkTables t;
    __shared__ uint32_t nd;
    extern __shared__ uint64_t memo_smem[];
    uint64_t* ht = memo_smem;                                   /* [kMemoHT] */
    uint64_t* Kp = ht + kMemoHT;                                /* [kMemoRunsMax] prefix K of each run */
    uint16_t* rep = reinterpret_cast<uint16_t*>(Kp + kMemoRunsMax); /* run -> representative run -> row */
    uint16_t* did = rep + kMemoRunsMax;                         /* representative run -> row */
    uint16_t* repr = did + kMemoRunsMax;                        /* row -> representative run */
    MemoRun<SMAX>* R = scratch_runs + (size_t)blockIdx.x * stride; /* stride = n!/120 runs per set */
    uint64_t* rows = scratch_rows + (size_t)blockIdx.x * stride * kMemoRow;
    MemoRowStat* rst = scratch_rst + (size_t)blockIdx.x * stride * (kMemoD + 1); /* rows' extremes */
    MemoRowStat* pst = rst + stride;                                            /* parts' extremes */
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    NoRec nr;
    for (uint32_t set = blockIdx.x; set < n_sets; set += gridDim.x) {
        __syncthreads(); /* the previous set is done with the shared arrays */
        for (uint32_t i = tid; i < kMemoHT; i += nth) ht[i] = ~0ull;
        if (tid == 0) nd = 0;
        load_tables(t, tabs + set); /* (includes the barrier) */
        const RkGTab& g = t.g;
        const uint32_t n = g.n;
        const uint32_t runs = (uint32_t)(g.fact[n] / kMemoRow);
        /* (A) the (n-5)-prefix of run r = indices [120 r, 120 r + 120) */
        for (uint32_t r = tid; r < runs; r += nth) {
            St<SMAX> s;
            st_fresh<SMAX, FULL>(s, g);
            uint64_t L = identity_list(n);
            uint32_t rem = r * kMemoRow;
            for (uint32_t j = 0; j + kMemoD < n; j++) {
                const uint32_t f = (uint32_t)g.fact[n - 1 - j];
                const uint32_t d = rem / f;
                rem -= d * f;
                const uint32_t k = take_nibble(L, d);
                place<SMAX, FULL>(s, s, t.k[k], k, g, nr);
            }
            Kp[r] = s.K;
            R[r].s = s;
            R[r].L = (uint32_t)L;
        }
        __syncthreads();
        /* (B) exact dedup: the CAS winner of a fingerprint represents every run
         * whose full state equals its own; a fingerprint collision probes on */
        for (uint32_t r = tid; r < runs; r += nth) {
            const MemoRun<SMAX> me = R[r];
            const uint64_t fp = memo_fp<SMAX>(me.s, me.L);
            uint32_t slot = (uint32_t)fp & (kMemoHT - 1u);
            uint32_t q;
            for (;;) {
                uint64_t v = ht[slot];
                if (v == ~0ull) {
                    v = atomicCAS((unsigned long long*)&ht[slot], ~0ull, (fp << 20) | r);
                    if (v == ~0ull) {
                        q = r;
                        break;
                    }
                }
                if ((v >> 20) == fp) {
                    q = (uint32_t)v & 0xFFFFFu;
                    if (memo_eq<SMAX>(me, R[q])) break;
                }
                slot = (slot + 1u) & (kMemoHT - 1u);
            }
            rep[r] = (uint16_t)q;
        }
        __syncthreads();
        for (uint32_t r = tid; r < runs; r += nth)
            if (rep[r] == r) {
                const uint32_t d = atomicAdd(&nd, 1u);
                did[r] = (uint16_t)d;
                repr[d] = (uint16_t)r;
            }
        __syncthreads();
        for (uint32_t r = tid; r < runs; r += nth) rep[r] = did[rep[r]];
        const uint32_t ndist = nd;
        /* (C) row d, part a: the a-th remaining kernel first, then its 4! orders */
        for (uint32_t it = tid; it < ndist * kMemoD; it += nth) {
            const uint32_t d = it / kMemoD, a = it - d * kMemoD;
            const MemoRun<SMAX>& m = R[repr[d]];
            St<SMAX> s = m.s;
            s.K = 0;
            const uint32_t sh = 4u * a, ka = (m.L >> sh) & 15u;
            const uint32_t rest = (m.L & ((1u << sh) - 1u)) | ((m.L >> (sh + 4u)) << sh);
            St<SMAX> s1;
            place<SMAX, FULL>(s, s1, t.k[ka], ka, g, nr);
            RowLeaf lf{rows + (size_t)d * kMemoRow, ~0ull, 0ull, 0u, 0u};
            dfs<SMAX, FULL, kMemoD - 1>(t, s1, rest, a * cfact(kMemoD - 1), lf);
            pst[it] = MemoRowStat{lf.mn, lf.mx, lf.an | lf.ax << 8};
        }
        __syncthreads();
        /* (D) row extremes from its five parts (in offset order: smallest offset on ties) */
        for (uint32_t d = tid; d < ndist; d += nth) {
            MemoRowStat r = pst[d * kMemoD];
#pragma unroll
            for (uint32_t a = 1; a < (uint32_t)kMemoD; a++) {
                const MemoRowStat p = pst[d * kMemoD + a];
                if (p.mn < r.mn) r.a = (r.a & ~0xFFu) | (p.a & 0xFFu), r.mn = p.mn;
                if (p.mx > r.mx) r.a = (r.a & 0xFFu) | (p.a & ~0xFFu), r.mx = p.mx;
            }
            rst[d] = r;
        }
        __syncthreads();
        const uint32_t lane = tid & 31u;
        /* (E) orders 120 run + j, keys Kp[run] + row[rep[run]][j]: extremes from
         * the row's, counts below / equal to the candidate from the row's range;
         * a row that straddles the candidate is counted by the whole warp */
        const uint64_t cand = cand_keys[set];
        TStats ts;
        ts.init();
        for (uint32_t r0 = 0; r0 < runs; r0 += nth) {
            const uint32_t r = r0 + tid;
            const bool live = r < runs;
            uint32_t d = 0;
            uint64_t thr = 0;
            bool straddle = false;
            if (live) {
                d = rep[r];
                const uint64_t K0 = Kp[r];
                const MemoRowStat rs = rst[d];
                const uint64_t base = (uint64_t)r * kMemoRow;
                if (K0 + rs.mn < ts.kmin) { ts.kmin = K0 + rs.mn; ts.amin = base + (rs.a & 0xFFu); }
                if (K0 + rs.mx > ts.kmax) { ts.kmax = K0 + rs.mx; ts.amax = base + (rs.a >> 8); }
                ts.cnt += kMemoRow;
                if (cand >= K0) {
                    thr = cand - K0; /* K < cand  <=>  row value < thr */
                    if (thr > rs.mx) ts.nlt += kMemoRow;
                    else straddle = thr >= rs.mn;
                }
            }
            uint32_t mask = __ballot_sync(~0u, straddle);
            while (mask) {
                const uint32_t src = __ffs(mask) - 1u;
                mask &= mask - 1u;
                const uint64_t th = __shfl_sync(~0u, thr, src);
                const uint64_t* row = rows + (size_t)__shfl_sync(~0u, d, src) * kMemoRow;
                uint32_t lt = 0, eq = 0;
#pragma unroll
                for (uint32_t j0 = 0; j0 < 128u; j0 += 32u) {
                    const uint32_t j = j0 + lane;
                    const uint64_t v = j < kMemoRow ? row[j] : ~0ull;
                    lt += __popc(__ballot_sync(~0u, j < kMemoRow && v < th));
                    eq += __popc(__ballot_sync(~0u, j < kMemoRow && v == th));
                }
                if (lane == src) {
                    ts.nlt += lt;
                    ts.neq += eq;
                }
            }
        }
        const rk_stats rs = block_reduce(to_rec(ts));
        if (tid == 0) out[set] = rs;
    }
}

/* merge groups of `per` consecutive records: one warp per group */
__global__ void rk_merge_groups_kernel(const rk_stats* __restrict__ in, uint32_t groups, uint32_t per,
                                       rk_stats* __restrict__ out) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= groups) return; /* whole warps exit together */
    rk_stats v{};
    v.evaluated = 0;
    for (uint32_t i = lane; i < per; i += 32) merge_into(v, in[(size_t)w * per + i]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        rk_stats o = shfl_rec(v, off);
        merge_into(v, o);
    }
    if (lane == 0) out[w] = v;
}

/* keys of explicit indices; per_set: item i uses tabs[i], else tabs[0] */
template <int SMAX, bool FULL>
__global__ void rk_keys_of_kernel(const RkTables* __restrict__ tabs, const uint64_t* __restrict__ idx, uint32_t m,
                                  int per_set, uint64_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    NoRec nr;
    out[i] = eval_index<SMAX, FULL>(tabs[per_set ? i : 0], idx[i], nr);
}

template <int SMAX, bool FULL>
__global__ void rk_key_of_index_kernel(const RkTables* __restrict__ tab, uint64_t index, uint64_t* __restrict__ out) {
    __shared__ RkTables t;
    load_tables(t, tab);
    if (threadIdx.x == 0) {
        NoRec nr;
        *out = eval_index<SMAX, FULL>(t, index, nr);
    }
}

template <int SMAX, bool FULL>
__global__ void rk_simulate_kernel(const RkTables* __restrict__ tab, const int32_t* __restrict__ order,
                                   uint32_t* rounds, uint32_t max_rounds, uint32_t* n_rounds, uint64_t* key) {
    const RkTables& t = *tab;
    const uint32_t n = t.g.n;
    for (uint32_t i = 0; i < max_rounds * n; i++) rounds[i] = 0;
    Rec rec{rounds, max_rounds, n, 0, t.g.blkscale};
    St<SMAX> s;
    st_fresh<SMAX, FULL>(s, t.g);
    for (uint32_t j = 0; j + 1 < n; j++) place<SMAX, FULL>(s, s, t.k[order[j]], (uint32_t)order[j], t.g, rec);
    *key = finish<SMAX>(s, t.k[order[n - 1]], (uint32_t)order[n - 1], t.g, rec);
    *n_rounds = rec.r;
}

/* ---- Model-reading policies -------------
 * RK_FLAG_STRICT_RR (L4 read literally): a block is offered to the
 * SM under the cursor only.  RK_FLAG_SKIP_AHEAD (the L5 alternative SPEC:262
 * rejects): a kernel whose next block fits nowhere waits for the next round
 * while the later kernels keep filling this one.  Under skip-ahead the state
 * after a prefix carries the pending blocks of earlier kernels, so there is no
 * prefix sharing or memoisation: one order per thread, the whole round loop,
 * on the register state (S' <= 32 super-SMs; the symmetry reduction holds:
 * every placement count stays a multiple of g). */
/* SM-state width: the smallest of {2, 8, 32} >= S' (runtime S inside) */

/* Blocks of kernel k the policy can place from cursor cur before one fails:
 * first fit (L4) takes up to F = sum c_s; strict round robin sends block b to
 * SM (cur + b) mod S, which fails first at b = min_s ((s - cur) mod S + c_s S). */
template <int kPolSmax>
__device__ __forceinline__ uint32_t pol_avail(const St<kPolSmax>& s, const RkKTab& k, const RkGTab& g, bool strict,
                                              uint32_t cur, uint32_t (&c)[kPolSmax]) {
    const CapK ck = capk(k);
    const uint32_t S = g.S;
    uint32_t F = 0, m = 0xFFFFFFFFu;
#pragma unroll
    for (int i = 0; i < kPolSmax; i++) {
        const bool live = (uint32_t)i < S;
        c[i] = live ? cap1(s.fa[i], s.fb[i], ck) : 0u;
        F += c[i];
        const uint32_t d = (uint32_t)i >= cur ? (uint32_t)i - cur : (uint32_t)i + S - cur;
        if (live) m = min(m, d + c[i] * S);
    }
    return strict ? m : F;
}

/* Place p (1 <= p <= pol_avail) blocks of kernel k from cursor cur; returns
 * the new cursor.  First fit is the water-fill of place_core (the SM of the
 * p-th block + 1); strict round robin gives SM s the blocks b < p with
 * b = (s - cur) mod S (mod S), and the cursor moves by p. */
template <int kPolSmax>
__device__ __forceinline__ uint32_t pol_place(St<kPolSmax>& s, uint32_t p, const uint32_t (&c)[kPolSmax],
                                              const RkKTab& k, const RkGTab& g, bool strict, uint32_t cur) {
    const uint32_t S = g.S;
    if (strict) {
#pragma unroll
        for (int i = 0; i < kPolSmax; i++) {
            if ((uint32_t)i >= S) continue;
            const uint32_t d = (uint32_t)i >= cur ? (uint32_t)i - cur : (uint32_t)i + S - cur;
            const uint32_t x = d < p ? (p - d - 1u) / S + 1u : 0u;
            s.fa[i] -= x * k.dA;
            s.fb[i] -= x * k.dB;
        }
        return (cur + p) % S;
    }
    uint32_t bfa[kPolSmax], bfb[kPolSmax];
#pragma unroll
    for (int i = 0; i < kPolSmax; i++) {
        bfa[i] = s.fa[i];
        bfb[i] = s.fb[i];
    }
    StoreUpd<kPolSmax> u{s};
    return water_fill<kPolSmax, false>(p, c, bfa, bfb, cur, k, g, u);
}

template <int kPolSmax>
__device__ __forceinline__ void pol_fresh(St<kPolSmax>& s, const RkGTab& g) {
#pragma unroll
    for (int i = 0; i < kPolSmax; i++) {
        s.fa[i] = (uint32_t)i < g.S ? g.freshA : 0u;
        s.fb[i] = (uint32_t)i < g.S ? g.freshB : 0u;
    }
}

/* The last rounds of one kernel alone, from a fresh round: both readings put
 * SC = S*C blocks in a fresh round (strict: min_s (s + C S) = C S at SM 0), so
 * the rounds are full ones and a remainder (as finish_key). */
template <class R>
__device__ __forceinline__ uint64_t pol_alone(uint32_t rem, const RkKTab& k, uint32_t kid, const RkGTab& g, R& rec) {
    const uint32_t nfull = full_rounds(rem - 1u, k);
    rec.full(kid, nfull, k.SC);
    rem -= nfull * k.SC;
    rec.add(kid, rem);
    rec.close();
    return (uint64_t)nfull * k.fullkey + round_key((uint64_t)rem * k.cA, (uint64_t)rem * k.cM, g.num, g.den);
}

/* Exact key of one launch order (ord[0..n-1]) under the policy flags. */
template <int kPolSmax, class R>
__device__ uint64_t pol_key(const RkTables& t, const uint8_t (&ord)[RK_MAX_N], R& rec) {
    const RkGTab& g = t.g;
    const uint32_t n = g.n;
    const bool strict = (g.flags & RK_FLAG_STRICT_RR) != 0, perk = (g.flags & RK_FLAG_CURSOR_PER_KERNEL) != 0;
    St<kPolSmax> s;
    uint32_t c[kPolSmax];
    uint64_t K = 0, I = 0, M = 0;
    uint32_t cur = 0;
    pol_fresh(s, g);
    if (!(g.flags & RK_FLAG_SKIP_AHEAD)) {
        /* in-order dispatch (L5): a block that cannot be placed closes the round */
        for (uint32_t j = 0; j < n; j++) {
            const uint32_t kid = ord[j];
            const RkKTab& k = t.k[kid];
            uint32_t rem = k.T;
            if (perk) cur = 0;
            const uint32_t p = min(rem, pol_avail(s, k, g, strict, cur, c));
            if (p) {
                cur = pol_place(s, p, c, k, g, strict, cur);
                I += (uint64_t)p * k.cA;
                M += (uint64_t)p * k.cM;
                rec.add(kid, p);
                rem -= p;
            }
            if (rem) { /* close the round; full rounds of k alone; the rest opens a fresh round */
                K += round_key(I, M, g.num, g.den);
                rec.close();
                const uint32_t nfull = full_rounds(rem - 1u, k);
                rec.full(kid, nfull, k.SC);
                K += (uint64_t)nfull * k.fullkey;
                rem -= nfull * k.SC;
                pol_fresh(s, g);
                pol_avail(s, k, g, strict, 0u, c); /* fresh capacities: 1 <= rem <= SC */
                cur = pol_place(s, rem, c, k, g, strict, 0u);
                I = (uint64_t)rem * k.cA;
                M = (uint64_t)rem * k.cM;
                rec.add(kid, rem);
            }
        }
        rec.close();
        return K + round_key(I, M, g.num, g.den);
    }
    /* skip-ahead: every round offers each kernel with pending blocks, in launch order */
    uint32_t pend[RK_MAX_N];
    uint32_t npend = n;
    for (uint32_t j = 0; j < n; j++) pend[j] = t.k[ord[j]].T;
    while (npend) {
        if (npend == 1) {
            for (uint32_t j = 0; j < n; j++)
                if (pend[j]) return K + pol_alone(pend[j], t.k[ord[j]], ord[j], g, rec);
        }
        pol_fresh(s, g);
        cur = 0;
        I = M = 0;
        for (uint32_t j = 0; j < n; j++) {
            if (!pend[j]) continue;
            const uint32_t kid = ord[j];
            const RkKTab& k = t.k[kid];
            if (perk) cur = 0;
            const uint32_t p = min(pend[j], pol_avail(s, k, g, strict, cur, c));
            if (!p) continue; /* waits for the next round */
            cur = pol_place(s, p, c, k, g, strict, cur);
            I += (uint64_t)p * k.cA;
            M += (uint64_t)p * k.cM;
            rec.add(kid, p);
            pend[j] -= p;
            if (!pend[j]) npend--;
        }
        K += round_key(I, M, g.num, g.den);
        rec.close();
    }
    return K;
}

/* lexicographic unrank into kernel ids (O2's digits) */
__device__ __forceinline__ void pol_unrank(const RkGTab& g, uint64_t idx, uint8_t (&ord)[RK_MAX_N]) {
    uint64_t L = identity_list(g.n);
    for (uint32_t j = 0; j < g.n; j++) {
        const uint64_t f = g.fact[g.n - 1 - j];
        const uint32_t d = (uint32_t)(idx / f);
        idx -= (uint64_t)d * f;
        ord[j] = (uint8_t)take_nibble(L, d);
    }
}

/* stats (+ optional keys) of [first, first+count): grid-stride over indices */
template <int kPolSmax>
__global__ void __launch_bounds__(kThreads) rk_policy_eval_kernel(const RkTables* __restrict__ tab, uint64_t first,
                                                                   uint64_t count, const uint64_t* cand_dev,
                                                                   uint64_t cand_imm, rk_stats* out, uint64_t* keys,
                                                                   rk_stats* recs, uint32_t* counter) {
    __shared__ RkTables t;
    load_tables(t, tab);
    const uint64_t cand = cand_dev ? *cand_dev : cand_imm;
    TStats ts;
    ts.init();
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    NoRec nr;
    uint8_t ord[RK_MAX_N];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += nth) {
        const uint64_t idx = first + i;
        pol_unrank(t.g, idx, ord);
        const uint64_t key = pol_key<kPolSmax>(t, ord, nr);
        if (keys) keys[i] = key;
        if (key < ts.kmin) { ts.kmin = key; ts.amin = idx; } /* increasing indices: strict keeps the smallest (L12) */
        if (key > ts.kmax || ts.cnt == 0) { ts.kmax = key; ts.amax = idx; }
        ts.nlt += key < cand ? 1u : 0u;
        ts.neq += key == cand ? 1u : 0u;
        ts.cnt++;
    }
    const rk_stats r = block_reduce(to_rec(ts));
    commit(r, recs, counter, out);
}

/* C5 batch under a policy: blockIdx.y = set, blockIdx.x = chunk of its indices */
template <int kPolSmax>
__global__ void __launch_bounds__(kThreads) rk_policy_batch_kernel(const RkTables* __restrict__ tabs,
                                                                    const uint64_t* __restrict__ cand_keys,
                                                                    rk_stats* recs) {
    __shared__ RkTables t;
    const uint32_t set = blockIdx.y;
    load_tables(t, tabs + set);
    const uint64_t cand = cand_keys[set], total = t.g.fact[t.g.n];
    const uint64_t per = (total + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = min(total, (uint64_t)blockIdx.x * per), hi = min(total, lo + per);
    TStats ts;
    ts.init();
    NoRec nr;
    uint8_t ord[RK_MAX_N];
    for (uint64_t idx = lo + threadIdx.x; idx < hi; idx += blockDim.x) {
        pol_unrank(t.g, idx, ord);
        const uint64_t key = pol_key<kPolSmax>(t, ord, nr);
        if (key < ts.kmin) { ts.kmin = key; ts.amin = idx; }
        if (key > ts.kmax || ts.cnt == 0) { ts.kmax = key; ts.amax = idx; }
        ts.nlt += key < cand ? 1u : 0u;
        ts.neq += key == cand ? 1u : 0u;
        ts.cnt++;
    }
    const rk_stats r = block_reduce(to_rec(ts));
    if (threadIdx.x == 0) recs[set * gridDim.x + blockIdx.x] = r;
}

/* keys of explicit indices; per_set: item i uses tabs[i], else tabs[0] */
template <int kPolSmax>
__global__ void rk_policy_keys_of_kernel(const RkTables* __restrict__ tabs, const uint64_t* __restrict__ idx,
                                         uint32_t m, int per_set, uint64_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const RkTables& t = tabs[per_set ? i : 0];
    NoRec nr;
    uint8_t ord[RK_MAX_N];
    pol_unrank(t.g, idx[i], ord);
    out[i] = pol_key<kPolSmax>(t, ord, nr);
}

template <int kPolSmax>
__global__ void rk_policy_key_of_index_kernel(const RkTables* __restrict__ tab, uint64_t index,
                                              uint64_t* __restrict__ out) {
    if (threadIdx.x) return;
    NoRec nr;
    uint8_t ord[RK_MAX_N];
    pol_unrank(tab->g, index, ord);
    *out = pol_key<kPolSmax>(*tab, ord, nr);
}

/* one order -> round partition (1 thread) */
template <int kPolSmax>
__global__ void rk_policy_simulate_kernel(const RkTables* __restrict__ tab, const int32_t* __restrict__ order,
                                          uint32_t* rounds, uint32_t max_rounds, uint32_t* n_rounds, uint64_t* key) {
    const RkTables& t = *tab;
    const uint32_t n = t.g.n;
    for (uint32_t i = 0; i < max_rounds * n; i++) rounds[i] = 0;
    Rec rec{rounds, max_rounds, n, 0, t.g.blkscale};
    uint8_t ord[RK_MAX_N];
    for (uint32_t j = 0; j < n; j++) ord[j] = (uint8_t)order[j];
    *key = pol_key<kPolSmax>(t, ord, rec);
    *n_rounds = rec.r;
}

/* Fig. 1 histogram: exact integer bins over [kmin, kmax]:
 * bin = min(B-1, floor((K-kmin)*B / (kmax-kmin))).  HBM-bound pass: each
 * thread reads 8 consecutive keys (two 32-B vector loads; a warp reads 2 KB
 * contiguous), run-length merges equal bins (lexicographic neighbours have
 * close keys) before one shared-memory atomic per run; u64 global atomics at
 * the end (integer adds: order-free, bit-exact). */
/* RANGE = false: Fig. 1 bins over [kmin, kmax] (last bin closed).
 * RANGE = true: order-statistic refinement — `bins` half-open bins over
 * [kmin_imm, kmin_imm + kmax_imm) (kmax_imm = span), keys outside ignored. */
template <bool RANGE, class KT>
__global__ void __launch_bounds__(256) rk_hist_kernel(const KT* __restrict__ keys, uint64_t count,
                                                      uint64_t kmin_imm, uint64_t kmax_imm,
                                                      const rk_stats* __restrict__ range, uint32_t bins,
                                                      uint64_t* __restrict__ hist, uint64_t key_base) {
    extern __shared__ uint32_t sh[];
    const bool smem_bins = bins <= kSmemBins; /* else accumulate straight into global u64 bins */
    BinCalc bc;
    if (RANGE) bc.init_span(kmin_imm, kmax_imm, bins);
    else bc.init(range ? range->key_min : kmin_imm, range ? range->key_max : kmax_imm, bins);
    if (smem_bins)
        for (uint32_t i = threadIdx.x; i < bins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    uint32_t cur = 0xFFFFFFFFu, run = 0;
    auto flush = [&]() {
        if (!run) return;
        if (smem_bins) sh_bin_add(sh, hist, cur, run);
        else atomicAdd((unsigned long long*)&hist[cur], (unsigned long long)run);
    };
    auto put = [&](uint32_t b) {
        if (RANGE && b == 0xFFFFFFFFu) return; /* outside the refinement range */
        if (b == cur && run < (1u << 20)) {
            run++;
        } else {
            flush();
            cur = b;
            run = 1;
        }
    };
    auto binof = [&](uint64_t Kraw) -> uint32_t {
        const uint64_t K = sizeof(KT) == 4 ? key_base + Kraw : Kraw; /* u32 keys are offsets */
        if (RANGE && K - bc.kmin >= bc.D) return 0xFFFFFFFFu;
        return bc(K);
    };
    const uint64_t nchunks = count / 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(keys) & 15) == 0;
    if (aligned) {
        if constexpr (sizeof(KT) == 8) {
            /* software-pipelined: the next chunk's 64 B are in flight while this one is binned */
            const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys);
            uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
            ulonglong2 a, b, d, e;
            if (c < nchunks) {
                a = __ldcs(k2 + 4 * c); b = __ldcs(k2 + 4 * c + 1);
                d = __ldcs(k2 + 4 * c + 2); e = __ldcs(k2 + 4 * c + 3);
            }
            for (; c < nchunks; c += stride) {
                const ulonglong2 a0 = a, b0 = b, d0 = d, e0 = e;
                const uint64_t cn = c + stride;
                if (cn < nchunks) {
                    a = __ldcs(k2 + 4 * cn); b = __ldcs(k2 + 4 * cn + 1);
                    d = __ldcs(k2 + 4 * cn + 2); e = __ldcs(k2 + 4 * cn + 3);
                }
                put(binof(a0.x)); put(binof(a0.y)); put(binof(b0.x)); put(binof(b0.y));
                put(binof(d0.x)); put(binof(d0.y)); put(binof(e0.x)); put(binof(e0.y));
            }
        } else {
            const uint4* k4 = reinterpret_cast<const uint4*>(keys);
            for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += stride) {
                const uint4 a = __ldcs(k4 + 2 * c), b = __ldcs(k4 + 2 * c + 1);
                put(binof(a.x)); put(binof(a.y)); put(binof(a.z)); put(binof(a.w));
                put(binof(b.x)); put(binof(b.y)); put(binof(b.z)); put(binof(b.w));
            }
        }
    }
    for (uint64_t i = (aligned ? nchunks * 8 : 0) + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += stride)
        put(binof(keys[i]));
    flush();
    if (!smem_bins) return;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < bins; i += blockDim.x)
        if (sh[i]) atomicAdd((unsigned long long*)&hist[i], (unsigned long long)sh[i]);
}

/* ==================== Algorithm 1 on the device ====================
 * One thread per kernel set: the paper's greedy launch-order algorithm
 * with the readings of DESIGN.md §3, in the same fixed double
 * operation order as the host implementation (every operation an explicitly
 * rounded IEEE op, no contraction), so orders are bit-identical. */
struct DProf {
    uint64_t shm, regs, warps, blocks;
    double inst, ratio;
};

__device__ __forceinline__ DProf d_combine(const DProf& a, const DProf& b) {
    DProf c;
    c.shm = a.shm + b.shm;
    c.regs = a.regs + b.regs;
    c.warps = a.warps + b.warps;
    c.blocks = a.blocks + b.blocks;
    c.inst = __dadd_rn(a.inst, b.inst);
    c.ratio = __ddiv_rn(__dadd_rn(a.inst, b.inst), __dadd_rn(__ddiv_rn(a.inst, a.ratio), __ddiv_rn(b.inst, b.ratio)));
    return c;
}
__device__ __forceinline__ bool d_fits(const rk_gpu_params& p, const DProf& a, const DProf& b) {
    return a.shm + b.shm <= p.shm_bytes_per_sm && a.regs + b.regs <= p.regs_per_sm &&
           a.warps + b.warps <= p.max_warps_per_sm && a.blocks + b.blocks <= p.max_blocks_per_sm;
}
__device__ __forceinline__ double d_slack(uint64_t cap, uint64_t x, uint64_t y) {
    const double v = __ddiv_rn((double)((int64_t)cap - (int64_t)x - (int64_t)y), (double)cap);
    return v > 0.0 ? v : 0.0;
}
__device__ __forceinline__ double d_score(const rk_gpu_params& p, double RB, const DProf& a, const DProf& b) {
    double s = 0.0;
    s = __dadd_rn(s, d_slack(p.shm_bytes_per_sm, a.shm, b.shm));
    s = __dadd_rn(s, d_slack(p.regs_per_sm, a.regs, b.regs));
    s = __dadd_rn(s, d_slack(p.max_warps_per_sm, a.warps, b.warps));
    if ((a.ratio <= RB && RB <= b.ratio) || (b.ratio <= RB && RB <= a.ratio)) {
        const double rc =
            __ddiv_rn(__dadd_rn(a.inst, b.inst), __dadd_rn(__ddiv_rn(a.inst, a.ratio), __ddiv_rn(b.inst, b.ratio)));
        const double bonus = __dsub_rn(1.0, __ddiv_rn(fabs(__dsub_rn(rc, RB)), RB));
        s = __dadd_rn(s, bonus > 0.0 ? bonus : 0.0);
    }
    return s;
}

__global__ void rk_heuristic_kernel(const rk_kernel* __restrict__ sets, uint32_t n, uint32_t n_sets,
                                    rk_gpu_params p, int32_t* __restrict__ orders, uint64_t* __restrict__ index) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_sets) return;
    const rk_kernel* ks = sets + (size_t)q * n;
    const double RB = __ddiv_rn((double)p.rb_num, (double)p.rb_den);
    DProf f[RK_MAX_N];
    for (uint32_t i = 0; i < n; i++) {
        const uint64_t per_sm = (ks[i].grid_blocks + p.n_sm - 1) / p.n_sm; /* ceil(N_tblk/N_SM) */
        f[i].shm = (uint64_t)ks[i].shm_bytes_per_block * per_sm;
        f[i].regs = (uint64_t)ks[i].regs_per_thread * ks[i].threads_per_block * per_sm;
        f[i].warps = (uint64_t)((ks[i].threads_per_block + 31u) / 32u) * per_sm;
        f[i].blocks = per_sm;
        f[i].inst = __dmul_rn((double)ks[i].grid_blocks, (double)ks[i].inst_per_block);
        f[i].ratio = __ddiv_rn((double)ks[i].inst_per_block, (double)ks[i].mem_per_block);
    }
    uint32_t used = 0, pos = 0;
    int32_t out[RK_MAX_N];
    while (pos < n) {
        if (pos + 1 == n) { /* lone kernel: singleton round */
            for (uint32_t i = 0; i < n; i++)
                if (!(used >> i & 1u)) out[pos++] = (int32_t)i;
            break;
        }
        int ba = -1, bb = -1;
        double bs = 0.0;
        for (uint32_t a = 0; a < n; a++) {
            if (used >> a & 1u) continue;
            for (uint32_t b = a + 1; b < n; b++) {
                if ((used >> b & 1u) || !d_fits(p, f[a], f[b])) continue;
                const double sc = d_score(p, RB, f[a], f[b]);
                if (ba < 0 || sc > bs) { ba = (int)a; bb = (int)b; bs = sc; }
            }
        }
        if (ba < 0) { /* no feasible pair: singletons by decreasing shm, index order on ties */
            while (pos < n) {
                int best = -1;
                for (uint32_t i = 0; i < n; i++)
                    if (!(used >> i & 1u) && (best < 0 || f[i].shm > f[best].shm)) best = (int)i;
                used |= 1u << best;
                out[pos++] = best;
            }
            break;
        }
        int32_t rd[RK_MAX_N];
        uint32_t m = 2;
        if (f[bb].shm > f[ba].shm) { rd[0] = bb; rd[1] = ba; }
        else { rd[0] = ba; rd[1] = bb; }
        used |= (1u << ba) | (1u << bb);
        DProf comb = d_combine(f[ba], f[bb]);
        for (;;) {
            int bc = -1;
            double cs = 0.0;
            for (uint32_t x = 0; x < n; x++) {
                if ((used >> x & 1u) || !d_fits(p, comb, f[x])) continue;
                const double sc = d_score(p, RB, comb, f[x]);
                if (bc < 0 || sc > cs) { bc = (int)x; cs = sc; }
            }
            if (bc < 0) break;
            uint32_t at = 0; /* stable decreasing-shm insertion (reading L17) */
            while (at < m && f[rd[at]].shm >= f[bc].shm) at++;
            for (uint32_t j = m; j > at; j--) rd[j] = rd[j - 1];
            rd[at] = bc;
            m++;
            comb = d_combine(comb, f[bc]);
            used |= 1u << bc;
        }
        for (uint32_t j = 0; j < m; j++) out[pos++] = rd[j];
    }
    /* lexicographic rank of the order (factorial number system) */
    uint64_t idx = 0;
    uint32_t seen = 0;
    for (uint32_t j = 0; j < n; j++) {
        const uint32_t x = (uint32_t)out[j];
        idx = idx * (n - j) + (uint32_t)__popc(~seen & ((1u << x) - 1u));
        seen |= 1u << x;
        if (orders) orders[(size_t)q * n + j] = out[j];
    }
    index[q] = idx;
}

/* ============ Branch-and-bound exact optimum (n >= 13) ============
 * A lower bound on every completion of a node (state s after a prefix, remaining
 * set R): the open round and all later rounds together cost
 * sum_r max(den I_r, num M_r) >= max(sum_r den I_r, sum_r num M_r) (SPEC:255 round
 * key is a max of the two sums), and those sums are fixed by R, so
 *   LB = K + max(dI + sum_{k in R} T_k dA_k, nM + sum_{k in R} T_k nM_k).
 * The pruning is STRICT (LB > best): every leaf whose key equals the final minimum
 * is visited, so one pass yields the minimum AND its smallest index (the argmin
 * of the full sweep, SPEC:300 ties -> smallest index).  Work units are the
 * n!/(n-P)! prefixes of depth P, handed out by an atomic counter (dynamic
 * balance: subtree sizes after pruning vary by orders of magnitude); below a unit
 * an explicit-stack DFS in lexicographic order, so leaf indices are ascending
 * inside a unit. */
struct BnbGlobal {             /* device scratch; host zeroes it (best = seed) */
    unsigned long long best;   /* running minimum key (seeded with an order's key) */
    unsigned long long nodes;  /* placements performed */
    unsigned int next_unit;
    unsigned int done;         /* CTAs finished (last one merges) */
    unsigned long long key, index; /* result */
};

__device__ __forceinline__ uint32_t nth_set_bit(uint32_t m, uint32_t r) { /* 0-based r-th set bit of m */
    for (uint32_t q = 0; q < r; q++) m &= m - 1u;
    return (uint32_t)__ffs(m) - 1u;
}

__device__ __forceinline__ bool lex_less(uint64_t ka, uint64_t ia, uint64_t kb, uint64_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

constexpr int kBnbThreads = 128;

template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kBnbThreads) rk_bnb_kernel(const RkTables* __restrict__ tab, uint32_t P,
                                                            uint64_t n_units, BnbGlobal* gb,
                                                            unsigned long long* __restrict__ recs) {
    __shared__ RkTables t;
    __shared__ uint64_t totA[RK_MAX_N], totM[RK_MAX_N];
    __shared__ uint64_t wk[kBnbThreads / 32], wi[kBnbThreads / 32];
    __shared__ bool last;
    load_tables(t, tab);
    const RkGTab& g = t.g;
    const uint32_t n = g.n;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        totA[i] = (uint64_t)t.k[i].T * t.k[i].cA;
        totM[i] = (uint64_t)t.k[i].T * t.k[i].cM;
    }
    __syncthreads();
    uint64_t sumA = 0, sumM = 0;
    for (uint32_t i = 0; i < n; i++) {
        sumA += totA[i];
        sumM += totM[i];
    }
    uint64_t span = 1; /* (n-P)! leaves per unit */
    for (uint32_t i = 2; i <= n - P; i++) span *= i;
    const uint32_t full = (1u << n) - 1u;

    NoRec nr;
    St<SMAX> st[RK_MAX_N];
    uint32_t rmask[RK_MAX_N], child[RK_MAX_N];
    uint64_t ra[RK_MAX_N], rm[RK_MAX_N], ioff[RK_MAX_N];
    uint64_t nodes = 0, my_key = ~0ull, my_idx = ~0ull;
    uint64_t best = *(volatile unsigned long long*)&gb->best;
    for (;;) {
        const uint64_t u = atomicAdd(&gb->next_unit, 1u);
        if (u >= n_units) break;
        best = *(volatile unsigned long long*)&gb->best;
        /* the P-prefix of unit u: mixed radix (n, n-1, ..., n-P+1), lexicographic */
        uint64_t rem = u;
        uint32_t dig[RK_MAX_N];
        for (int j = (int)P - 1; j >= 0; j--) {
            const uint32_t base = n - (uint32_t)j;
            dig[j] = (uint32_t)(rem % base);
            rem /= base;
        }
        st_fresh<SMAX, FULL>(st[0], g);
        uint32_t mask = full;
        uint64_t sa = sumA, sm = sumM;
        bool pruned = false;
        for (uint32_t j = 0; j < P && !pruned; j++) {
            const uint32_t k = nth_set_bit(mask, dig[j]);
            mask &= ~(1u << k);
            sa -= totA[k];
            sm -= totM[k];
            place<SMAX, FULL>(st[0], st[0], t.k[k], k, g, nr);
            nodes++;
            const uint64_t x = st[0].I + sa, y = st[0].M + sm;
            pruned = st[0].K + (x >= y ? x : y) > best;
        }
        if (pruned) continue;
        int l = 0;
        rmask[0] = mask;
        child[0] = 0;
        ra[0] = sa;
        rm[0] = sm;
        ioff[0] = u * span;
        while (l >= 0) {
            const uint32_t left = (uint32_t)__popc(rmask[l]);
            if (child[l] >= left) { l--; continue; }
            const uint32_t c = child[l]++;
            const uint32_t k = nth_set_bit(rmask[l], c);
            uint64_t sub = 1; /* (left-1)! leaves below each child */
            for (uint32_t i = 2; i < left; i++) sub *= i;
            const uint64_t idx = ioff[l] + (uint64_t)c * sub;
            if (left == 1) {
                const uint64_t key = finish<SMAX>(st[l], t.k[k], k, g, nr);
                nodes++;
                if (lex_less(key, idx, my_key, my_idx)) {
                    my_key = key;
                    my_idx = idx;
                }
                if (key < best) {
                    const unsigned long long old = atomicMin(&gb->best, (unsigned long long)key);
                    best = old < key ? old : key;
                }
                continue;
            }
            place<SMAX, FULL>(st[l], st[l + 1], t.k[k], k, g, nr);
            nodes++;
            const uint64_t sa2 = ra[l] - totA[k], sm2 = rm[l] - totM[k];
            const uint64_t x = st[l + 1].I + sa2, y = st[l + 1].M + sm2;
            if ((nodes & 255u) == 0) best = *(volatile unsigned long long*)&gb->best;
            if (st[l + 1].K + (x >= y ? x : y) > best) continue;
            l++;
            rmask[l] = rmask[l - 1] & ~(1u << k);
            child[l] = 0;
            ra[l] = sa2;
            rm[l] = sm2;
            ioff[l] = idx;
        }
    }
    atomicAdd(&gb->nodes, (unsigned long long)nodes);
    /* CTA lexicographic min of (key, index), then the last CTA merges */
    for (int o = 16; o; o >>= 1) {
        const uint64_t k2 = __shfl_xor_sync(0xFFFFFFFFu, my_key, o), i2 = __shfl_xor_sync(0xFFFFFFFFu, my_idx, o);
        if (lex_less(k2, i2, my_key, my_idx)) {
            my_key = k2;
            my_idx = i2;
        }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        wk[w] = my_key;
        wi[w] = my_idx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < kBnbThreads / 32; q++)
            if (lex_less(wk[q], wi[q], wk[0], wi[0])) {
                wk[0] = wk[q];
                wi[0] = wi[q];
            }
        recs[2 * blockIdx.x] = wk[0];
        recs[2 * blockIdx.x + 1] = wi[0];
        __threadfence();
        last = atomicAdd(&gb->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        uint64_t bk = ~0ull, bi = ~0ull;
        for (unsigned q = 0; q < gridDim.x; q++) {
            const uint64_t k2 = ((volatile unsigned long long*)recs)[2 * q];
            const uint64_t i2 = ((volatile unsigned long long*)recs)[2 * q + 1];
            if (lex_less(k2, i2, bk, bi)) {
                bk = k2;
                bi = i2;
            }
        }
        gb->key = bk;
        gb->index = bi;
    }
}

/* ==================== Suffix memoisation ====================
 * The key of an order is K(prefix) + f(state after the prefix, suffix): the
 * closed rounds' key is additive and everything after depends only on the SM
 * state, the cursor, the open round's (dI, nM) and the remaining set.  Many
 * prefixes reach the same (remaining set, state) (C4: 3,991,680 prefixes of
 * length 7, 42,706 distinct).  So, exactly:
 *   levels j = 0..P-1: expand every distinct node of level j by every unused
 *     kernel, deduplicate the results in a hash table -> level j+1 nodes, and
 *     record the transition (node id, closed-round key increment dK);
 *   suffix: for each distinct level-P node, the D! suffix keys f[u][sigma];
 *   per run (D! consecutive indices sharing a P-prefix): walk the P
 *     transitions -> (u, Kc); key(run, sigma) = Kc + f[u][sigma].
 * Every key is the same exact integer the direct evaluation produces. */
template <int SMAX>
struct DNode {
    uint32_t fa[SMAX], fb[SMAX];
    uint32_t cur, mask;
    uint64_t I, M;
};
constexpr uint32_t kDpEmpty = 0xFFFFFFFFu, kDpBusy = 0xFFFFFFFEu;
constexpr int kDpThreads = 256;
constexpr int kDpWarps = kDpThreads / 32;

template <int SMAX>
__device__ __forceinline__ uint64_t dnode_hash(const DNode<SMAX>& x) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&x);
    uint64_t h = 0x243F6A8885A308D3ull;
#pragma unroll
    for (int i = 0; i < (int)(sizeof(DNode<SMAX>) / 4); i++) h = (h ^ w[i]) * 0x9E3779B97F4A7C15ull;
    return h ^ (h >> 29);
}

template <int SMAX>
__device__ __forceinline__ bool dnode_eq_ldcg(const DNode<SMAX>* stored, const DNode<SMAX>& x) {
    const uint32_t* a = reinterpret_cast<const uint32_t*>(stored);
    const uint32_t* b = reinterpret_cast<const uint32_t*>(&x);
    bool eq = true;
#pragma unroll
    for (int i = 0; i < (int)(sizeof(DNode<SMAX>) / 4); i++) eq &= __ldcg(a + i) == b[i];
    return eq;
}

/* run-length nodes (S' > 32): unused run slots are zero, so equal states have
 * equal words (hash and compare) */
template <>
struct DNode<0> {
    uint32_t fa[RK_RUNS], fb[RK_RUNS], st[RK_RUNS];
    uint32_t nr, cur, mask, pad;
    uint64_t I, M;
};

template <int SMAX, bool FULL>
__device__ __forceinline__ void dnode_fresh(DNode<SMAX>& d, const RkGTab& g) {
    if constexpr (SMAX == 0) {
        for (int i = 0; i < RK_RUNS; i++) d.fa[i] = d.fb[i] = d.st[i] = 0;
        d.fa[0] = g.freshA;
        d.fb[0] = g.freshB;
        d.nr = 1;
        d.pad = 0;
    } else {
#pragma unroll
        for (int i = 0; i < SMAX; i++) {
            d.fa[i] = live_sm<SMAX, FULL>(i, g) ? g.freshA : 0u;
            d.fb[i] = live_sm<SMAX, FULL>(i, g) ? g.freshB : 0u;
        }
    }
    d.cur = d.mask = 0;
    d.I = d.M = 0;
}

/* node -> placement state (closed key 0) */
template <int SMAX>
__device__ __forceinline__ void node_to_st(const DNode<SMAX>& d, St<SMAX>& s) {
    if constexpr (SMAX == 0) {
        for (int i = 0; i < RK_RUNS; i++) {
            s.fa[i] = d.fa[i];
            s.fb[i] = d.fb[i];
            s.st[i] = d.st[i];
        }
        s.nr = d.nr;
    } else {
#pragma unroll
        for (int i = 0; i < SMAX; i++) {
            s.fa[i] = d.fa[i];
            s.fb[i] = d.fb[i];
        }
    }
    s.cur = d.cur;
    s.I = d.I;
    s.M = d.M;
    s.K = 0;
}

/* placement state -> canonical node words */
template <int SMAX>
__device__ __forceinline__ void st_to_node(const St<SMAX>& s, uint32_t mask, DNode<SMAX>& d) {
    if constexpr (SMAX == 0) {
        for (int i = 0; i < RK_RUNS; i++) {
            const bool used = (uint32_t)i < s.nr;
            d.fa[i] = used ? s.fa[i] : 0u;
            d.fb[i] = used ? s.fb[i] : 0u;
            d.st[i] = used ? s.st[i] : 0u;
        }
        d.nr = s.nr;
        d.pad = 0;
    } else {
#pragma unroll
        for (int i = 0; i < SMAX; i++) {
            d.fa[i] = s.fa[i];
            d.fb[i] = s.fb[i];
        }
    }
    d.cur = s.cur;
    d.mask = mask;
    d.I = s.I;
    d.M = s.M;
}

/* Prefix expansion, level j -> j+1, breadth-first over a range's prefixes:
 * entry i of level j+1 (lexicographic prefix index) has parent i / (n-j) and
 * takes the (i mod (n-j))-th unused kernel of the parent (ascending): the same
 * factorial-number-system digits as the unranking (reading L11).  Entries are
 * {node, used mask, K_closed lo, hi}; level 0 is the root. */
struct ExpArgs {
    const uint4* Rj;
    uint64_t aj;
    uint4* Rn;
    uint64_t an, cnt;
    uint32_t j;
    const uint32_t* tid;
    const uint64_t* dk;
};
/* COH: coherent (L2) loads, for tables written earlier in the same (cooperative) launch; else the
 * read-only path */
template <bool COH = false>
__device__ __forceinline__ uint4 expand_one(const ExpArgs& x, uint64_t i0, uint32_t n) {
    const uint32_t full = (1u << n) - 1u;
    const uint64_t i = x.an + i0, parent = i / (n - x.j);
    const uint32_t d = (uint32_t)(i - parent * (n - x.j));
    const uint4 e = x.j ? (COH ? __ldcg(x.Rj + (parent - x.aj)) : __ldg(x.Rj + (parent - x.aj))) : make_uint4(0, 0, 0, 0);
    const uint32_t k = nth_set_bit(full & ~e.y, d);
    const uint32_t c = e.x * n + k;
    const uint64_t Kc = (((uint64_t)e.w << 32) | e.z) + (COH ? __ldcg(x.dk + c) : __ldg(x.dk + c));
    const uint4 r = make_uint4(COH ? __ldcg(x.tid + c) : __ldg(x.tid + c), e.y | (1u << k), (uint32_t)Kc,
                               (uint32_t)(Kc >> 32));
    if (x.Rn) x.Rn[i0] = r; /* the last level is recomputed by the passes that need it, not stored */
    return r;
}

/* One level's arguments (rk_dp_level / the cooperative multi-level launch). */
template <int SMAX>
struct LevelArgs {
    const DNode<SMAX>* Uj;
    const uint32_t* cnt_j;
    DNode<SMAX>* Un;
    uint32_t* cnt_n;
    uint32_t cap_n;
    uint32_t* table;
    uint32_t tmask;
    uint32_t* tid;
    uint64_t* dk;
    uint32_t* ovf;
    ExpArgs xp;
    uint32_t nrem;
};

template <int SMAX, bool FULL, bool COH>
__device__ __forceinline__ void level_body(const RkTables& t, const LevelArgs<SMAX>& a, uint64_t gtid, uint64_t nth) {
    const RkGTab& g = t.g;
    const uint32_t n = g.n, full = (1u << n) - 1u;
    const DNode<SMAX>* __restrict__ Uj = a.Uj;
    DNode<SMAX>* Un = a.Un;
    uint32_t* table = a.table;
    const uint32_t tmask = a.tmask, cap_n = a.cap_n, nrem = a.nrem;
    uint32_t* ovf = a.ovf;
    /* an overflowed level (capped planning capacities) stops every
     * later level: its count may exceed the nodes it stored */
    const uint32_t m = Uj ? (*(volatile uint32_t*)ovf ? 0u : *(volatile const uint32_t*)a.cnt_j) : 1u;
    NoRec nr;
    for (uint64_t x = gtid; x < a.xp.cnt; x += nth) expand_one<COH>(a.xp, x, n);
    /* one item per live child: node u of level j by its d-th unused kernel (every node of a level
     * has nrem = n - j unused kernels); transitions stay at u * n + k, entries of used kernels are
     * never read (nor written) */
    for (uint64_t w = gtid; w < (uint64_t)m * nrem; w += nth) {
        const uint32_t u = (uint32_t)(w / nrem), d = (uint32_t)(w - (uint64_t)u * nrem);
        DNode<SMAX> nd;
        if (Uj) {
            if constexpr (COH) { /* written by the previous level of this launch: through L2 */
                uint32_t* w32 = reinterpret_cast<uint32_t*>(&nd);
                const uint32_t* src = reinterpret_cast<const uint32_t*>(Uj + u);
#pragma unroll
                for (int q = 0; q < (int)(sizeof(DNode<SMAX>) / 4); q++) w32[q] = __ldcg(src + q);
            } else {
                nd = Uj[u];
            }
        } else {
            dnode_fresh<SMAX, FULL>(nd, g);
        }
        const uint32_t k = nth_set_bit(full & ~nd.mask, d), c = u * n + k;
        St<SMAX> s, s2;
        node_to_st<SMAX>(nd, s);
        place<SMAX, FULL>(s, s2, t.k[k], k, g, nr);
        DNode<SMAX> o;
        st_to_node<SMAX>(s2, nd.mask | (1u << k), o);
        uint32_t pos = (uint32_t)dnode_hash(o) & tmask, id = kDpEmpty;
        for (uint32_t probes = 0;; probes++) {
            if (probes > tmask) { /* table full (only with capped planning capacities) */
                atomicOr(ovf, 1u);
                break;
            }
            uint32_t v;
            /* test, then test-and-set: most children of the big levels find their state already
             * published (C4 level 8: 213k children, 42.6k states), so a load (acquire: a published
             * id makes its record visible, paired with the release below) spares the CAS that would
             * serialise on a popular slot */
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(table + pos) : "memory");
            if (v == kDpEmpty)
                asm volatile("atom.acquire.gpu.global.cas.b32 %0, [%1], %2, %3;"
                             : "=r"(v)
                             : "l"(table + pos), "r"(kDpEmpty), "r"(kDpBusy)
                             : "memory");
            if (v == kDpEmpty) { /* claimed: allocate, write the record, publish the id (release) */
                /* warp-aggregated id allocation: one atomic per group of claimants (every claim
                 * of a level hits this one counter, so per-thread atomics serialise at L2) */
                const cg::coalesced_group cl = cg::coalesced_threads();
                uint32_t base = 0;
                if (cl.thread_rank() == 0) base = atomicAdd(a.cnt_n, cl.size());
                id = cl.shfl(base, 0) + cl.thread_rank();
                if (id < cap_n) Un[id] = o;
                else atomicOr(ovf, 1u);
                uint32_t old;
                asm volatile("atom.release.gpu.global.exch.b32 %0, [%1], %2;"
                             : "=r"(old)
                             : "l"(table + pos), "r"(id)
                             : "memory");
                (void)old;
                break;
            }
            while (v == kDpBusy) {
                __nanosleep(32);
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(table + pos) : "memory");
            }
            if (v >= cap_n) { /* an overflowed entry: the result is discarded (plan re-sizes) */
                atomicOr(ovf, 1u);
                id = v;
                break;
            }
            if (dnode_eq_ldcg(Un + v, o)) {
                id = v;
                break;
            }
            pos = (pos + 1u) & tmask;
        }
        a.tid[c] = id;
        a.dk[c] = s2.K;
    }
}

/* One level: nodes of level j (count *cnt_j; nullptr = the fresh root) x unused
 * kernels; the same launch also runs the previous level's prefix expansion (xp). */
template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kDpThreads) rk_dp_level_kernel(const RkTables* __restrict__ tab,
                                                                const LevelArgs<SMAX> a) {
    __shared__ RkTables t;
    load_tables(t, tab);
    level_body<SMAX, FULL, false>(t, a, blockIdx.x * (uint64_t)blockDim.x + threadIdx.x,
                                  gridDim.x * (uint64_t)blockDim.x);
}

/* Several small levels in one cooperative launch (grid-wide barrier between
 * levels instead of launch boundaries; the levels of a few hundred to a few
 * ten thousand items are each one dependent chain per item, so a launch per
 * level mostly pays its own start-up). */
constexpr int kCoopMaxLevels = 8;
template <int SMAX>
struct LevelBatch {
    LevelArgs<SMAX> a[kCoopMaxLevels];
    uint32_t nl;
};
template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kDpThreads) rk_dp_levels_coop_kernel(const RkTables* __restrict__ tab,
                                                                      const LevelBatch<SMAX> b) {
    __shared__ RkTables t;
    load_tables(t, tab);
    cg::grid_group grid = cg::this_grid();
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nth = gridDim.x * (uint64_t)blockDim.x;
    for (uint32_t l = 0; l < b.nl; l++) {
        if (l) {
            __threadfence();
            grid.sync();
        }
        level_body<SMAX, FULL, true>(t, b.a[l], gtid, nth);
    }
}

/* The first levels in ONE CTA (shared memory; no global atomics, no fences).
 * Per level: every live child's state is staged in shared memory; after a
 * barrier each child inserts its staging index into a shared hash table and,
 * since every record is already visible, compares records directly (no
 * claim/publish protocol); the children that own their slot are the level's
 * distinct states and take ids in item order (a block scan: deterministic
 * ids); nodes, transitions and the count go to the level arrays in global
 * memory, and the range's level-(j-1) prefix expansion runs as in the level
 * kernel.  C4: levels 0-2 (12 + 132 + 1140 children). */
constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxLevels = 4;
template <int SMAX>
struct SmallLevels {
    LevelArgs<SMAX> a[kSmallMaxLevels];
    uint32_t nl, items_max, hmask; /* hash slots = hmask + 1 >= 2 * items_max */
};
template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kSmallThreads) rk_dp_small_levels_kernel(const RkTables* __restrict__ tab,
                                                                          const SmallLevels<SMAX> b) {
    __shared__ RkTables t;
    __shared__ uint32_t s_warp[kSmallThreads / 32];
    __shared__ uint32_t s_m;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    load_tables(t, tab);
    const RkGTab& g = t.g;
    const uint32_t n = g.n, full = (1u << n) - 1u, IM = b.items_max;
    DNode<SMAX>* cur = reinterpret_cast<DNode<SMAX>*>(sm_raw);            /* level j nodes (<= IM) */
    DNode<SMAX>* stg = cur + IM;                                           /* staged children */
    uint64_t* sdk = reinterpret_cast<uint64_t*>(stg + IM);                 /* their closed-key increments */
    uint32_t* sc = reinterpret_cast<uint32_t*>(sdk + IM);                  /* their transition index u*n+k */
    uint32_t* sown = sc + IM;                                              /* their slot owner (staging index) */
    uint32_t* sid = sown + IM;                                             /* owner -> id (exclusive scan) */
    uint32_t* ht = sid + IM;                                               /* hash slots */
    const uint32_t tidx = threadIdx.x, lane = tidx & 31u, wid = tidx >> 5;
    if (tidx == 0) {
        dnode_fresh<SMAX, FULL>(cur[0], g);
        s_m = 1;
    }
    __syncthreads();
    for (uint32_t l = 0; l < b.nl; l++) {
        const LevelArgs<SMAX>& a = b.a[l];
        const uint32_t m = s_m, nrem = a.nrem, items = m * nrem;
        if (items > IM) { /* more children than the staging holds (planning capacities): flag, stop */
            if (tidx == 0) atomicOr(a.ovf, 1u);
            return;
        }
        /* the range's level j-1 -> j prefix expansion (tables written earlier in this launch) */
        for (uint64_t x = tidx; x < a.xp.cnt; x += kSmallThreads) expand_one<true>(a.xp, x, n);
        for (uint32_t i = tidx; i <= b.hmask; i += kSmallThreads) ht[i] = kDpEmpty;
        NoRec nr;
        for (uint32_t w = tidx; w < items; w += kSmallThreads) { /* stage every live child */
            const uint32_t u = w / nrem, d = w - u * nrem;
            const DNode<SMAX> nd = cur[u];
            const uint32_t k = nth_set_bit(full & ~nd.mask, d);
            St<SMAX> s0, s2;
            node_to_st<SMAX>(nd, s0);
            place<SMAX, FULL>(s0, s2, t.k[k], k, g, nr);
            st_to_node<SMAX>(s2, nd.mask | (1u << k), stg[w]);
            sdk[w] = s2.K;
            sc[w] = u * n + k;
        }
        __syncthreads();
        for (uint32_t w = tidx; w < items; w += kSmallThreads) { /* insert by staging index, compare records */
            const DNode<SMAX>& o = stg[w];
            uint32_t pos = (uint32_t)dnode_hash(o) & b.hmask, own = w;
            for (;;) {
                const uint32_t v = atomicCAS(ht + pos, kDpEmpty, w);
                if (v == kDpEmpty) break;
                const uint32_t* x = reinterpret_cast<const uint32_t*>(stg + v);
                const uint32_t* y = reinterpret_cast<const uint32_t*>(&o);
                bool eq = true;
#pragma unroll
                for (int q = 0; q < (int)(sizeof(DNode<SMAX>) / 4); q++) eq &= x[q] == y[q];
                if (eq) {
                    own = v;
                    break;
                }
                pos = (pos + 1u) & b.hmask;
            }
            sown[w] = own;
        }
        __syncthreads();
        /* ids: owners in item order (block-wide exclusive scan of the owner flags) */
        uint32_t cnt = 0, flags = 0;
        const uint32_t per = (items + kSmallThreads - 1) / kSmallThreads, w0 = tidx * per;
        for (uint32_t q = 0; q < per; q++) {
            const uint32_t w = w0 + q;
            const bool f = w < items && sown[w] == w;
            flags |= (f ? 1u : 0u) << q;
            cnt += f ? 1u : 0u;
        }
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            uint32_t v = lane < kSmallThreads / 32 ? s_warp[lane] : 0u, vi = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, vi, o);
                if (lane >= (uint32_t)o) vi += y;
            }
            if (lane < kSmallThreads / 32) s_warp[lane] = vi - v; /* exclusive warp offsets */
            if (lane == 31) s_m = vi;                             /* the level's distinct states */
        }
        __syncthreads();
        uint32_t id = s_warp[wid] + incl - cnt;
        for (uint32_t q = 0; q < per; q++)
            if ((flags >> q) & 1u) sid[w0 + q] = id++;
        __syncthreads();
        const uint32_t mn = s_m;
        if (tidx == 0) *a.cnt_n = min(mn, a.cap_n);
        if (mn > a.cap_n || mn > IM) { /* does not fit (planning capacities): flag, stop */
            if (tidx == 0) atomicOr(a.ovf, 1u);
            return;
        }
        for (uint32_t w = tidx; w < items; w += kSmallThreads) {
            const uint32_t own = sown[w], nid = sid[own];
            a.tid[sc[w]] = nid;
            a.dk[sc[w]] = sdk[w];
            if (own == w) { /* the node, and its id in the level's global table (distinct states: no compare) */
                a.Un[nid] = stg[w];
                uint32_t pos = (uint32_t)dnode_hash(stg[w]) & a.tmask;
                while (atomicCAS(a.table + pos, kDpEmpty, nid) != kDpEmpty) pos = (pos + 1u) & a.tmask;
            }
        }
        __syncthreads();
        for (uint32_t w = tidx; w < items; w += kSmallThreads) /* the next level's nodes */
            if (sown[w] == w) cur[sid[w]] = stg[w];
        __syncthreads();
    }
}

/* Race audit of one level's lock-free hash table after a build (no sanitizer
 * on this pool): bad[0] count over capacity, bad[1] slots left
 * BUSY (a claim never published), bad[2] published ids >= count, bad[3] nodes
 * whose probe from their own hash meets an EMPTY slot or another id with an
 * equal record first (lost publish / duplicate state), bad[4] live
 * transitions of the previous level (unused kernels) that are not < count, bad[5]
 * published slots (must equal the count). */
template <int SMAX>
__global__ void rk_dp_audit_kernel(const DNode<SMAX>* __restrict__ U, const uint32_t* cnt_p, uint32_t cap,
                                   const uint32_t* __restrict__ table, uint32_t tmask,
                                   const uint32_t* __restrict__ tid_prev, uint64_t work_prev,
                                   const DNode<SMAX>* __restrict__ Uprev, uint32_t n, unsigned long long* bad) {
    const uint32_t cnt = *cnt_p, c = min(cnt, cap);
    const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nth = gridDim.x * (uint64_t)blockDim.x;
    if (gt == 0 && cnt > cap) atomicAdd(bad + 0, 1ull);
    for (uint64_t i = gt; i <= (uint64_t)tmask; i += nth) {
        const uint32_t v = table[i];
        if (v == kDpBusy) atomicAdd(bad + 1, 1ull);
        else if (v != kDpEmpty) atomicAdd(bad + (v >= c ? 2 : 5), 1ull);
    }
    for (uint64_t id = gt; id < c; id += nth) {
        const DNode<SMAX> x = U[id];
        uint32_t pos = (uint32_t)dnode_hash(x) & tmask;
        bool ok = false;
        for (uint32_t p = 0; p <= tmask; p++) {
            const uint32_t v = table[pos];
            if (v == kDpEmpty) break;
            if (v < c && dnode_eq_ldcg(U + v, x)) {
                ok = v == (uint32_t)id;
                break;
            }
            pos = (pos + 1u) & tmask;
        }
        if (!ok) atomicAdd(bad + 3, 1ull);
    }
    for (uint64_t i = gt; i < work_prev; i += nth) { /* live transitions (unused kernels) only */
        const uint64_t u = i / n;
        const uint32_t k = (uint32_t)(i - u * n);
        if (Uprev && ((Uprev[u].mask >> k) & 1u)) continue;
        const uint32_t v = tid_prev[i];
        if (v >= c) atomicAdd(bad + 4, 1ull);
    }
}

/* Suffix tables: for node u of level P, the D! = 120 keys (from K = 0) of its
 * remaining kernels' orders, lexicographic in the remaining ascending ids.  A
 * warp per node: lanes 0..19 take the 20 (first, second) suffix kernels and
 * evaluate the 6 orders below each; the row is then encoded as its sorted
 * distinct values dv (with multiplicities dc; ~14 per row on C4) and one byte
 * code per order (code = rank of its key among dv), plus min/max/argmin/argmax. */

constexpr uint32_t kDF = 120; /* D! for the memo suffix depth D = 5 */

/* The (D-1)! = 24 suffix keys (from K = 0) of every level-(P+1) node, in the
 * lexicographic order of its 4 remaining kernels (ascending ids): thread per
 * (node, first, second) triple places the first two and evaluates both orders
 * of the last two (place + finish). */
template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kDpThreads) rk_dp_row24_kernel(const RkTables* __restrict__ tab,
                                                                const DNode<SMAX>* __restrict__ U,
                                                                const uint32_t* __restrict__ cnt,
                                                                uint64_t* __restrict__ row24) {
    __shared__ RkTables t;
    load_tables(t, tab);
    const RkGTab& g = t.g;
    const uint32_t n = g.n, m = *cnt;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < (uint64_t)m * 12u;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t w = (uint32_t)(x / 12u), ab = (uint32_t)(x - (uint64_t)w * 12u);
        const DNode<SMAX> nd0 = U[w];
        uint32_t rem = 0, q0 = 0;
        for (uint32_t k = 0; k < n; k++)
            if (!((nd0.mask >> k) & 1u)) rem |= k << (4u * q0++);
        const uint32_t a = ab / 3u, b = ab - 3u * a;
        const uint32_t ka = (rem >> (4u * a)) & 15u;
        const uint32_t r3 = (rem & ((1u << (4u * a)) - 1u)) | ((rem >> (4u * a + 4u)) << (4u * a));
        const uint32_t kb = (r3 >> (4u * b)) & 15u;
        const uint32_t r2 = (r3 & ((1u << (4u * b)) - 1u)) | ((r3 >> (4u * b + 4u)) << (4u * b));
        const uint32_t kc = r2 & 15u, kd = (r2 >> 4) & 15u; /* kc < kd */
        St<SMAX> s, s1, s2;
        node_to_st<SMAX>(nd0, s);
        NoRec nr;
        place<SMAX, FULL>(s, s1, t.k[ka], ka, g, nr);
        place<SMAX, FULL>(s1, s2, t.k[kb], kb, g, nr);
        uint64_t* o = row24 + (uint64_t)w * 24u + 6u * a + 2u * b;
        o[0] = place_finish<SMAX, FULL>(s2, t.k[kc], kc, t.k[kd], kd, g);
        o[1] = place_finish<SMAX, FULL>(s2, t.k[kd], kd, t.k[kc], kc, g);
    }
}

/* Suffix rows of the level-P nodes: the 120 keys (from K = 0) of a node's 5
 * remaining kernels' orders, lexicographic in the remaining ascending ids —
 * order a*24 + r is the a-th remaining kernel first: key = dK(u, k_a) +
 * row24[child(u, k_a)][r] through the level-P transitions (the same additivity
 * as the memo itself).  A warp per node encodes the row as its sorted
 * distinct values dv (with multiplicities dc; ~14 per row on C4) and one byte
 * code per order (code = rank of its key among dv), the decoded 32-bit
 * offsets from the row minimum, plus min/max/argmin/argmax. */
template <int SMAX, bool FULL>
__global__ void __launch_bounds__(kDpThreads) rk_dp_suffix_kernel(const RkTables* __restrict__ tab,
                                                                 const DNode<SMAX>* __restrict__ UP,
                                                                 const uint32_t* __restrict__ cnt_P,
                                                                 const uint32_t* __restrict__ tidP,
                                                                 const uint64_t* __restrict__ dkP,
                                                                 const uint64_t* __restrict__ row24,
                                                                 uint8_t* __restrict__ code, ulonglong2* __restrict__ dvc,
                                                                 uint2* __restrict__ dvp, uint32_t* __restrict__ nd,
                                                                 uint64_t* __restrict__ fst, uint32_t* __restrict__ offs) {
    const uint32_t n = tab->g.n, lane = threadIdx.x & 31u;
    const uint32_t m = *cnt_P;
    for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < m; u += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t mask = UP[u].mask;
        uint32_t rem = 0, q0 = 0;
        for (uint32_t k = 0; k < n; k++)
            if (!((mask >> k) & 1u)) rem |= k << (4u * q0++);
        uint64_t v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint32_t sg = lane + 32u * q, a = sg / 24u, r = sg - 24u * a;
            v[q] = ~0ull;
            if (sg < kDF) {
                const uint32_t c = u * n + ((rem >> (4u * a)) & 15u);
                v[q] = __ldg(dkP + c) + __ldg(row24 + (uint64_t)__ldg(tidP + c) * 24u + r);
            }
        }
        /* distinct values in increasing order by repeated warp minimum (~14 rounds) */
        uint32_t done = 0, rank = 0, cdw = 0; /* done: bit q; cdw: the lane's 4 codes, one byte each */
#pragma unroll
        for (int q = 0; q < 4; q++) done |= (lane + 32u * q < kDF ? 0u : 1u) << q;
        uint64_t mn = 0, mx = 0;
        uint32_t amn = 0, amx = 0;
        /* the row's range: when it spans < 2^32 (the common case) the rounds run on
         * 32-bit offsets with one REDUX.MIN per round */
        uint64_t r_lo = ~0ull, r_hi = 0;
#pragma unroll
        for (int q = 0; q < 4; q++)
            if (!((done >> q) & 1u)) {
                r_lo = v[q] < r_lo ? v[q] : r_lo;
                r_hi = v[q] > r_hi ? v[q] : r_hi;
            }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t y = __shfl_xor_sync(0xFFFFFFFFu, r_lo, o), z = __shfl_xor_sync(0xFFFFFFFFu, r_hi, o);
            r_lo = y < r_lo ? y : r_lo;
            r_hi = z > r_hi ? z : r_hi;
        }
        const bool narrow = ((r_hi - r_lo) >> 32) == 0;
        for (uint32_t processed = 0; narrow && processed < kDF;) {
            uint32_t w32[4], lm = 0xFFFFFFFFu;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                w32[q] = (uint32_t)(v[q] - r_lo);
                if (!((done >> q) & 1u) && w32[q] < lm) lm = w32[q];
            }
            lm = __reduce_min_sync(0xFFFFFFFFu, lm);
            uint32_t cnt = 0, firstsg = 0xFFFFFFFFu;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const bool hit = !((done >> q) & 1u) && w32[q] == lm;
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, hit);
                cnt += __popc(bal);
                if (bal && firstsg == 0xFFFFFFFFu) firstsg = 32u * q + (uint32_t)(__ffs(bal) - 1);
                if (hit) {
                    done |= 1u << q;
                    cdw |= rank << (8 * q);
                }
            }
            const uint64_t val = r_lo + lm;
            if (rank == 0) {
                mn = val;
                amn = firstsg;
            }
            if (lane == 0) {
                dvc[(uint64_t)u * kDF + rank] = make_ulonglong2(val, cnt);
                dvp[(uint64_t)u * kDF + rank] = make_uint2(lm, cnt);
            }
            mx = val;
            amx = firstsg;
            rank++;
            processed += cnt;
        }
        for (; !narrow;) {
            uint64_t lm = ~0ull;
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (!((done >> q) & 1u) && v[q] < lm) lm = v[q];
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const uint64_t y = __shfl_xor_sync(0xFFFFFFFFu, lm, o);
                lm = y < lm ? y : lm;
            }
            if (lm == ~0ull) break; /* keys < 2^63: the sentinel means all done */
            uint32_t cnt = 0, firstsg = 0xFFFFFFFFu;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const bool hit = !((done >> q) & 1u) && v[q] == lm;
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, hit);
                cnt += __popc(bal);
                if (bal && firstsg == 0xFFFFFFFFu) firstsg = 32u * q + (uint32_t)(__ffs(bal) - 1);
                if (hit) {
                    done |= 1u << q;
                    cdw |= rank << (8 * q);
                }
            }
            if (rank == 0) {
                mn = lm;
                amn = firstsg;
            }
            if (lane == 0) {
                dvc[(uint64_t)u * kDF + rank] = make_ulonglong2(lm, cnt);
                dvp[(uint64_t)u * kDF + rank] = make_uint2((uint32_t)(lm - mn), cnt); /* offset exact when the row spans < 2^32 */
            }
            mx = lm;
            amx = firstsg;
            rank++;
        }
        /* codes and decoded 32-bit offsets from the row minimum: sigma = lane + 32q */
#pragma unroll
        for (int q = 0; q < 4; q++)
            if (lane + 32u * q < kDF) {
                code[(uint64_t)u * kDF + lane + 32u * q] = (uint8_t)(cdw >> (8 * q));
                offs[(uint64_t)u * kDF + lane + 32u * q] = (uint32_t)v[q]; /* low 32 bits of the suffix key */
            }
        if (lane == 0) {
            nd[u] = rank | ((mx - mn) >> 32 ? 0x80000000u : 0u); /* bit 31: offsets do not fit 32 bits */
            fst[4 * (uint64_t)u] = mn;
            fst[4 * (uint64_t)u + 1] = mx;
            fst[4 * (uint64_t)u + 2] = amn;
            fst[4 * (uint64_t)u + 3] = amx;
        }
        __syncwarp();
    }
}

/* (node, closed key) of run `run`: the P-prefix of index run*D! through the transitions */
__device__ __forceinline__ void dp_walk(const RkGTab& g, const DPView& v, uint64_t run, uint32_t& u, uint64_t& Kc) {
    const uint32_t n = g.n;
    uint64_t L = identity_list(n);
    uint64_t rem = run * v.Dfact;
    u = 0;
    Kc = 0;
    for (uint32_t j = 0; j < v.P; j++) {
        const uint64_t f = g.fact[n - 1 - j];
        const uint32_t d = (rem < (1ull << 32) && f < (1ull << 32)) ? (uint32_t)rem / (uint32_t)f : (uint32_t)(rem / f);
        rem -= (uint64_t)d * f;
        const uint32_t k = take_nibble(L, d);
        const uint32_t c = u * n + k;
        Kc += __ldg(v.dk[j] + c);
        u = __ldg(v.tid[j] + c);
    }
}

constexpr uint32_t kDpEdgeBins = 32768; /* histogram up to this many shared-memory bins */

/* (node, closed key) of run `run` of a pass over the runs [rb, re): from the
 * range's last prefix-expansion level (recomputed from level P-1 in L2, never
 * stored), else by walking the P transitions */
__device__ __forceinline__ void dp_src(const RkGTab& g, const DPView& v, const ExpArgs& xp, uint64_t run, uint64_t rb,
                                       uint32_t& u, uint64_t& Kc) {
    if (xp.cnt) {
        const uint4 e = expand_one(xp, run - rb, g.n);
        u = e.x;
        Kc = ((uint64_t)e.w << 32) | e.z;
    } else {
        dp_walk(g, v, run, u, Kc);
    }
}

/* key of suffix order q of node u after a prefix with closed key Kc (Kb = Kc +
 * the row minimum): decoded 32-bit offsets, or byte codes into the 64-bit
 * distinct values when the row spans >= 2^32 (nd bit 31) */
__device__ __forceinline__ uint64_t dp_key(const DPView& v, uint32_t u, bool wide, uint64_t Kc, uint64_t Kb,
                                           uint32_t q) {
    const uint64_t at = (uint64_t)u * v.Dfact + q;
    if (!wide) return Kb + (uint32_t)(__ldg(v.offs + at) - (uint32_t)(Kb - Kc)); /* offset from the row min */
    const uint8_t c = __ldg(v.code + at);
    return Kc + __ldg(&reinterpret_cast<const ulonglong2*>(v.dvc)[(uint64_t)u * v.Dfact + c].x);
}

/* Row multiset of a range: the runs of [first, first+count) as
 * distinct rows (node, K_closed) with multiplicities — C4's 3,991,680 runs are
 * 217,659 distinct rows, so pass 2 counts and bins 18x fewer rows.  Open
 * addressing over 16-B slots {node, 1, K_closed}: one 128-bit CAS
 * (EMPTY = all zero -> the key) claims a slot or reports its occupant, so no
 * flag protocol (and no acquire fence, which costs an L1 invalidation per
 * load) is needed; the multiplicity is added to one of 8 counters per slot,
 * chosen by CTA index (C4's heaviest row has 11,056 runs).  A run that finds
 * no slot within kRowProbes probes, or a range-edge run, is appended to the
 * run list instead (pass 2 processes it on its own).  Slots and counters are
 * zeroed before the run pass. */
constexpr uint32_t kRowProbes = 32u;
constexpr uint32_t kMultShards = 8; /* multiplicity counters per slot (summed by pass 2) */
struct RowSet {
    uint4* slot;       /* nullptr: no multiset (every run is an item) */
    uint32_t* mult;    /* kMultShards per slot */
    uint32_t mask;     /* slots - 1 */
    uint32_t* list;    /* run offsets from rb */
    uint32_t* nlist;   /* device counter */
    uint32_t* minrun;  /* per slot: the smallest run offset (from rb) in the row (argmin/argmax) */
    uint4* wlist;      /* weighted rows that found no slot: {node, m, K_closed lo, hi} */
    uint32_t* wminrun; /* their smallest run offsets */
    uint32_t* nwlist;  /* device counter */
};
__device__ __forceinline__ uint32_t row_hash(uint32_t uw, uint64_t Kb) {
    uint64_t h = (Kb ^ ((uint64_t)uw << 40) ^ uw) * 0x9E3779B97F4A7C15ull;
    return (uint32_t)(h >> 32) ^ (uint32_t)h;
}
__device__ __forceinline__ void cas128(uint4* p, uint64_t v0, uint64_t v1, uint64_t& r0, uint64_t& r1) {
    const uint64_t z = 0;
    asm volatile("{\n .reg .b128 c, v, d;\n mov.b128 c, {%2, %2};\n mov.b128 v, {%3, %4};\n"
                 " atom.relaxed.gpu.global.cas.b128 d, [%5], c, v;\n mov.b128 {%0, %1}, d;\n}"
                 : "=l"(r0), "=l"(r1)
                 : "l"(z), "l"(v0), "l"(v1), "l"(p)
                 : "memory");
}
__device__ __forceinline__ bool row_insert(const RowSet& rs, uint32_t uw, uint64_t Kb, uint32_t off,
                                           uint32_t w = 1u, uint32_t tag = 1u) {
    const uint64_t k0 = (uint64_t)uw | ((uint64_t)tag << 32), k1 = Kb; /* little-endian {uw, tag != 0, Kb lo, hi} */
    uint32_t h = row_hash(uw, Kb) & rs.mask;
    for (uint32_t p = 0; p < kRowProbes; p++, h = (h + 1u) & rs.mask) {
        uint64_t o0, o1;
        cas128(rs.slot + h, k0, k1, o0, o1);
        if ((o0 == 0 && o1 == 0) || (o0 == k0 && o1 == k1)) { /* claimed, or already this row */
            atomicAdd(rs.mult + (uint64_t)h * kMultShards + (blockIdx.x & (kMultShards - 1u)), w);
            /* runs arrive roughly in index order: test first, so a heavy row's later runs
             * (C4: up to 11,056 per row) do not serialise on one address */
            if (off < __ldcg(rs.minrun + h)) atomicMin(rs.minrun + h, off);
            return true;
        }
    }
    return false;
}

/* Pass 1's run pass (lane per run; runs beside the suffix-row build on a side
 * stream — it needs only the levels): per run of [first, first+count) its
 * (node, K_closed) from the range's last prefix-expansion level (recomputed,
 * or by walking the P transitions) into meta_u / meta_K, and, with a row
 * multiset, whole runs enter their row (node, K_closed); range-edge runs and
 * probe overflows go to the run list. */
__global__ void __launch_bounds__(kDpThreads) rk_dp_runs_kernel(const RkTables* __restrict__ tab, DPView v,
                                                               uint64_t first, uint64_t count, uint32_t* meta_u,
                                                               uint64_t* meta_K, RowSet rs, ExpArgs xp) {
    __shared__ RkTables t;
    load_tables(t, tab);
    const RkGTab& g = t.g;
    constexpr uint32_t DF = kDF;
    const uint64_t lo = first, hi = first + count;
    const uint64_t rb = lo / DF, re = (hi + DF - 1) / DF;
    for (uint64_t run = rb + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; run < re;
         run += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u;
        uint64_t Kc;
        dp_src(g, v, xp, run, rb, u, Kc);
        meta_u[run - rb] = u;
        meta_K[run - rb] = Kc;
        if (rs.slot) {
            const uint64_t idx0 = run * DF;
            const bool whole = idx0 >= lo && idx0 + DF <= hi;
            if (!whole || !row_insert(rs, u, Kc, (uint32_t)(run - rb)))
                rs.list[atomicAdd(rs.nlist, 1u)] = (uint32_t)(run - rb);
        }
    }
}

/* The row multiset without a pass over every run (the range's prefixes are
 * expanded breadth-first, level P-1 stored): (1) rk_dp_parents_kernel
 * collapses the level-(P-1) prefixes whose D' = n - P + 1 child runs are all
 * whole runs of the range into a parent multiset of distinct (node, K_closed)
 * (C4: 665,280 prefixes -> ~10^5 distinct pairs; the node's used mask rides in
 * the slot's tag word); their other runs go to the run list.  (2)
 * rk_dp_children_kernel expands every distinct parent by its D' unused kernels
 * through the level-(P-1) transitions into the row multiset with the parent's
 * multiplicity, and the child run of its smallest parent (offset
 * (parent * D' + d) - rb) as the row's smallest run; a row that finds no slot
 * goes to the weighted list. */
__global__ void __launch_bounds__(kDpThreads) rk_dp_parents_kernel(ExpArgs xp, uint32_t n, uint64_t first,
                                                                  uint64_t count, RowSet ps, RowSet rs) {
    constexpr uint32_t DF = kDF;
    const uint64_t lo = first, hi = first + count;
    const uint64_t rb = lo / DF, re = (hi + DF - 1) / DF;
    const uint32_t D1 = n - xp.j;
    const uint64_t npar = (re - 1) / D1 - xp.aj + 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npar;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = xp.aj + i, r0 = p * D1, r1 = r0 + D1;
        const bool whole = r0 * DF >= lo && r1 * DF <= hi;
        if (whole) {
            const uint4 e = __ldg(xp.Rj + i);
            if (row_insert(ps, e.x, ((uint64_t)e.w << 32) | e.z, (uint32_t)i, 1u, e.y | 0x80000000u)) continue;
        }
        for (uint64_t r = max(r0, rb); r < min(r1, re); r++) rs.list[atomicAdd(rs.nlist, 1u)] = (uint32_t)(r - rb);
    }
}

__global__ void __launch_bounds__(kDpThreads) rk_dp_children_kernel(ExpArgs xp, uint32_t n, uint64_t rb, RowSet ps,
                                                                   RowSet rs) {
    const uint32_t D1 = n - xp.j, full = (1u << n) - 1u;
    const uint64_t items = ((uint64_t)ps.mask + 1u) * D1;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < items;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = x / D1;
        const uint32_t d = (uint32_t)(x - i * D1);
        const uint4 key = ps.slot[i];
        if (!key.y) continue;
        const uint4* ms = reinterpret_cast<const uint4*>(ps.mult + i * kMultShards);
        const uint4 a0 = ms[0], a1 = ms[1];
        const uint32_t m = a0.x + a0.y + a0.z + a0.w + a1.x + a1.y + a1.z + a1.w;
        const uint32_t k = nth_set_bit(full & ~(key.y & 0xFFFFu), d);
        const uint32_t c = key.x * n + k;
        const uint32_t u = __ldg(xp.tid + c);
        const uint64_t Kc = (((uint64_t)key.w << 32) | key.z) + __ldg(xp.dk + c);
        const uint32_t off = (uint32_t)((xp.aj + ps.minrun[i]) * D1 + d - rb);
        if (!row_insert(rs, u, Kc, off, m)) {
            const uint32_t q = atomicAdd(rs.nwlist, 1u);
            rs.wlist[q] = make_uint4(u, m, (uint32_t)Kc, (uint32_t)(Kc >> 32));
            rs.wminrun[q] = off;
        }
    }
}

/* Pass 1's extremes (after the run pass and the suffix rows): the range's
 * min/argmin and max/argmax (smallest index on ties, reading L12) from the
 * row multiset — a distinct row (node, K_closed) of multiplicity m whose
 * smallest run is r has its minimum K_closed + row min at index
 * (rb + r) * D! + row argmin, likewise the maximum — plus the run list (range
 * edges key by key, probe overflows whole), or every run without a multiset.
 * out = {extremes, n_lt = n_eq = 0, n_gt = evaluated = count} (pass 2 adds the
 * counts). */
__global__ void __launch_bounds__(kDpThreads) rk_dp_ext_kernel(DPView v, uint64_t first, uint64_t count, RowSet rs,
                                                              const uint32_t* __restrict__ meta_u,
                                                              const uint64_t* __restrict__ meta_K, rk_stats* out,
                                                              rk_stats* recs, uint32_t* counter) {
    constexpr uint32_t DF = kDF;
    const uint64_t lo = first, hi = first + count;
    const uint64_t rb = lo / DF, re = (hi + DF - 1) / DF;
    const bool direct = rs.slot == nullptr;
    const uint64_t nslot = direct ? 0u : (uint64_t)rs.mask + 1u, nl = direct ? re - rb : *rs.nlist;
    const uint64_t nitems = nslot + nl + (direct ? 0u : *rs.nwlist);
    uint64_t kmin = ~0ull, kmax = 0, amin = ~0ull, amax = ~0ull, cnt = 0;
    auto whole_row = [&](uint32_t u, uint64_t Kc, uint64_t r, uint64_t orders) {
        const ulonglong2 mm = __ldg(reinterpret_cast<const ulonglong2*>(v.fst + 4ull * u));     /* min, max */
        const ulonglong2 ai = __ldg(reinterpret_cast<const ulonglong2*>(v.fst + 4ull * u) + 1); /* argmin, argmax */
        const uint64_t idx0 = (rb + r) * DF, K0 = Kc + mm.x, K1 = Kc + mm.y, am = idx0 + ai.x, ax = idx0 + ai.y;
        if (lex_less(K0, am, kmin, amin)) { kmin = K0; amin = am; }
        if (K1 > kmax || (K1 == kmax && ax < amax)) { kmax = K1; amax = ax; }
        cnt += orders;
    };
    for (uint64_t it = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; it < nitems;
         it += (uint64_t)gridDim.x * blockDim.x) {
        if (it < nslot) { /* a distinct row */
            const uint4 key = rs.slot[it];
            if (!key.y) continue;
            const uint4* ms = reinterpret_cast<const uint4*>(rs.mult + it * kMultShards);
            const uint4 a0 = ms[0], a1 = ms[1];
            const uint32_t m = a0.x + a0.y + a0.z + a0.w + a1.x + a1.y + a1.z + a1.w;
            whole_row(key.x, ((uint64_t)key.w << 32) | key.z, rs.minrun[it], (uint64_t)m * DF);
            continue;
        }
        if (it >= nslot + nl) { /* a weighted row without a slot */
            const uint4 e = rs.wlist[it - nslot - nl];
            whole_row(e.x, ((uint64_t)e.w << 32) | e.z, rs.wminrun[it - nslot - nl], (uint64_t)e.y * DF);
            continue;
        }
        const uint32_t off = direct ? (uint32_t)it : rs.list[it - nslot];
        const uint32_t u = __ldg(meta_u + off);
        const uint64_t Kc = __ldg(meta_K + off), idx0 = (rb + off) * DF;
        const uint32_t olo = lo > idx0 ? (uint32_t)(lo - idx0) : 0u;
        const uint32_t ohi = hi < idx0 + DF ? (uint32_t)(hi - idx0) : DF;
        if (olo == 0 && ohi == DF) {
            whole_row(u, Kc, off, DF);
        } else { /* range-edge run (at most two per range): key by key */
            const uint64_t Kb = Kc + __ldg(v.fst + 4ull * u);
            const bool wide = (__ldg(v.nd + u) >> 31) != 0;
            for (uint32_t q = olo; q < ohi; q++) {
                const uint64_t K = dp_key(v, u, wide, Kc, Kb, q), ix = idx0 + q;
                if (lex_less(K, ix, kmin, amin)) { kmin = K; amin = ix; }
                if (K > kmax || (K == kmax && ix < amax)) { kmax = K; amax = ix; }
                cnt++;
            }
        }
    }
    rk_stats r{};
    r.key_min = kmin;
    r.key_max = kmax;
    r.argmin = amin;
    r.argmax = amax;
    r.n_gt = cnt;
    r.evaluated = cnt;
    r = block_reduce(r);
    commit(r, recs, counter, out);
}

/* Pass 2's counts against the candidate (reading L13) and Fig. 1 histogram over
 * range's [key_min, key_max] (reading L14), from the
 * range's row multiset: item i < slots is a distinct row (node, Kb) with
 * multiplicity m (weight m); item slots + j is run list entry j (weight 1;
 * range-edge runs restricted to the range).  Without a multiset (rs.slot ==
 * nullptr) every run of the range is an item of weight 1.
 * Per row: wholly below the candidate counts m x D!, within one bin adds m x
 * D! to it; otherwise its sorted distinct values (two per 16-B load, 8 in
 * flight; lane l starts at pair l, so lanes rarely collide on a bin) count
 * against the candidate (rows containing it) and add m x count to their bins
 * in the warp's private shared bins.  u64 counts; rows heavier than kHeavy add
 * to the u64 global bins directly, and the shared u32 bins are flushed before
 * their bound can reach 2^31. */
constexpr uint32_t kPrivBins = 1024; /* per-warp private bins up to this many bins */
constexpr uint32_t kHeavy = 2048;    /* heavier rows add to the global bins directly */
__global__ void __launch_bounds__(kDpThreads) rk_dp_rows_kernel(const RkTables* __restrict__ tab, DPView v,
                                                               uint64_t first, uint64_t count,
                                                               const uint64_t* __restrict__ cand_dev,
                                                               const rk_stats* __restrict__ range, uint32_t bins,
                                                               uint64_t* hist, RowSet rs,
                                                               const uint32_t* __restrict__ meta_u,
                                                               const uint64_t* __restrict__ meta_K, rk_stats* rec) {
    __shared__ unsigned long long cnt_lt, cnt_eq;
    __shared__ BinCalc sbc;
    __shared__ uint32_t smx[2];
    extern __shared__ uint32_t shist[]; /* bins x (warps if private) */
    const bool H = hist != nullptr;
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const bool priv = bins <= kPrivBins;
    const uint32_t nsh = H ? (priv ? bins * kDpWarps : bins) : 0u;
    for (uint32_t i = threadIdx.x; i < nsh; i += blockDim.x) shist[i] = 0;
    uint32_t* wh = shist + (priv ? wid * bins : 0u); /* this warp's bins */
    if (threadIdx.x == 0) {
        cnt_lt = cnt_eq = 0;
        smx[0] = smx[1] = 0;
        if (H) sbc.init(range->key_min, range->key_max, bins);
    }
    __syncthreads();
    const BinCalc bc = sbc;
    const uint64_t cand = *cand_dev;
    (void)tab;
    constexpr uint32_t DF = kDF;
    const uint64_t lo = first, hi = first + count;
    const uint64_t rb = lo / DF;
    const bool direct = rs.slot == nullptr; /* no multiset: every run of the range is an item */
    const uint64_t nrun = (hi + DF - 1) / DF - rb;
    const uint64_t nslot = direct ? 0u : (uint64_t)rs.mask + 1u, nl = direct ? nrun : *rs.nlist;
    const uint64_t nitems = nslot + nl + (direct ? 0u : *rs.nwlist);
    uint64_t nlt = 0, neq = 0;
    uint32_t iter = 0, pass = 0;
    /* a narrow row whose distinct values must be visited one by one is deferred to the
     * warp-cooperative loop below (lanes over its values): {node, Kb, m, ndv | in << 30 | mb << 31} */
    bool defer;
    uint32_t d_u, d_m, d_nf;
    uint64_t d_Kb;
    /* one row (node u, Kb) of weight m; range-edge rows key by key over [olo, ohi) */
    auto do_row = [&](uint32_t u, uint64_t Kb, uint32_t m, uint32_t olo, uint32_t ohi) {
        auto add_bin = [&](uint32_t b, uint64_t w) {
            if (m > kHeavy) atomicAdd((unsigned long long*)&hist[b], (unsigned long long)w);
            else atomicAdd(&wh[b], (uint32_t)w);
        };
        const ulonglong2 mm = __ldg(reinterpret_cast<const ulonglong2*>(v.fst + 4ull * u)); /* min, max */
        const uint64_t Kc = Kb - mm.x;
        const uint32_t ndr = __ldg(v.nd + u);
        const bool wide = (ndr >> 31) != 0;
        if (olo != 0 || ohi != DF) { /* range-edge run: key by key */
            for (uint32_t q = olo; q < ohi; q++) {
                const uint64_t K = dp_key(v, u, wide, Kc, Kb, q);
                nlt += K < cand ? 1u : 0u;
                neq += K == cand ? 1u : 0u;
                if (H) atomicAdd(&wh[bc(K)], 1u);
            }
            return;
        }
        const uint64_t Kx = Kc + mm.y;
        const bool in = cand >= Kb && cand <= Kx; /* the candidate inside the row */
        if (cand > Kx) nlt += (uint64_t)m * DF;
        const uint32_t b0 = H ? bc(Kb) : 0u, b1 = H ? bc(Kx) : 0u;
        const bool mb = b0 != b1;
        if (H && !mb) add_bin(b0, (uint64_t)m * DF); /* one bin */
        if (!in && !mb) return;
        const uint32_t ndv = ndr & 0x7FFFFFFFu;
        if (wide) { /* rows spanning >= 2^32 (rare): value by value */
            const ulonglong2* dr = reinterpret_cast<const ulonglong2*>(v.dvc) + (uint64_t)u * DF;
            for (uint32_t q = 0; q < ndv; q++) {
                const ulonglong2 e = __ldg(dr + q);
                const uint64_t K = Kc + e.x;
                if (in) {
                    nlt += K < cand ? m * e.y : 0ull;
                    neq += K == cand ? m * e.y : 0ull;
                }
                if (mb) add_bin(bc(K), (uint64_t)m * e.y);
            }
            return;
        }
        defer = true; /* the distinct values: warp-cooperative, below */
        d_u = u;
        d_Kb = Kb;
        d_m = m;
        d_nf = ndv | (in ? 0x40000000u : 0u) | (mb ? 0x80000000u : 0u);
    };
    for (uint64_t bbase = (uint64_t)blockIdx.x * blockDim.x; bbase < nitems;
         bbase += (uint64_t)gridDim.x * blockDim.x) { /* block-uniform trip count */
        const uint64_t it = bbase + threadIdx.x;
        uint32_t m = 0;
        defer = false;
        if (it < nitems) {
            if (it >= nslot + nl) { /* a weighted row without a slot */
                const uint4 e = rs.wlist[it - nslot - nl];
                m = e.y;
                do_row(e.x, (((uint64_t)e.w << 32) | e.z) + __ldg(v.fst + 4ull * e.x), m, 0u, DF);
            } else if (it < nslot) { /* a distinct row (node, K_closed) of multiplicity m */
                const uint4 key = rs.slot[it];
                if (key.y) {
                    const uint4* ms = reinterpret_cast<const uint4*>(rs.mult + it * kMultShards);
                    const uint4 a0 = ms[0], a1 = ms[1];
                    m = a0.x + a0.y + a0.z + a0.w + a1.x + a1.y + a1.z + a1.w;
                    const uint32_t u = key.x; /* the slot holds (node, K_closed): Kb = K_closed + the row min */
                    do_row(u, (((uint64_t)key.w << 32) | key.z) + __ldg(v.fst + 4ull * u), m, 0u, DF);
                }
            } else { /* a run: listed, or every run (direct) */
                const uint32_t off = direct ? (uint32_t)it : rs.list[it - nslot];
                const uint64_t idx0 = (rb + off) * DF;
                m = 1u;
                const uint32_t u = __ldg(meta_u + off); /* the run pass's (node, K_closed) */
                do_row(u, __ldg(meta_K + off) + __ldg(v.fst + 4ull * u), 1u,
                       lo > idx0 ? (uint32_t)(lo - idx0) : 0u, hi < idx0 + DF ? (uint32_t)(hi - idx0) : DF);
            }
        }
        /* the deferred rows, one at a time per warp, lanes over their distinct values (8-B {offset,
         * count} loads; converged, unlike a lane-per-row loop over ~14 values) */
        for (uint32_t todo = __ballot_sync(0xFFFFFFFFu, defer); todo; todo &= todo - 1u) {
            const int src = __ffs(todo) - 1;
            const uint32_t u = __shfl_sync(0xFFFFFFFFu, d_u, src), wm = __shfl_sync(0xFFFFFFFFu, d_m, src);
            const uint32_t nf = __shfl_sync(0xFFFFFFFFu, d_nf, src);
            const uint64_t Kb = __shfl_sync(0xFFFFFFFFu, d_Kb, src);
            const bool in = (nf >> 30) & 1u, mb = nf >> 31;
            const uint32_t ndv = nf & 0x3FFFFFFFu;
            for (uint32_t i = lane; i < ndv; i += 32u) {
                const uint2 e = __ldg(v.dvp + (uint64_t)u * DF + i);
                const uint64_t K = Kb + e.x;
                if (in) {
                    nlt += K < cand ? (uint64_t)wm * e.y : 0ull;
                    neq += K == cand ? (uint64_t)wm * e.y : 0ull;
                }
                if (mb) {
                    const uint32_t bn = bc(K);
                    if (wm > kHeavy) atomicAdd((unsigned long long*)&hist[bn], (unsigned long long)wm * e.y);
                    else atomicAdd(&wh[bn], wm * e.y);
                }
            }
        }
        if (H) { /* flush before a shared bin can wrap: an iteration adds <= 256 x 120 x min(max m, kHeavy) */
            const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, min(m, kHeavy));
            uint32_t* sm = smx + (pass & 1u); /* double-buffered: slot pass+1 was read by all last pass */
            if (lane == 0) atomicMax(sm, mx);
            __syncthreads();
            iter += *sm;
            if (threadIdx.x == 0) smx[(pass + 1u) & 1u] = 0;
            pass++;
            if (iter >= (1u << 15)) { /* 2^15 x 30720 + 256 x 120 x kHeavy < 2^31 */
                for (uint32_t i = threadIdx.x; i < nsh; i += blockDim.x) {
                    if (shist[i]) atomicAdd((unsigned long long*)&hist[i % bins], (unsigned long long)shist[i]);
                    shist[i] = 0;
                }
                iter = 0;
                __syncthreads();
            }
        }
    }
    unsigned long long x = nlt, y = neq;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
        y += __shfl_xor_sync(0xFFFFFFFFu, y, o);
    }
    if (lane == 0 && (x || y)) {
        atomicAdd(&cnt_lt, x);
        atomicAdd(&cnt_eq, y);
    }
    __syncthreads();
    if (threadIdx.x == 0 && rec && (cnt_lt || cnt_eq)) {
        atomicAdd((unsigned long long*)&rec->n_lt, cnt_lt);
        atomicAdd((unsigned long long*)&rec->n_eq, cnt_eq);
        atomicAdd((unsigned long long*)&rec->n_gt, 0ull - (cnt_lt + cnt_eq));
    }
    if (H)
        for (uint32_t i = threadIdx.x; i < bins; i += blockDim.x) {
            uint64_t s = 0;
            for (uint32_t w = 0; w < (priv ? (uint32_t)kDpWarps : 1u); w++) s += shist[w * bins + i];
            if (s) atomicAdd((unsigned long long*)&hist[i], (unsigned long long)s);
        }
}

/* Pass 2, the key stream (bandwidth-bound; the step's dominant kernel): every
 * key of [first, first+count) to HBM, u64 index-major.  A one-shot grid (no
 * grid-stride loop: CTAs in index order sweep the key array once, which
 * measured 0.51 ms for 3.83 GB vs 0.62-0.75 ms for persistent grid-stride
 * layouts, tools/micro/store_patterns.cu): a warp owns kKeyRunsPerWarp
 * consecutive runs, two per step; lane l stores the key pairs p = l + 32q of
 * the step's 2 x 60 pairs (one contiguous 1920-B block per step, 16-B
 * streaming stores) from the 8-B offset pairs of its run's node row (L2).
 * rb = first / D! and re = ceil((first + count) / D!) come from the host. */
constexpr uint32_t kKeyRunsPerWarp = 4;
__global__ void __launch_bounds__(kDpThreads) rk_dp_keys_kernel(DPView v, uint64_t first, uint64_t count,
                                                               uint64_t rb, uint64_t re,
                                                               const uint32_t* __restrict__ meta_u,
                                                               const uint64_t* __restrict__ meta_K, uint64_t* keys) {
    constexpr uint32_t DF = kDF, PR = kDF / 2; /* key pairs per run */
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t lo = first, hi = first + count;
    const uint64_t base = rb + (uint64_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kKeyRunsPerWarp;
    if (base >= re) return;
    const uint32_t nr = (uint32_t)min((uint64_t)kKeyRunsPerWarp, re - base);
    /* the warp's runs: lane r loads run r's metadata, each step broadcasts two */
    /* lane r < nr: run r's (node, K_closed) -> node | wide << 31 and Kb = K_closed + row min */
    uint32_t umy = 0u, mmy = 0u; /* mmy: low 32 bits of the row minimum (offsets = raw32 - mmy) */
    uint64_t Kmy = 0ull;
    if (lane < nr) {
        const uint32_t u = __ldg(meta_u + (base - rb + lane));
        const uint64_t mn = __ldg(v.fst + 4ull * u);
        Kmy = __ldg(meta_K + (base - rb + lane)) + mn;
        mmy = (uint32_t)mn;
        umy = u | (__ldg(v.nd + u) & 0x80000000u);
    }
    const bool whole = base * DF >= lo && (base + nr) * DF <= hi; /* no range-edge run among them */
    uint64_t* const o0 = keys + (base * DF - lo);
    const bool aligned = (reinterpret_cast<uintptr_t>(o0) & 15u) == 0; /* DF even: every step block alike */
#pragma unroll
    for (uint32_t s = 0; s < kKeyRunsPerWarp / 2; s++) {
        if (2u * s >= nr) break;
        const uint32_t uA = __shfl_sync(0xFFFFFFFFu, umy, 2 * s), uB = __shfl_sync(0xFFFFFFFFu, umy, 2 * s + 1);
        const uint64_t KA = __shfl_sync(0xFFFFFFFFu, Kmy, 2 * s), KB = __shfl_sync(0xFFFFFFFFu, Kmy, 2 * s + 1);
        const uint32_t mA = __shfl_sync(0xFFFFFFFFu, mmy, 2 * s), mB = __shfl_sync(0xFFFFFFFFu, mmy, 2 * s + 1);
        const bool twoB = 2u * s + 1u < nr;
        const uint2* rA = reinterpret_cast<const uint2*>(v.offs + (uint64_t)(uA & 0x7FFFFFFFu) * DF);
        const uint2* rB = reinterpret_cast<const uint2*>(v.offs + (uint64_t)(uB & 0x7FFFFFFFu) * DF);
        uint64_t* o = o0 + 2u * s * DF;
        if (!((uA | (twoB ? uB : 0u)) >> 31)) { /* 32-bit offsets from the row minimum (the common case) */
            uint2 of[4];
#pragma unroll
            for (int q = 0; q < 4; q++) { /* pair p = lane + 32q: run A for p < 60, else run B pair p - 60 */
                const uint32_t p = lane + 32u * q;
                const bool a = p < PR;
                const bool ok = a || (twoB && p < 2u * PR);
                of[q] = ok ? __ldg((a ? rA : rB) + (a ? p : p - PR)) : make_uint2(0, 0);
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t p = lane + 32u * q;
                const bool a = p < PR;
                if (!(a || (twoB && p < 2u * PR))) continue;
                const uint64_t Ki = a ? KA : KB;
                const uint32_t mi = a ? mA : mB;
                const uint64_t k0 = Ki + (uint32_t)(of[q].x - mi), k1 = Ki + (uint32_t)(of[q].y - mi);
                if (whole && aligned) {
                    __stcs(reinterpret_cast<ulonglong2*>(o + 2u * p), make_ulonglong2(k0, k1));
                } else {
                    const uint64_t ix = (base + 2u * s) * DF + 2u * p;
                    if (ix >= lo && ix < hi) __stcs(o + 2u * p, k0);
                    if (ix + 1 >= lo && ix + 1 < hi) __stcs(o + 2u * p + 1, k1);
                }
            }
        } else { /* a row spanning >= 2^32: codes into the 64-bit distinct values */
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t p = lane + 32u * q;
                const bool a = p < PR;
                if (!(a || (twoB && p < 2u * PR))) continue;
                const uint32_t ui = a ? uA : uB, un = ui & 0x7FFFFFFFu, c = a ? p : p - PR;
                const uint64_t Ki = a ? KA : KB;
                uint64_t kk[2];
                if (!(ui >> 31)) {
                    const uint2 of = __ldg(reinterpret_cast<const uint2*>(v.offs + (uint64_t)un * DF) + c);
                    const uint32_t mi = a ? mA : mB;
                    kk[0] = Ki + (uint32_t)(of.x - mi);
                    kk[1] = Ki + (uint32_t)(of.y - mi);
                } else {
                    const ulonglong2* dr = reinterpret_cast<const ulonglong2*>(v.dvc) + (uint64_t)un * DF;
                    const uint64_t Kc = Ki - __ldg(v.fst + 4ull * un);
                    const uint8_t* cr = v.code + (uint64_t)un * DF;
                    kk[0] = Kc + __ldg(&dr[__ldg(cr + 2 * c)].x);
                    kk[1] = Kc + __ldg(&dr[__ldg(cr + 2 * c + 1)].x);
                }
                const uint64_t ix = (base + 2u * s) * DF + 2u * p;
#pragma unroll
                for (int h = 0; h < 2; h++)
                    if (ix + h >= lo && ix + h < hi) __stcs(o + 2u * p + h, kk[h]);
            }
        }
    }
}

/* runs per warp of the compact stream: twice the u64 stream's, so a CTA moves
 * as many bytes (the one-shot grid would otherwise be CTA-launch bound) */
constexpr uint32_t kKey32RunsPerWarp = 8; /* measured: 4 / 8 / 16 within 1 % */
/* Pass 2's key stream with compact keys: every key of [first, first+count) as
 * the exact u32 offset key - key_base from the set's exact lower bound
 * (rk_key_lower_bound), index-major — half the HBM bytes of the u64
 * stream.  A one-shot grid; a warp owns kKeyRunsPerWarp consecutive runs, two
 * per step: a run's 120 keys are 30 16-B chunks, lane l stores chunks l and
 * l + 32 of the step's 60 (one contiguous 960-B block) from 16-B loads of the
 * node's 32-bit offsets (L2).  Overflow is decided once, from the range's
 * record: if range->key_max >= key_base + 2^32 (which also covers every row
 * whose offsets do not fit 32 bits) *ovf is set and nothing is written (the
 * caller re-runs with u64 keys); otherwise every key fits and the stream is
 * plain 32-bit adds. */
template <uint32_t RPW>
__global__ void __launch_bounds__(kDpThreads) rk_dp_keys32_kernel(DPView v, uint64_t first, uint64_t count,
                                                                 uint64_t rb, uint64_t re,
                                                                 const uint32_t* __restrict__ meta_u,
                                                                 const uint64_t* __restrict__ meta_K,
                                                                 uint32_t* keys, uint64_t key_base, uint32_t* ovf,
                                                                 const rk_stats* __restrict__ range) {
    constexpr uint32_t DF = kDF, CH = kDF / 4; /* 16-B chunks per run */
    if ((range->key_max - key_base) >> 32) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(ovf, 1u);
        return;
    }
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t lo = first, hi = first + count;
    const uint64_t base = rb + (uint64_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * RPW;
    if (base >= re) return;
    const uint32_t nr = (uint32_t)min((uint64_t)RPW, re - base);
    /* lane r < nr: run r's node and K_closed.  key - key_base = (K_closed - key_base) + suffix key, and
     * both it and every key's offset are < 2^32 (the range check above; no row is wide then), so the
     * low 32 bits add exactly: offset = low32(K_closed - key_base) + the row's raw32 entry (mod 2^32) */
    uint32_t umy = 0u;
    uint64_t Kmy = 0ull;
    if (lane < nr) {
        umy = __ldg(meta_u + (base - rb + lane));
        Kmy = __ldg(meta_K + (base - rb + lane));
    }
    const bool whole = base * DF >= lo && (base + nr) * DF <= hi;
    uint32_t* const o0 = keys + (base * DF - lo);
    const bool aligned = (reinterpret_cast<uintptr_t>(o0) & 15u) == 0; /* DF % 4 == 0: every run block alike */
    if (whole && aligned && nr == RPW) { /* the common case: every load of the warp's runs issued up front */
        const uint32_t dmy = (uint32_t)(Kmy - key_base); /* every key - key_base < 2^32 */
        uint4 of[RPW / 2][2];
#pragma unroll
        for (uint32_t s = 0; s < RPW / 2; s++)
#pragma unroll
            for (int q = 0; q < 2; q++) { /* chunk p = lane + 32q: run 2s for p < 30, run 2s+1 for 30 <= p < 60 */
                const uint32_t p = lane + 32u * q, r = 2u * s + (p < CH ? 0u : 1u);
                const uint32_t un = __shfl_sync(0xFFFFFFFFu, umy, r) & 0x7FFFFFFFu;
                of[s][q] = p < 2u * CH
                               ? __ldg(reinterpret_cast<const uint4*>(v.offs + (uint64_t)un * DF) + (p < CH ? p : p - CH))
                               : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
        for (uint32_t s = 0; s < RPW / 2; s++)
#pragma unroll
            for (int q = 0; q < 2; q++) {
                const uint32_t p = lane + 32u * q, r = 2u * s + (p < CH ? 0u : 1u);
                const uint32_t d32 = __shfl_sync(0xFFFFFFFFu, dmy, r);
                if (p < 2u * CH)
                    __stcs(reinterpret_cast<uint4*>(o0 + 2u * s * DF + 4u * p),
                           make_uint4(d32 + of[s][q].x, d32 + of[s][q].y, d32 + of[s][q].z, d32 + of[s][q].w));
            }
        return;
    }
#pragma unroll
    for (uint32_t s = 0; s < RPW / 2; s++) {
        if (2u * s >= nr) break;
        const uint32_t uA = __shfl_sync(0xFFFFFFFFu, umy, 2 * s), uB = __shfl_sync(0xFFFFFFFFu, umy, 2 * s + 1);
        const uint64_t KA = __shfl_sync(0xFFFFFFFFu, Kmy, 2 * s), KB = __shfl_sync(0xFFFFFFFFu, Kmy, 2 * s + 1);
        const bool twoB = 2u * s + 1u < nr;
        uint32_t* o = o0 + 2u * s * DF;
        uint4 of[2];
#pragma unroll
        for (int q = 0; q < 2; q++) { /* chunk p = lane + 32q: run A for p < 30, else run B chunk p - 30 */
            const uint32_t p = lane + 32u * q;
            const bool a = p < CH, ok = a || (twoB && p < 2u * CH);
            const uint32_t un = (a ? uA : uB) & 0x7FFFFFFFu;
            of[q] = ok ? __ldg(reinterpret_cast<const uint4*>(v.offs + (uint64_t)un * DF) + (a ? p : p - CH))
                       : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int q = 0; q < 2; q++) {
            const uint32_t p = lane + 32u * q;
            const bool a = p < CH;
            if (!(a || (twoB && p < 2u * CH))) continue;
            const uint32_t d32 = (uint32_t)((a ? KA : KB) - key_base); /* every key - key_base < 2^32 */
            const uint32_t k0 = d32 + of[q].x, k1 = d32 + of[q].y, k2 = d32 + of[q].z, k3 = d32 + of[q].w;
            if (whole && aligned) {
                __stcs(reinterpret_cast<uint4*>(o + 4u * p), make_uint4(k0, k1, k2, k3));
            } else {
                const uint64_t ix = (base + 2u * s) * DF + 4u * p;
                const uint32_t kk[4] = {k0, k1, k2, k3};
#pragma unroll
                for (int h = 0; h < 4; h++)
                    if (ix + h >= lo && ix + h < hi) __stcs(o + 4u * p + h, kk[h]);
            }
        }
    }
}


/* Per-device caches of launch-sizing queries (SM count, occupancy): keyed by the
 * current device, written once with relaxed atomics (idempotent values), so
 * contexts on different devices or host threads never size a grid for another
 * GPU or race on the cache. */
constexpr int kMaxDev = 64;
int cur_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < kMaxDev ? dev : 0;
}
int num_sms() {
    static int cache[kMaxDev];
    const int dev = cur_device();
    int v = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        __atomic_store_n(&cache[dev], v, __ATOMIC_RELAXED);
    }
    return v;
}

template <int SMAX, bool FULL>
int eval_ctas_per_sm() {
    static int cache[kMaxDev];
    const int dev = cur_device();
    int v = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
    if (!v) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, rk_eval_kernel<SMAX, FULL>, kThreads, 0);
        if (v <= 0) v = 1;
        __atomic_store_n(&cache[dev], v, __ATOMIC_RELAXED);
    }
    return v;
}

template <int W>
int policy_ctas_per_sm_w() {
    static int cache[kMaxDev];
    const int dev = cur_device();
    int v = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
    if (!v) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, rk_policy_eval_kernel<W>, kThreads, 0);
        if (v <= 0) v = 1;
        __atomic_store_n(&cache[dev], v, __ATOMIC_RELAXED);
    }
    return v;
}
int policy_ctas_per_sm(uint32_t S) {
    return S <= 2 ? policy_ctas_per_sm_w<2>() : (S <= 8 ? policy_ctas_per_sm_w<8>() : policy_ctas_per_sm_w<32>());
}

/* variant index for a (reduced) SM count S: the smallest power of two >= S,
 * FULL when equal */
int variant(uint32_t S) {
    if (S <= 1) return 0;
    if (S == 2) return 1;
    if (S < 4) return 2;
    if (S == 4) return 3;
    if (S < 8) return 4;
    if (S == 8) return 5;
    if (S < 16) return 6;
    if (S == 16) return 7;
    if (S < 32) return 8;
    if (S == 32) return 9;
    return 10; /* run-length state */
}

} /* namespace */

/* Instantiate KERNEL<SMAX, FULL> for the (reduced) SM count. */
#define RK_DISPATCH(S, KERNEL, CFG, ...)                                     \
    do {                                                                      \
        switch (variant(S)) {                                                 \
            case 0: KERNEL<1, true><<<CFG>>>(__VA_ARGS__); break;             \
            case 1: KERNEL<2, true><<<CFG>>>(__VA_ARGS__); break;             \
            case 2: KERNEL<4, false><<<CFG>>>(__VA_ARGS__); break;            \
            case 3: KERNEL<4, true><<<CFG>>>(__VA_ARGS__); break;             \
            case 4: KERNEL<8, false><<<CFG>>>(__VA_ARGS__); break;            \
            case 5: KERNEL<8, true><<<CFG>>>(__VA_ARGS__); break;             \
            case 6: KERNEL<16, false><<<CFG>>>(__VA_ARGS__); break;           \
            case 7: KERNEL<16, true><<<CFG>>>(__VA_ARGS__); break;            \
            case 8: KERNEL<32, false><<<CFG>>>(__VA_ARGS__); break;           \
            case 9: KERNEL<32, true><<<CFG>>>(__VA_ARGS__); break;            \
            default: KERNEL<0, false><<<CFG>>>(__VA_ARGS__); break;           \
        }                                                                     \
    } while (0)
/* generic (runtime-S) variant for the single-thread helpers */
#define RK_DISPATCH_GENERIC(S, KERNEL, CFG, ...)                              \
    do {                                                                      \
        if ((S) <= 16) KERNEL<16, false><<<CFG>>>(__VA_ARGS__);               \
        else if ((S) <= 32) KERNEL<32, false><<<CFG>>>(__VA_ARGS__);          \
        else KERNEL<0, false><<<CFG>>>(__VA_ARGS__);                          \
    } while (0)
#define RK_CFG(...) __VA_ARGS__
/* model-reading policy kernels: state width 2, 8 or 32 (S' <= 32) */
#define RK_DISPATCH_POLICY(S, KERNEL, CFG, ...)                               \
    do {                                                                      \
        const uint32_t s_ = (S) & ~RK_S_POLICY;                               \
        if (s_ <= 2) KERNEL<2><<<CFG>>>(__VA_ARGS__);                         \
        else if (s_ <= 8) KERNEL<8><<<CFG>>>(__VA_ARGS__);                    \
        else KERNEL<32><<<CFG>>>(__VA_ARGS__);                                \
    } while (0)

int rk_eval_max_ctas(uint32_t S, int) {
    int per;
    switch (variant(S)) {
        case 0: per = eval_ctas_per_sm<1, true>(); break;
        case 1: per = eval_ctas_per_sm<2, true>(); break;
        case 2: per = eval_ctas_per_sm<4, false>(); break;
        case 3: per = eval_ctas_per_sm<4, true>(); break;
        case 4: per = eval_ctas_per_sm<8, false>(); break;
        case 5: per = eval_ctas_per_sm<8, true>(); break;
        case 6: per = eval_ctas_per_sm<16, false>(); break;
        case 7: per = eval_ctas_per_sm<16, true>(); break;
        case 8: per = eval_ctas_per_sm<32, false>(); break;
        case 9: per = eval_ctas_per_sm<32, true>(); break;
        default: per = eval_ctas_per_sm<0, false>(); break;
    }
    return per * num_sms();
}

int rk_launch_eval(const RkTables* tab_dev, uint32_t n, uint32_t S, uint64_t first, uint64_t count,
                   const uint64_t* cand_key_dev, uint64_t cand_key_imm, rk_stats* stats_dev, uint64_t* keys_dev,
                   rk_stats* recs, uint32_t* counter, uint32_t max_ctas, void* stream, uint32_t* launches,
                   uint32_t* keys32_dev, uint64_t key_base, uint32_t* ovf_dev, const rk_stats* hist_range,
                   uint32_t bins, uint64_t* hist_dev) {
    cudaStream_t st = (cudaStream_t)stream;
    if (S & RK_S_POLICY) { /* model-reading policy: one order per thread (no fused extras) */
        if (keys32_dev || hist_dev) return (int)cudaErrorNotSupported;
        uint64_t ctas = (count + kThreads - 1) / kThreads;
        const uint64_t cap = (uint64_t)policy_ctas_per_sm(S & ~RK_S_POLICY) * num_sms();
        if (ctas > cap) ctas = cap;
        if (ctas > max_ctas) ctas = max_ctas;
        if (ctas < 1) ctas = 1;
        RK_DISPATCH_POLICY(S, rk_policy_eval_kernel, RK_CFG((unsigned)ctas, kThreads, 0, st), tab_dev, first, count,
                           cand_key_dev, cand_key_imm, stats_dev, keys_dev, recs, counter);
        if (launches) (*launches)++;
        return (int)cudaGetLastError();
    }
    const uint32_t dm = S <= 2 ? (uint32_t)RK_DEPTH_SMALL : (S <= 8 ? 4u : (uint32_t)RK_DEPTH_LARGE);
    uint64_t R = 1;
    for (uint32_t i = 2; i <= (n < dm ? n : dm); i++) R *= i;
    const uint64_t units = (first + count + R - 1) / R - first / R;
    uint64_t ctas = (units + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)rk_eval_max_ctas(S, 0);
    if (ctas > cap) ctas = cap;
    if (ctas > max_ctas) ctas = max_ctas;
    if (ctas < 1) ctas = 1;
    const size_t smem = hist_dev ? (size_t)bins * 4 : 0;
    if (keys32_dev || hist_dev) {
        if (smem > 48 * 1024) {
            cudaFuncSetAttribute(rk_eval_x_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(rk_eval_x_kernel<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        }
        RK_DISPATCH(S, rk_eval_x_kernel, RK_CFG((unsigned)ctas, kThreads, smem, st), tab_dev, first, count,
                    cand_key_dev, cand_key_imm, stats_dev, keys_dev, recs, counter, keys32_dev, key_base, ovf_dev,
                    hist_range, bins, hist_dev);
        if (launches) (*launches)++;
        return (int)cudaGetLastError();
    }
    RK_DISPATCH(S, rk_eval_kernel, RK_CFG((unsigned)ctas, kThreads, 0, st), tab_dev, first, count, cand_key_dev,
                cand_key_imm, stats_dev, keys_dev, recs, counter, nullptr, 0ull, nullptr, nullptr, 0u, nullptr);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_merge(const rk_stats* in_dev, uint32_t n_records, rk_stats* out_dev, void* stream, uint32_t* launches) {
    rk_merge_groups_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(in_dev, 1, n_records, out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_histogram(const uint64_t* keys_dev, uint64_t count, uint64_t kmin, uint64_t kmax,
                        const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, void* stream,
                        uint32_t* launches) {
    uint64_t ctas = (count / 8 + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * 8;
    if (ctas > cap) ctas = cap;
    if (ctas < 1) ctas = 1;
    const size_t smem = bins <= kSmemBins ? (size_t)bins * 4 : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rk_hist_kernel<false, uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    rk_hist_kernel<false, uint64_t><<<(unsigned)ctas, 256, smem, (cudaStream_t)stream>>>(
        keys_dev, count, kmin, kmax, range_dev, bins, hist_dev, 0ull);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_range_histogram(const uint64_t* keys_dev, uint64_t count, uint64_t lo, uint64_t span, uint32_t bins,
                              uint64_t* hist_dev, void* stream, uint32_t* launches) {
    uint64_t ctas = (count / 8 + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * 8;
    if (ctas > cap) ctas = cap;
    if (ctas < 1) ctas = 1;
    const size_t smem = bins <= kSmemBins ? (size_t)bins * 4 : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rk_hist_kernel<true, uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rk_hist_kernel<true, uint64_t><<<(unsigned)ctas, 256, smem, (cudaStream_t)stream>>>(keys_dev, count, lo, span,
                                                                                          nullptr, bins, hist_dev, 0ull);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_range_histogram32(const uint32_t* keys_dev, uint64_t count, uint64_t key_base, uint64_t lo,
                                uint64_t span, uint32_t bins, uint64_t* hist_dev, void* stream, uint32_t* launches) {
    uint64_t ctas = (count / 8 + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * 8;
    if (ctas > cap) ctas = cap;
    if (ctas < 1) ctas = 1;
    const size_t smem = bins <= kSmemBins ? (size_t)bins * 4 : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rk_hist_kernel<true, uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rk_hist_kernel<true, uint32_t><<<(unsigned)ctas, 256, smem, (cudaStream_t)stream>>>(keys_dev, count, lo, span,
                                                                                          nullptr, bins, hist_dev,
                                                                                          key_base);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_histogram32(const uint32_t* keys_dev, uint64_t count, uint64_t key_base, const rk_stats* range_dev,
                          uint32_t bins, uint64_t* hist_dev, void* stream, uint32_t* launches) {
    uint64_t ctas = (count / 8 + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * 8;
    if (ctas > cap) ctas = cap;
    if (ctas < 1) ctas = 1;
    const size_t smem = bins <= kSmemBins ? (size_t)bins * 4 : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rk_hist_kernel<false, uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    rk_hist_kernel<false, uint32_t><<<(unsigned)ctas, 256, smem, (cudaStream_t)stream>>>(
        keys_dev, count, 0ull, 0ull, range_dev, bins, hist_dev, key_base);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_keys_of(const RkTables* tabs_dev, uint32_t n, uint32_t S, const uint64_t* idx_dev, uint32_t m,
                      uint64_t* out_dev, void* stream, uint32_t* launches) {
    (void)n;
    const unsigned blocks = (m + 127) / 128;
    if (S & RK_S_POLICY)
        RK_DISPATCH_POLICY(S, rk_policy_keys_of_kernel, RK_CFG(blocks, 128, 0, (cudaStream_t)stream), tabs_dev, idx_dev,
                           m, 1, out_dev);
    else
        RK_DISPATCH_GENERIC(S, rk_keys_of_kernel, RK_CFG(blocks, 128, 0, (cudaStream_t)stream), tabs_dev, idx_dev, m, 1,
                            out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_keys_of_same(const RkTables* tab_dev, uint32_t S, const uint64_t* idx_dev, uint32_t m,
                           uint64_t* out_dev, void* stream, uint32_t* launches) {
    const unsigned blocks = (m + 127) / 128;
    if (S & RK_S_POLICY)
        RK_DISPATCH_POLICY(S, rk_policy_keys_of_kernel, RK_CFG(blocks, 128, 0, (cudaStream_t)stream), tab_dev, idx_dev,
                           m, 0, out_dev);
    else
        RK_DISPATCH_GENERIC(S, rk_keys_of_kernel, RK_CFG(blocks, 128, 0, (cudaStream_t)stream), tab_dev, idx_dev, m, 0,
                            out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_key_of_index(const RkTables* tab_dev, uint32_t S, uint64_t index, uint64_t* out_dev, void* stream,
                           uint32_t* launches) {
    if (S & RK_S_POLICY)
        RK_DISPATCH_POLICY(S, rk_policy_key_of_index_kernel, RK_CFG(1, 32, 0, (cudaStream_t)stream), tab_dev, index,
                           out_dev);
    else
        RK_DISPATCH(S, rk_key_of_index_kernel, RK_CFG(1, 32, 0, (cudaStream_t)stream), tab_dev, index, out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_simulate(const RkTables* tab_dev, uint32_t n, uint32_t S, const int32_t* order_dev, uint32_t* rounds_dev,
                       uint32_t max_rounds, uint32_t* n_rounds_dev, uint64_t* key_dev, void* stream,
                       uint32_t* launches) {
    (void)n;
    if (S & RK_S_POLICY)
        RK_DISPATCH_POLICY(S, rk_policy_simulate_kernel, RK_CFG(1, 1, 0, (cudaStream_t)stream), tab_dev, order_dev,
                           rounds_dev, max_rounds, n_rounds_dev, key_dev);
    else
        RK_DISPATCH_GENERIC(S, rk_simulate_kernel, RK_CFG(1, 1, 0, (cudaStream_t)stream), tab_dev, order_dev,
                            rounds_dev, max_rounds, n_rounds_dev, key_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_batch_chunks_per_set(uint32_t n, uint32_t S) {
    if (S & RK_S_POLICY) { /* one order per thread, ~8 per thread */
        uint64_t f = 1;
        for (uint32_t i = 2; i <= n; i++) f *= i;
        const uint64_t chunks = (f + kThreads * 8 - 1) / (kThreads * 8);
        return (int)(chunks < 1 ? 1 : (chunks > 65535 ? 65535 : chunks));
    }
    if (n < 3) return 1;
    const uint32_t dm = S <= 2 ? (uint32_t)RK_DEPTH_SMALL : (S <= 8 ? 4u : (uint32_t)RK_DEPTH_LARGE);
    uint64_t f = 1, R = 1;
    for (uint32_t i = 2; i <= n; i++) f *= i;
    for (uint32_t i = 2; i <= (n < dm ? n : dm); i++) R *= i;
    const uint64_t runs = (f + R - 1) / R;
    uint64_t chunks = (runs + kThreads * 2 - 1) / (kThreads * 2); /* ~2 runs per thread */
    if (chunks < 1) chunks = 1;
    if (chunks > 65535) chunks = 65535;
    return (int)chunks;
}

int rk_launch_batch(const RkTables* tabs_dev, uint32_t n, uint32_t S, uint32_t n_sets, const uint64_t* cand_keys_dev,
                    rk_stats* out_dev, rk_stats* recs, uint32_t chunks, void* stream, uint32_t* launches) {
    (void)n;
    cudaStream_t st = (cudaStream_t)stream;
    const dim3 grid(chunks, n_sets);
    /* S = max reduced SM count over the batch, | 0x80000000 when every set has
     * the same reduced count (then the compile-time variant is exact); otherwise
     * the runtime-S variant runs every set with its own count. */
    const bool uniform = (S & 0x80000000u) != 0;
    const uint32_t Sm = S & 0x7FFFFFFFu;
    if (Sm & RK_S_POLICY) {
        RK_DISPATCH_POLICY(Sm, rk_policy_batch_kernel, RK_CFG(grid, kThreads, 0, st), tabs_dev, cand_keys_dev, recs);
    } else if (uniform) {
        RK_DISPATCH(Sm, rk_batch_kernel, RK_CFG(grid, kThreads, 0, st), tabs_dev, cand_keys_dev, recs);
    } else {
        RK_DISPATCH_GENERIC(Sm, rk_batch_kernel, RK_CFG(grid, kThreads, 0, st), tabs_dev, cand_keys_dev, recs);
    }
    if (launches) (*launches)++;
    const int e = (int)cudaGetLastError();
    if (e) return e;
    const unsigned blocks = (n_sets * 32 + 255) / 256;
    rk_merge_groups_kernel<<<blocks, 256, 0, st>>>(recs, n_sets, chunks, out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

/* memoised batch (rk_batch_memo_kernel): sets with 6 <= n <= 9 on one or two
 * super-SMs (the compile-time FULL variants whose rows are 5! deep) */
bool rk_batch_memo_ok(uint32_t n, uint32_t S) { return n >= 6 && n <= 9 && S >= 1 && S <= 2; }

template <int SMAX>
static int memo_grid(uint32_t n_sets) {
    static int occ = -1;
    if (occ < 0) {
        cudaFuncSetAttribute(rk_batch_memo_kernel<SMAX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kMemoSmem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rk_batch_memo_kernel<SMAX, true>, kThreads,
                                                          kMemoSmem) != cudaSuccess || occ < 1)
            occ = 1;
    }
    const uint64_t cap = (uint64_t)occ * num_sms();
    return (int)(n_sets < cap ? n_sets : cap);
}

int rk_batch_memo_grid(uint32_t S, uint32_t n_sets) { return S == 1 ? memo_grid<1>(n_sets) : memo_grid<2>(n_sets); }

static uint32_t memo_runs(uint32_t n) {
    uint32_t f = 1;
    for (uint32_t i = 6; i <= n; i++) f *= i;
    return f; /* n! / 5! */
}

size_t rk_batch_memo_scratch(uint32_t n, uint32_t S, uint32_t grid) {
    const size_t run = S == 1 ? sizeof(MemoRun<1>) : sizeof(MemoRun<2>);
    return (size_t)grid * memo_runs(n) * (run + kMemoRow * sizeof(uint64_t) + (kMemoD + 1) * sizeof(MemoRowStat));
}

int rk_launch_batch_memo(const RkTables* tabs_dev, uint32_t n, uint32_t S, uint32_t n_sets,
                         const uint64_t* cand_keys_dev, rk_stats* out_dev, void* scratch, uint32_t grid, void* stream,
                         uint32_t* launches) {
    cudaStream_t st = (cudaStream_t)stream;
    const uint32_t stride = memo_runs(n);
    uint64_t* rows = reinterpret_cast<uint64_t*>(scratch);
    MemoRowStat* rst = reinterpret_cast<MemoRowStat*>(rows + (size_t)grid * stride * kMemoRow);
    char* runs = reinterpret_cast<char*>(rst + (size_t)grid * stride * (kMemoD + 1));
    if (S == 1)
        rk_batch_memo_kernel<1, true><<<grid, kThreads, kMemoSmem, st>>>(
            tabs_dev, cand_keys_dev, n_sets, stride, reinterpret_cast<MemoRun<1>*>(runs), rows, rst, out_dev);
    else
        rk_batch_memo_kernel<2, true><<<grid, kThreads, kMemoSmem, st>>>(
            tabs_dev, cand_keys_dev, n_sets, stride, reinterpret_cast<MemoRun<2>*>(runs), rows, rst, out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_heuristic(const rk_kernel* sets_dev, uint32_t n, uint32_t n_sets, const rk_gpu_params* p,
                        int32_t* orders_dev, uint64_t* index_dev, void* stream, uint32_t* launches) {
    const unsigned blocks = (n_sets + 127) / 128;
    rk_heuristic_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(sets_dev, n, n_sets, *p, orders_dev, index_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_bnb_ctas() { return num_sms() * 4; }

int rk_launch_bnb(const RkTables* tab_dev, uint32_t S, uint32_t P, uint64_t n_units, void* gb_dev,
                  unsigned long long* recs_dev, void* stream, uint32_t* launches) {
    if (S & RK_S_POLICY) return (int)cudaErrorNotSupported; /* the host refuses first (RK_EUNSUPPORTED) */
    RK_DISPATCH(S, rk_bnb_kernel, RK_CFG((unsigned)rk_bnb_ctas(), kBnbThreads, 0, (cudaStream_t)stream), tab_dev,
                P, n_units, (BnbGlobal*)gb_dev, recs_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

/* ---- suffix memoisation launchers (register-state variants only) ---- */
namespace {
unsigned dp_grid(uint64_t work) {
    const uint64_t cap = (uint64_t)num_sms() * 8;
    uint64_t b = (work + kDpThreads - 1) / kDpThreads;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}
/* grid-stride kernels: one resident wave (no tail wave) */
template <class K>
unsigned dp_grid_wave(uint64_t work, K kernel, size_t smem) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kDpThreads, smem);
    const uint64_t cap = (uint64_t)num_sms() * (uint64_t)(per > 0 ? per : 1);
    uint64_t b = (work + kDpThreads - 1) / kDpThreads;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}
}  // namespace

uint32_t rk_dp_node_bytes(uint32_t S) {
    switch (variant(S)) {
        case 0: return sizeof(DNode<1>);
        case 1: return sizeof(DNode<2>);
        case 2: case 3: return sizeof(DNode<4>);
        case 4: case 5: return sizeof(DNode<8>);
        case 6: case 7: return sizeof(DNode<16>);
        case 8: case 9: return sizeof(DNode<32>);
        default: return sizeof(DNode<0>);
    }
}

namespace {
template <int SMAX>
LevelArgs<SMAX> level_args(const RkLevel& l) {
    ExpArgs xp{};
    if (l.ex) xp = ExpArgs{(const uint4*)l.ex->Rj, l.ex->aj, (uint4*)l.ex->Rn, l.ex->an, l.ex->cnt, l.ex->j, l.ex->tid,
                           l.ex->dk};
    return LevelArgs<SMAX>{(const DNode<SMAX>*)l.Uj, l.cnt_j, (DNode<SMAX>*)l.Un, l.cnt_n, l.cap_n, l.table, l.tmask,
                           l.tid, l.dk, l.ovf, xp, l.nrem};
}
template <int SMAX, bool FULL>
int launch_levels(const RkTables* tab, const RkLevel* lv, uint32_t nl, cudaStream_t st) {
    if (nl == 1) {
        const RkLevel& l = lv[0];
        const uint64_t xc = l.ex ? l.ex->cnt : 0;
        rk_dp_level_kernel<SMAX, FULL><<<dp_grid(l.work > xc ? l.work : xc), kDpThreads, 0, st>>>(tab,
                                                                                               level_args<SMAX>(l));
        return (int)cudaGetLastError();
    }
    LevelBatch<SMAX> b{};
    b.nl = nl;
    for (uint32_t i = 0; i < nl; i++) b.a[i] = level_args<SMAX>(lv[i]);
    static int cached[64];
    const int dev = cur_device();
    int per = __atomic_load_n(&cached[dev], __ATOMIC_RELAXED);
    if (!per) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rk_dp_levels_coop_kernel<SMAX, FULL>, kDpThreads, 0);
        if (per <= 0) per = 1;
        __atomic_store_n(&cached[dev], per, __ATOMIC_RELAXED);
    }
    const unsigned grid = (unsigned)num_sms() * (unsigned)std::min(per, 2);
    void* args[] = {(void*)&tab, (void*)&b};
    return (int)cudaLaunchCooperativeKernel((const void*)rk_dp_levels_coop_kernel<SMAX, FULL>, grid, kDpThreads, args,
                                            0, st);
}
}  // namespace

namespace {
template <int SMAX, bool FULL>
int launch_small(const RkTables* tab, const RkLevel* lv, uint32_t nl, uint32_t items_max, cudaStream_t st) {
    SmallLevels<SMAX> b{};
    b.nl = nl;
    b.items_max = items_max;
    uint32_t h = 1;
    while (h < 2 * items_max) h <<= 1;
    b.hmask = h - 1;
    for (uint32_t i = 0; i < nl; i++) b.a[i] = level_args<SMAX>(lv[i]);
    const size_t smem = (size_t)items_max * (2 * sizeof(DNode<SMAX>) + 8 + 4 * 3) + (size_t)h * 4;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rk_dp_small_levels_kernel<SMAX, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    rk_dp_small_levels_kernel<SMAX, FULL><<<1, kSmallThreads, smem, st>>>(tab, b);
    return (int)cudaGetLastError();
}
}  // namespace

uint32_t rk_dp_small_items_max(uint32_t S) {
    const size_t budget = 190 * 1024; /* dynamic shared memory of the small-levels kernel */
    size_t node;
    switch (variant(S)) {
        case 0: node = sizeof(DNode<1>); break;
        case 1: node = sizeof(DNode<2>); break;
        case 2: case 3: node = sizeof(DNode<4>); break;
        case 4: case 5: node = sizeof(DNode<8>); break;
        case 6: case 7: node = sizeof(DNode<16>); break;
        case 8: case 9: node = sizeof(DNode<32>); break;
        default: return 0; /* run-length nodes: no small-levels kernel */
    }
    return (uint32_t)(budget / (2 * node + 8 + 12 + 8)) & ~31u;
}

int rk_dp_small_levels(const RkTables* tab, uint32_t S, const RkLevel* lv, uint32_t nl, uint32_t items_max,
                       void* stream, uint32_t* launches) {
    if (nl == 0) return 0;
    if (nl > (uint32_t)kSmallMaxLevels) return (int)cudaErrorInvalidValue;
    cudaStream_t st = (cudaStream_t)stream;
    int e;
    switch (variant(S)) {
        case 0: e = launch_small<1, true>(tab, lv, nl, items_max, st); break;
        case 1: e = launch_small<2, true>(tab, lv, nl, items_max, st); break;
        case 2: e = launch_small<4, false>(tab, lv, nl, items_max, st); break;
        case 3: e = launch_small<4, true>(tab, lv, nl, items_max, st); break;
        case 4: e = launch_small<8, false>(tab, lv, nl, items_max, st); break;
        case 5: e = launch_small<8, true>(tab, lv, nl, items_max, st); break;
        case 6: e = launch_small<16, false>(tab, lv, nl, items_max, st); break;
        case 7: e = launch_small<16, true>(tab, lv, nl, items_max, st); break;
        case 8: e = launch_small<32, false>(tab, lv, nl, items_max, st); break;
        case 9: e = launch_small<32, true>(tab, lv, nl, items_max, st); break;
        default: return (int)cudaErrorInvalidValue;
    }
    if (launches) (*launches)++;
    return e;
}

int rk_dp_levels(const RkTables* tab, uint32_t S, const RkLevel* lv, uint32_t nl, void* stream, uint32_t* launches) {
    if (nl == 0) return 0;
    if (nl > (uint32_t)kCoopMaxLevels) return (int)cudaErrorInvalidValue;
    cudaStream_t st = (cudaStream_t)stream;
    int e;
    switch (variant(S)) {
        case 0: e = launch_levels<1, true>(tab, lv, nl, st); break;
        case 1: e = launch_levels<2, true>(tab, lv, nl, st); break;
        case 2: e = launch_levels<4, false>(tab, lv, nl, st); break;
        case 3: e = launch_levels<4, true>(tab, lv, nl, st); break;
        case 4: e = launch_levels<8, false>(tab, lv, nl, st); break;
        case 5: e = launch_levels<8, true>(tab, lv, nl, st); break;
        case 6: e = launch_levels<16, false>(tab, lv, nl, st); break;
        case 7: e = launch_levels<16, true>(tab, lv, nl, st); break;
        case 8: e = launch_levels<32, false>(tab, lv, nl, st); break;
        case 9: e = launch_levels<32, true>(tab, lv, nl, st); break;
        default: e = launch_levels<0, false>(tab, lv, nl, st); break;
    }
    if (launches) (*launches)++;
    return e;
}

int rk_dp_audit(uint32_t S, const void* U, const uint32_t* cnt, uint32_t cap, const uint32_t* table, uint32_t tmask,
                const uint32_t* tid_prev, uint64_t work_prev, const void* Uprev, uint32_t n, unsigned long long* bad,
                void* stream) {
#define RK_DP_AUDIT_ARGS(SMAX) (const DNode<SMAX>*)U, cnt, cap, table, tmask, tid_prev, work_prev, \
                               (const DNode<SMAX>*)Uprev, n, bad
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned grid = 4u * (unsigned)num_sms();
    switch (variant(S)) {
        case 0: rk_dp_audit_kernel<1><<<grid, 256, 0, st>>>(RK_DP_AUDIT_ARGS(1)); break;
        case 1: rk_dp_audit_kernel<2><<<grid, 256, 0, st>>>(RK_DP_AUDIT_ARGS(2)); break;
        case 2: case 3: rk_dp_audit_kernel<4><<<grid, 256, 0, st>>>(RK_DP_AUDIT_ARGS(4)); break;
        case 4: case 5: rk_dp_audit_kernel<8><<<grid, 256, 0, st>>>(RK_DP_AUDIT_ARGS(8)); break;
        case 6: case 7: rk_dp_audit_kernel<16><<<grid, 256, 0, st>>>(RK_DP_AUDIT_ARGS(16)); break;
        case 8: case 9: rk_dp_audit_kernel<32><<<grid, 256, 0, st>>>(RK_DP_AUDIT_ARGS(32)); break;
        default: rk_dp_audit_kernel<0><<<grid, 256, 0, st>>>(RK_DP_AUDIT_ARGS(0)); break;
    }
#undef RK_DP_AUDIT_ARGS
    return (int)cudaGetLastError();
}

int rk_dp_row24(const RkTables* tab, uint32_t S, const void* U, const uint32_t* cnt, uint64_t* row24, uint64_t nodes,
                void* stream, uint32_t* launches) {
#define RK_DP_R24_ARGS(SMAX) tab, (const DNode<SMAX>*)U, cnt, row24
    const unsigned grid = dp_grid(nodes * 12);
    cudaStream_t st = (cudaStream_t)stream;
    switch (variant(S)) {
        case 0: rk_dp_row24_kernel<1, true><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(1)); break;
        case 1: rk_dp_row24_kernel<2, true><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(2)); break;
        case 2: rk_dp_row24_kernel<4, false><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(4)); break;
        case 3: rk_dp_row24_kernel<4, true><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(4)); break;
        case 4: rk_dp_row24_kernel<8, false><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(8)); break;
        case 5: rk_dp_row24_kernel<8, true><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(8)); break;
        case 6: rk_dp_row24_kernel<16, false><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(16)); break;
        case 7: rk_dp_row24_kernel<16, true><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(16)); break;
        case 8: rk_dp_row24_kernel<32, false><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(32)); break;
        case 9: rk_dp_row24_kernel<32, true><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(32)); break;
        default: rk_dp_row24_kernel<0, false><<<grid, kDpThreads, 0, st>>>(RK_DP_R24_ARGS(0)); break;
    }
#undef RK_DP_R24_ARGS
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_dp_suffix(const RkTables* tab, uint32_t S, const void* UP, const uint32_t* cnt_P, const uint32_t* tidP,
                 const uint64_t* dkP, const uint64_t* row24, uint8_t* code, void* dvc, void* dvp, uint32_t* nd,
                 uint64_t* fst, uint32_t* offs, uint64_t nodes, void* stream, uint32_t* launches) {
#define RK_DP_SUF_ARGS(SMAX) tab, (const DNode<SMAX>*)UP, cnt_P, tidP, dkP, row24, code, (ulonglong2*)dvc, (uint2*)dvp, \
                             nd, fst, offs
    const unsigned grid = dp_grid(nodes * 32);
    cudaStream_t st = (cudaStream_t)stream;
    switch (variant(S)) {
        case 0: rk_dp_suffix_kernel<1, true><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(1)); break;
        case 1: rk_dp_suffix_kernel<2, true><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(2)); break;
        case 2: rk_dp_suffix_kernel<4, false><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(4)); break;
        case 3: rk_dp_suffix_kernel<4, true><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(4)); break;
        case 4: rk_dp_suffix_kernel<8, false><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(8)); break;
        case 5: rk_dp_suffix_kernel<8, true><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(8)); break;
        case 6: rk_dp_suffix_kernel<16, false><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(16)); break;
        case 7: rk_dp_suffix_kernel<16, true><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(16)); break;
        case 8: rk_dp_suffix_kernel<32, false><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(32)); break;
        case 9: rk_dp_suffix_kernel<32, true><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(32)); break;
        default: rk_dp_suffix_kernel<0, false><<<grid, kDpThreads, 0, st>>>(RK_DP_SUF_ARGS(0)); break;
    }
#undef RK_DP_SUF_ARGS
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

namespace {
ExpArgs exp_args(const RkExpand* ex) {
    ExpArgs xp{};
    if (ex) xp = ExpArgs{(const uint4*)ex->Rj, ex->aj, (uint4*)ex->Rn, ex->an, ex->cnt, ex->j, ex->tid, ex->dk};
    return xp;
}
}  // namespace

namespace {
RowSet row_set(const RkRows& r) {
    return RowSet{(uint4*)r.slot, r.mult, r.mask, r.list, r.nlist, r.minrun, (uint4*)r.wlist, r.wminrun, r.nwlist};
}
}  // namespace

int rk_dp_runs(const RkTables* tab, const DPView& v, uint64_t first, uint64_t count, uint32_t* meta_u,
               uint64_t* meta_K, const RkRows& rows, const RkExpand* last, void* stream, uint32_t* launches) {
    const uint64_t runs = (first + count + v.Dfact - 1) / v.Dfact - first / v.Dfact;
    const unsigned grid = dp_grid_wave(runs, rk_dp_runs_kernel, 0);
    rk_dp_runs_kernel<<<grid, kDpThreads, 0, (cudaStream_t)stream>>>(tab, v, first, count, meta_u, meta_K,
                                                                     row_set(rows), exp_args(last));
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_dp_multiset(uint32_t n, uint64_t first, uint64_t count, const RkExpand* lastexp, const RkRows& parents,
                   const RkRows& rows, void* stream, uint32_t* launches) {
    const ExpArgs xp = exp_args(lastexp);
    const uint32_t D1 = n - xp.j;
    const uint64_t rb = first / kDF, re = (first + count + kDF - 1) / kDF;
    const uint64_t npar = (re - 1) / D1 - xp.aj + 1;
    cudaStream_t st = (cudaStream_t)stream;
    rk_dp_parents_kernel<<<dp_grid_wave(npar, rk_dp_parents_kernel, 0), kDpThreads, 0, st>>>(
        xp, n, first, count, row_set(parents), row_set(rows));
    if (launches) (*launches)++;
    int e = (int)cudaGetLastError();
    if (e) return e;
    rk_dp_children_kernel<<<dp_grid_wave(((uint64_t)parents.mask + 1u) * D1, rk_dp_children_kernel, 0), kDpThreads, 0,
                            st>>>(xp, n, rb, row_set(parents), row_set(rows));
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_dp_ext(const DPView& v, uint64_t first, uint64_t count, const RkRows& rows, const uint32_t* meta_u,
              const uint64_t* meta_K, rk_stats* out, rk_stats* recs, uint32_t* counter, uint32_t max_ctas,
              void* stream, uint32_t* launches) {
    const uint64_t runs = (first + count + v.Dfact - 1) / v.Dfact - first / v.Dfact;
    const uint64_t items = rows.slot ? (uint64_t)rows.mask + 1u + rows.list_hint / 64u : runs;
    unsigned grid = dp_grid_wave(items, rk_dp_ext_kernel, 0);
    if (grid > max_ctas) grid = max_ctas;
    rk_dp_ext_kernel<<<grid, kDpThreads, 0, (cudaStream_t)stream>>>(v, first, count, row_set(rows), meta_u, meta_K, out,
                                                                    recs, counter);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_dp_rows(const RkTables* tab, const DPView& v, uint64_t first, uint64_t count, const uint64_t* cand_dev,
               const rk_stats* range, uint32_t bins, uint64_t* hist, const RkRows& rows, const uint32_t* meta_u,
               const uint64_t* meta_K, rk_stats* rec, uint32_t max_ctas, void* stream, uint32_t* launches) {
    if (hist && (bins < 1 || bins > kDpEdgeBins)) return (int)cudaErrorInvalidValue;
    const size_t smem = hist ? (size_t)bins * 4 * (bins <= kPrivBins ? kDpWarps : 1) : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rk_dp_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint64_t items = rows.slot ? (uint64_t)rows.mask + 1u + rows.list_hint : rows.list_hint;
    unsigned grid = dp_grid_wave(items, rk_dp_rows_kernel, smem);
    if (max_ctas && grid > max_ctas) grid = max_ctas;
    rk_dp_rows_kernel<<<grid, kDpThreads, smem, (cudaStream_t)stream>>>(tab, v, first, count, cand_dev, range, bins,
                                                                         hist, row_set(rows), meta_u, meta_K, rec);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_dp_keys(const DPView& v, uint64_t first, uint64_t count, const uint32_t* meta_u, const uint64_t* meta_K,
               uint64_t* keys, void* stream, uint32_t* launches) {
    const uint64_t runs = (first + count + v.Dfact - 1) / v.Dfact - first / v.Dfact;
    const uint64_t per_cta = (uint64_t)kDpWarps * kKeyRunsPerWarp; /* one-shot grid */
    const uint64_t grid = (runs + per_cta - 1) / per_cta;
    if (grid > 0x7FFFFFFFull) return (int)cudaErrorInvalidValue;
    rk_dp_keys_kernel<<<(unsigned)(grid ? grid : 1), kDpThreads, 0, (cudaStream_t)stream>>>(
        v, first, count, first / v.Dfact, (first + count + v.Dfact - 1) / v.Dfact, meta_u, meta_K, keys);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_dp_keys32(const DPView& v, uint64_t first, uint64_t count, const uint32_t* meta_u, const uint64_t* meta_K,
                 uint32_t* keys32, uint64_t key_base, uint32_t* ovf, const rk_stats* range, void* stream,
                 uint32_t* launches) {
    const uint64_t runs = (first + count + v.Dfact - 1) / v.Dfact - first / v.Dfact;
    const uint32_t rpw = kKey32RunsPerWarp;
    const uint64_t per_cta = (uint64_t)kDpWarps * rpw; /* one-shot grid */
    const uint64_t grid = (runs + per_cta - 1) / per_cta;
    if (grid > 0x7FFFFFFFull) return (int)cudaErrorInvalidValue;
    const uint64_t rb = first / v.Dfact, re = (first + count + v.Dfact - 1) / v.Dfact;
    const unsigned g = (unsigned)(grid ? grid : 1);
    cudaStream_t st = (cudaStream_t)stream;
    rk_dp_keys32_kernel<kKey32RunsPerWarp><<<g, kDpThreads, 0, st>>>(v, first, count, rb, re, meta_u, meta_K, keys32,
                                                                      key_base, ovf, range);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

uint32_t rk_dp_max_fused_bins() { return kDpEdgeBins; }



