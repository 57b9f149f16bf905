/*
 * rk_kernels.cu — sm_100a kernels of the exhaustive launch-order evaluation
 * (arXiv 1511.07983).  Product path; shares nothing with oracle/.
 *
 * One thread evaluates a "run": the m! = 6 consecutive lexicographic indices
 * that share an (n-3)-prefix (SURVEY §7 "prefix sharing").  It unranks the
 * prefix (Lehmer code, PAPER:254 / SPEC:292), places the prefix kernels once,
 * then walks the 3-level suffix tree.  Placement of one kernel is the
 * closed-form "water-fill" equivalent of the paper's block-by-block
 * round-robin dispatch (derivation in DESIGN.md
 * §5): per SM the capacity c_s = min over the four limits of
 * floor(free/demand); blocks go round-robin over SMs with remaining capacity,
 * starting at the cursor, so after t full passes SM s holds min(c_s, t); the
 * pass holding the last block and the last block's SM follow from a binary
 * search on t and a select on the ring-rotated eligibility mask.  A block
 * that fits nowhere closes the execution round; rounds are
 * scored exactly as K += max(den*I_r, num*M_r) (reading L1).
 *
 * SM state lives in registers (2 packed u32 per SM, fully unrolled over
 * SMAX), kernel tables in shared memory, reductions via warp shuffles then
 * shared memory then a last-CTA merge (no extra launch).
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include "rk_internal.h"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

__device__ __forceinline__ uint64_t round_key(uint64_t I, uint64_t M, uint32_t num, uint32_t den) {
    uint64_t ci = I * den, cm = M * num; /* max(I_r, R_B M_r) * den, exact */
    return ci >= cm ? ci : cm;
}

template <int SMAX>
struct St {
    uint32_t fa[SMAX], fb[SMAX];
    uint32_t cur;
    uint64_t I, M, K; /* open round's inst/mem units; closed rounds' key */
};

struct NoRec {
    __device__ __forceinline__ void add(uint32_t, uint32_t) {}
    __device__ __forceinline__ void close() {}
    __device__ __forceinline__ void full(uint32_t, uint32_t, uint32_t) {}
};

/* Records the round partition p[r][i] for rk_simulate_order. */
struct Rec {
    uint32_t* rounds;
    uint32_t max_rounds, n, r;
    __device__ void add(uint32_t k, uint32_t cnt) {
        if (r < max_rounds) rounds[r * n + k] += cnt;
    }
    __device__ void close() { r++; }
    __device__ void full(uint32_t k, uint32_t nfull, uint32_t sc) {
        for (uint32_t q = 0; q < nfull; q++) {
            add(k, sc);
            close();
        }
    }
};

template <int SMAX>
__device__ __forceinline__ void st_fresh(St<SMAX>& s, const RkGTab& g) {
#pragma unroll
    for (int i = 0; i < SMAX; i++) {
        s.fa[i] = (uint32_t)i < g.S ? g.freshA : 0u;
        s.fb[i] = (uint32_t)i < g.S ? g.freshB : 0u;
    }
    s.cur = 0;
    s.I = s.M = s.K = 0;
}

/* c_s = min(floor(regs/dr), floor(shm/ds), floor(warps/dw), slots) per SM
 * (the four limits of PAPER:76-78, inclusive <=, reading L8). Returns sum. */
template <int SMAX>
__device__ __forceinline__ uint32_t sm_caps(const St<SMAX>& s, const RkKTab& k, uint32_t (&c)[SMAX]) {
    uint32_t F = 0;
#pragma unroll
    for (int i = 0; i < SMAX; i++) {
        uint32_t qr = mad_hi(s.fa[i] & 0xFFFFu, k.mr, k.zr);
        uint32_t qs = mad_hi(s.fa[i] >> 16, k.ms, k.zs);
        uint32_t qw = mad_hi(s.fb[i] & 0xFFFFu, k.mw, k.zw);
        uint32_t qb = s.fb[i] >> 17;
        c[i] = min(__vimin3_u32(qr, qs, qw), qb);
        F += c[i];
    }
    return F;
}

template <int SMAX>
__device__ __forceinline__ uint32_t rotr_s(uint32_t m, uint32_t r, uint32_t S) {
    uint64_t mm = (uint64_t)m | ((uint64_t)m << S);
    uint32_t full = (S >= 32) ? 0xFFFFFFFFu : ((1u << S) - 1u);
    return (uint32_t)(mm >> r) & full;
}

/* 0-based position of the r-th (1-based) set bit of m (r <= popc(m)). */
template <int SMAX>
__device__ __forceinline__ uint32_t select_bit(uint32_t m, uint32_t r) {
    uint32_t p = 0;
#pragma unroll
    for (int w = (SMAX > 16 ? 16 : 8); w >= 1; w >>= 1) {
        uint32_t lowc = __popc(m & ((1u << w) - 1u));
        if (lowc < r) {
            r -= lowc;
            m >>= w;
            p += (uint32_t)w;
        }
    }
    return p;
}

/* Dispatch all T_k blocks of kernel k into the open round. */
template <int SMAX, class R>
__device__ __forceinline__ void place(St<SMAX>& s, const RkKTab& k, uint32_t kid, const RkGTab& g, R& rec) {
    uint32_t c[SMAX];
    uint32_t F = sm_caps<SMAX>(s, k, c);
    uint32_t n = k.T;
    if (n > F) {
        /* every SM takes its c_s, the next block fits nowhere: the round closes
         * (PAPER:79-80); the rest starts fresh rounds at cursor 0 (reading L4). */
        s.I += (uint64_t)F * k.A;
        s.M += (uint64_t)F * k.M;
        rec.add(kid, F);
        s.K += round_key(s.I, s.M, g.num, g.den);
        rec.close();
        n -= F;
        uint32_t nfull = (n - 1u) / k.SC; /* complete single-kernel rounds */
        s.K += (uint64_t)nfull * k.fullkey;
        rec.full(kid, nfull, k.SC);
        n -= nfull * k.SC;
#pragma unroll
        for (int i = 0; i < SMAX; i++) {
            s.fa[i] = (uint32_t)i < g.S ? g.freshA : 0u;
            s.fb[i] = (uint32_t)i < g.S ? g.freshB : 0u;
            c[i] = (uint32_t)i < g.S ? k.C : 0u;
        }
        s.cur = 0;
        s.I = s.M = 0;
    }
    /* n in [1, sum c]: find the pass t1 = tlo+1 that holds the last block,
     * tlo = max{t : f(t) < n}, f(t) = sum_s min(c_s, t). */
    uint32_t tlo = 0, flo = 0;
    for (uint32_t b = g.tbits; b; b >>= 1) {
        uint32_t tt = tlo + b, f = 0;
#pragma unroll
        for (int i = 0; i < SMAX; i++) f += min(c[i], tt);
        if (f < n) {
            tlo = tt;
            flo = f;
        }
    }
    uint32_t r = n - flo; /* >= 1 blocks in pass t1, to SMs with c_s > tlo in ring order */
    uint32_t E = 0;
#pragma unroll
    for (int i = 0; i < SMAX; i++) E |= (c[i] > tlo ? 1u : 0u) << i;
    uint32_t Er = rotr_s<SMAX>(E, s.cur, g.S);
    uint32_t p = select_bit<SMAX>(Er, r);
    uint32_t Xr = Er & ((2u << p) - 1u);      /* first r eligible SMs from the cursor */
    uint32_t X = rotr_s<SMAX>(Xr, g.S - s.cur, g.S);
    uint32_t nc = s.cur + p + 1u;
    s.cur = nc >= g.S ? nc - g.S : nc;       /* cursor = SM of the last block + 1 */
#pragma unroll
    for (int i = 0; i < SMAX; i++) {
        uint32_t x = min(c[i], tlo) + ((X >> i) & 1u);
        s.fa[i] -= x * k.dA;
        s.fb[i] -= x * k.dB;
    }
    s.I += (uint64_t)n * k.A;
    s.M += (uint64_t)n * k.M;
    rec.add(kid, n);
}

/* Last kernel of an order: only its round split matters, not the SM state. */
template <int SMAX, class R>
__device__ __forceinline__ uint64_t finish(const St<SMAX>& s, const RkKTab& k, uint32_t kid, const RkGTab& g,
                                           R& rec) {
    uint32_t c[SMAX];
    uint32_t F = sm_caps<SMAX>(s, k, c);
    uint32_t n = k.T;
    uint64_t I = s.I, M = s.M, K = s.K;
    if (n <= F) {
        rec.add(kid, n);
        rec.close();
        return K + round_key(I + (uint64_t)n * k.A, M + (uint64_t)n * k.M, g.num, g.den);
    }
    rec.add(kid, F);
    rec.close();
    K += round_key(I + (uint64_t)F * k.A, M + (uint64_t)F * k.M, g.num, g.den);
    n -= F;
    uint32_t nfull = (n - 1u) / k.SC;
    K += (uint64_t)nfull * k.fullkey;
    rec.full(kid, nfull, k.SC);
    n -= nfull * k.SC;
    rec.add(kid, n);
    rec.close();
    return K + round_key((uint64_t)n * k.A, (uint64_t)n * k.M, g.num, g.den);
}

/* Nibble list of unused kernels, ascending: remove and return entry d. */
__device__ __forceinline__ uint32_t take_nibble(uint64_t& L, uint32_t d) {
    uint32_t sh = 4u * d;
    uint32_t v = (uint32_t)(L >> sh) & 15u;
    uint64_t low = L & ((1ull << sh) - 1ull);
    L = low | ((L >> (sh + 4u)) << sh);
    return v;
}
__device__ __forceinline__ uint64_t identity_list(uint32_t n) {
    uint64_t L = 0;
    for (uint32_t i = 0; i < n; i++) L |= (uint64_t)i << (4u * i);
    return L;
}

/* Key of one lexicographic index, from scratch (candidate, samples, n < 3). */
template <int SMAX, class R>
__device__ uint64_t eval_index(const RkTables& t, uint32_t idx, R& rec) {
    const RkGTab& g = t.g;
    const uint32_t n = g.n;
    St<SMAX> s;
    st_fresh<SMAX>(s, g);
    uint64_t L = identity_list(n);
    uint32_t rem = idx;
    for (uint32_t j = 0; j + 1 < n; j++) {
        uint32_t f = g.fact[n - 1 - j];
        uint32_t d = rem / f;
        rem -= d * f;
        uint32_t k = take_nibble(L, d);
        place<SMAX>(s, t.k[k], k, g, rec);
    }
    uint32_t k = (uint32_t)L & 15u;
    return finish<SMAX>(s, t.k[k], k, g, rec);
}

struct TStats {
    uint64_t kmin, kmax;
    uint32_t amin, amax, nlt, neq, cnt;
    __device__ __forceinline__ void init() {
        kmin = ~0ull;
        kmax = 0;
        amin = amax = 0xFFFFFFFFu;
        nlt = neq = cnt = 0;
    }
    __device__ __forceinline__ void add(uint64_t K, uint32_t idx, uint64_t cand) {
        /* indices arrive in increasing order per thread: strict compares keep
         * the smallest index on ties (reading L12) */
        if (K < kmin) { kmin = K; amin = idx; }
        if (K > kmax || cnt == 0) { kmax = K; amax = idx; }
        nlt += (K < cand) ? 1u : 0u;
        neq += (K == cand) ? 1u : 0u;
        cnt += 1u;
    }
};

__device__ __forceinline__ void merge_into(rk_stats& a, const rk_stats& b) {
    if (b.evaluated == 0) return;
    if (a.evaluated == 0) { a = b; return; }
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
    rk_stats r;
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
    rk_stats v;
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

template <int SMAX>
__device__ __forceinline__ void eval_run(const RkTables& t, uint32_t run, uint32_t lo, uint32_t hi, uint64_t cand,
                                         uint64_t* keys, uint32_t first, TStats& ts) {
    const RkGTab& g = t.g;
    const uint32_t n = g.n;
    NoRec nr;
    uint32_t idx0 = run * 6u;
    St<SMAX> s0;
    st_fresh<SMAX>(s0, g);
    uint64_t L = identity_list(n);
    uint32_t rem = idx0;
    for (uint32_t j = 0; j + 3 < n; j++) {
        uint32_t f = g.fact[n - 1 - j];
        uint32_t d = rem / f;
        rem -= d * f;
        uint32_t k = take_nibble(L, d);
        place<SMAX>(s0, t.k[k], k, g, nr);
    }
    const uint32_t r0 = (uint32_t)L & 15u, r1 = (uint32_t)(L >> 4) & 15u, r2 = (uint32_t)(L >> 8) & 15u;
#pragma unroll 1
    for (uint32_t a = 0; a < 3; a++) {
        const uint32_t ka = a == 0 ? r0 : (a == 1 ? r1 : r2);
        const uint32_t kb0 = a == 0 ? r1 : r0, kb1 = a == 2 ? r1 : r2;
        St<SMAX> s1 = s0;
        place<SMAX>(s1, t.k[ka], ka, g, nr);
#pragma unroll 1
        for (uint32_t b = 0; b < 2; b++) {
            const uint32_t kb = b == 0 ? kb0 : kb1, kc = b == 0 ? kb1 : kb0;
            St<SMAX> s2 = s1;
            place<SMAX>(s2, t.k[kb], kb, g, nr);
            uint64_t K = finish<SMAX>(s2, t.k[kc], kc, g, nr);
            uint32_t idx = idx0 + a * 2u + b;
            if (idx >= lo && idx < hi) {
                ts.add(K, idx, cand);
                if (keys) keys[idx - first] = K;
            }
        }
    }
}

__device__ __forceinline__ void load_tables(RkTables& sm, const RkTables* src) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(&sm);
    for (uint32_t i = threadIdx.x; i < sizeof(RkTables) / 4; i += blockDim.x) d[i] = s[i];
    __syncthreads();
}

template <int SMAX>
__global__ void __launch_bounds__(kThreads) rk_eval_kernel(const RkTables* __restrict__ tab, uint32_t first,
                                                          uint32_t count, const uint64_t* cand_dev,
                                                          uint64_t cand_imm, rk_stats* out, uint64_t* keys,
                                                          rk_stats* recs, uint32_t* counter) {
    __shared__ RkTables t;
    load_tables(t, tab);
    const uint64_t cand = cand_dev ? *cand_dev : cand_imm;
    const uint32_t lo = first, hi = first + count;
    TStats ts;
    ts.init();
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    if (t.g.n >= 3) {
        const uint32_t rb = lo / 6u, re = (hi + 5u) / 6u;
        for (uint32_t run = rb + gtid; run < re; run += nth) eval_run<SMAX>(t, run, lo, hi, cand, keys, first, ts);
    } else {
        NoRec nr;
        for (uint32_t idx = lo + gtid; idx < hi; idx += nth) {
            uint64_t K = eval_index<SMAX>(t, idx, nr);
            ts.add(K, idx, cand);
            if (keys) keys[idx - first] = K;
        }
    }
    rk_stats r = block_reduce(to_rec(ts));
    commit(r, recs, counter, out);
}

/* C5 batch: blockIdx.y = set, blockIdx.x = chunk of that set's runs. */
template <int SMAX>
__global__ void __launch_bounds__(kThreads) rk_batch_kernel(const RkTables* __restrict__ tabs,
                                                           const uint64_t* __restrict__ cand_keys,
                                                           rk_stats* recs) {
    __shared__ RkTables t;
    const uint32_t set = blockIdx.y;
    load_tables(t, tabs + set);
    const uint64_t cand = cand_keys[set];
    const uint32_t n = t.g.n;
    const uint32_t total = t.g.fact[n];
    TStats ts;
    ts.init();
    if (n >= 3) {
        const uint32_t runs = total / 6u;
        const uint32_t per = (runs + gridDim.x - 1) / gridDim.x;
        const uint32_t rb = blockIdx.x * per, re = min(runs, rb + per);
        for (uint32_t run = rb + threadIdx.x; run < re; run += blockDim.x)
            eval_run<SMAX>(t, run, 0u, total, cand, nullptr, 0u, ts);
    } else if (blockIdx.x == 0) {
        NoRec nr;
        for (uint32_t idx = threadIdx.x; idx < total; idx += blockDim.x) ts.add(eval_index<SMAX>(t, idx, nr), idx, cand);
    }
    rk_stats r = block_reduce(to_rec(ts));
    if (threadIdx.x == 0) recs[set * gridDim.x + blockIdx.x] = r;
}

/* merge groups of `per` consecutive records: one warp per group */
__global__ void rk_merge_groups_kernel(const rk_stats* __restrict__ in, uint32_t groups, uint32_t per,
                                       rk_stats* __restrict__ out) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= groups) return; /* whole warps exit together */
    rk_stats v;
    v.evaluated = 0;
    for (uint32_t i = lane; i < per; i += 32) merge_into(v, in[(size_t)w * per + i]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        rk_stats o = shfl_rec(v, off);
        merge_into(v, o);
    }
    if (lane == 0) out[w] = v;
}

template <int SMAX>
__global__ void rk_keys_of_kernel(const RkTables* __restrict__ tabs, const uint64_t* __restrict__ idx, uint32_t m,
                                  uint64_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    NoRec nr;
    out[i] = eval_index<SMAX>(tabs[i], (uint32_t)idx[i], nr);
}

template <int SMAX>
__global__ void rk_keys_of_same_kernel(const RkTables* __restrict__ tab, const uint64_t* __restrict__ idx,
                                       uint32_t m, uint64_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    NoRec nr;
    out[i] = eval_index<SMAX>(*tab, (uint32_t)idx[i], nr);
}

template <int SMAX>
__global__ void rk_key_of_index_kernel(const RkTables* __restrict__ tab, uint32_t index, uint64_t* __restrict__ out) {
    __shared__ RkTables t;
    load_tables(t, tab);
    if (threadIdx.x == 0) {
        NoRec nr;
        *out = eval_index<SMAX>(t, index, nr);
    }
}

template <int SMAX>
__global__ void rk_simulate_kernel(const RkTables* __restrict__ tab, const int32_t* __restrict__ order,
                                   uint32_t* rounds, uint32_t max_rounds, uint32_t* n_rounds, uint64_t* key) {
    const RkTables& t = *tab;
    const uint32_t n = t.g.n;
    for (uint32_t i = 0; i < max_rounds * n; i++) rounds[i] = 0;
    Rec rec{rounds, max_rounds, n, 0};
    St<SMAX> s;
    st_fresh<SMAX>(s, t.g);
    for (uint32_t j = 0; j + 1 < n; j++) place<SMAX>(s, t.k[order[j]], (uint32_t)order[j], t.g, rec);
    *key = finish<SMAX>(s, t.k[order[n - 1]], (uint32_t)order[n - 1], t.g, rec);
    *n_rounds = rec.r;
}

/* Fig. 1 histogram: exact integer bins over [kmin, kmax]. */
__global__ void rk_hist_kernel(const uint64_t* __restrict__ keys, uint64_t count, uint64_t kmin_imm,
                               uint64_t kmax_imm, const rk_stats* __restrict__ range, uint32_t bins,
                               uint64_t* __restrict__ hist) {
    extern __shared__ uint32_t sh[];
    const uint64_t kmin = range ? range->key_min : kmin_imm;
    const uint64_t kmax = range ? range->key_max : kmax_imm;
    const uint64_t D = kmax - kmin;
    for (uint32_t i = threadIdx.x; i < bins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const double scale = D ? (double)bins / (double)D : 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t K = keys[i];
        uint32_t b = 0;
        if (D) {
            const uint64_t x = K <= kmin ? 0ull : (K >= kmax ? D : K - kmin);
            /* estimate, then correct with exact 128-bit compares:
             * want b = floor(x*bins / D), i.e. b*D <= x*bins < (b+1)*D */
            double e = (double)x * scale;
            int64_t bb = (int64_t)e;
            if (bb < 0) bb = 0;
            if (bb > (int64_t)bins) bb = bins;
            const uint64_t plo = x * (uint64_t)bins, phi = __umul64hi(x, (uint64_t)bins);
            for (;;) { /* b*D > x*bins ? -> b-- */
                uint64_t qlo = (uint64_t)bb * D, qhi = __umul64hi((uint64_t)bb, D);
                if (qhi > phi || (qhi == phi && qlo > plo)) bb--;
                else break;
            }
            for (;;) { /* (b+1)*D <= x*bins ? -> b++ */
                uint64_t b1 = (uint64_t)bb + 1;
                uint64_t qlo = b1 * D, qhi = __umul64hi(b1, D);
                if (qhi < phi || (qhi == phi && qlo <= plo)) bb++;
                else break;
            }
            b = (uint32_t)bb;
            if (b > bins - 1) b = bins - 1;
        }
        atomicAdd(&sh[b], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < bins; i += blockDim.x)
        if (sh[i]) atomicAdd((unsigned long long*)&hist[i], (unsigned long long)sh[i]);
}

int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <int SMAX>
int eval_ctas_per_sm() {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, rk_eval_kernel<SMAX>, kThreads, 0);
    return b > 0 ? b : 1;
}

} /* namespace */

int rk_eval_max_ctas(uint32_t S, int) {
    int per = S <= 16 ? eval_ctas_per_sm<16>() : eval_ctas_per_sm<32>();
    return per * num_sms();
}

int rk_launch_eval(const RkTables* tab_dev, uint32_t n, uint32_t S, uint64_t first, uint64_t count,
                   const uint64_t* cand_key_dev, uint64_t cand_key_imm, rk_stats* stats_dev, uint64_t* keys_dev,
                   rk_stats* recs, uint32_t* counter, uint32_t max_ctas, void* stream, uint32_t* launches) {
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t units = n >= 3 ? ((first + count + 5) / 6 - first / 6) : count;
    uint64_t ctas = (units + kThreads - 1) / kThreads;
    if (ctas > max_ctas) ctas = max_ctas;
    if (ctas < 1) ctas = 1;
    if (S <= 16)
        rk_eval_kernel<16><<<(unsigned)ctas, kThreads, 0, st>>>(tab_dev, (uint32_t)first, (uint32_t)count,
                                                                  cand_key_dev, cand_key_imm, stats_dev, keys_dev,
                                                                  recs, counter);
    else
        rk_eval_kernel<32><<<(unsigned)ctas, kThreads, 0, st>>>(tab_dev, (uint32_t)first, (uint32_t)count,
                                                                  cand_key_dev, cand_key_imm, stats_dev, keys_dev,
                                                                  recs, counter);
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
    uint64_t ctas = (count + 1023) / 1024;
    uint64_t cap = (uint64_t)num_sms() * 8;
    if (ctas > cap) ctas = cap;
    if (ctas < 1) ctas = 1;
    size_t smem = (size_t)bins * 4;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(rk_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rk_hist_kernel<<<(unsigned)ctas, 256, smem, (cudaStream_t)stream>>>(keys_dev, count, kmin, kmax, range_dev, bins,
                                                                          hist_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_keys_of(const RkTables* tabs_dev, uint32_t n, uint32_t S, const uint64_t* idx_dev, uint32_t m,
                      uint64_t* out_dev, void* stream, uint32_t* launches) {
    (void)n;
    unsigned blocks = (m + 127) / 128;
    if (S <= 16) rk_keys_of_kernel<16><<<blocks, 128, 0, (cudaStream_t)stream>>>(tabs_dev, idx_dev, m, out_dev);
    else rk_keys_of_kernel<32><<<blocks, 128, 0, (cudaStream_t)stream>>>(tabs_dev, idx_dev, m, out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_keys_of_same(const RkTables* tab_dev, uint32_t S, const uint64_t* idx_dev, uint32_t m,
                           uint64_t* out_dev, void* stream, uint32_t* launches) {
    unsigned blocks = (m + 127) / 128;
    if (S <= 16) rk_keys_of_same_kernel<16><<<blocks, 128, 0, (cudaStream_t)stream>>>(tab_dev, idx_dev, m, out_dev);
    else rk_keys_of_same_kernel<32><<<blocks, 128, 0, (cudaStream_t)stream>>>(tab_dev, idx_dev, m, out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_key_of_index(const RkTables* tab_dev, uint32_t S, uint64_t index, uint64_t* out_dev, void* stream,
                           uint32_t* launches) {
    if (S <= 16) rk_key_of_index_kernel<16><<<1, 32, 0, (cudaStream_t)stream>>>(tab_dev, (uint32_t)index, out_dev);
    else rk_key_of_index_kernel<32><<<1, 32, 0, (cudaStream_t)stream>>>(tab_dev, (uint32_t)index, out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_launch_simulate(const RkTables* tab_dev, uint32_t n, uint32_t S, const int32_t* order_dev, uint32_t* rounds_dev,
                       uint32_t max_rounds, uint32_t* n_rounds_dev, uint64_t* key_dev, void* stream,
                       uint32_t* launches) {
    (void)n;
    if (S <= 16)
        rk_simulate_kernel<16><<<1, 1, 0, (cudaStream_t)stream>>>(tab_dev, order_dev, rounds_dev, max_rounds,
                                                                   n_rounds_dev, key_dev);
    else
        rk_simulate_kernel<32><<<1, 1, 0, (cudaStream_t)stream>>>(tab_dev, order_dev, rounds_dev, max_rounds,
                                                                   n_rounds_dev, key_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}

int rk_batch_chunks_per_set(uint32_t n) {
    if (n < 3) return 1;
    uint64_t f = 1;
    for (uint32_t i = 2; i <= n; i++) f *= i;
    uint64_t runs = f / 6;
    uint64_t chunks = (runs + kThreads * 4 - 1) / (kThreads * 4); /* ~4 runs per thread */
    if (chunks < 1) chunks = 1;
    if (chunks > 65535) chunks = 65535;
    return (int)chunks;
}

int rk_launch_batch(const RkTables* tabs_dev, uint32_t n, uint32_t S, uint32_t n_sets, const uint64_t* cand_keys_dev,
                    rk_stats* out_dev, rk_stats* recs, uint32_t chunks, void* stream, uint32_t* launches) {
    (void)n;
    cudaStream_t st = (cudaStream_t)stream;
    dim3 grid(chunks, n_sets);
    if (S <= 16) rk_batch_kernel<16><<<grid, kThreads, 0, st>>>(tabs_dev, cand_keys_dev, recs);
    else rk_batch_kernel<32><<<grid, kThreads, 0, st>>>(tabs_dev, cand_keys_dev, recs);
    if (launches) (*launches)++;
    int e = (int)cudaGetLastError();
    if (e) return e;
    unsigned blocks = (n_sets * 32 + 255) / 256;
    rk_merge_groups_kernel<<<blocks, 256, 0, st>>>(recs, n_sets, chunks, out_dev);
    if (launches) (*launches)++;
    return (int)cudaGetLastError();
}
