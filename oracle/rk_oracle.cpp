/*
 * rk_oracle.cpp — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the execution-round
 * cost model of Li, Narayana & El-Ghazawi, "Reordering GPU Kernel Launches to
 * Enable Efficient Concurrent Execution" (arXiv 1511.07983), evaluated over the
 * permutation space of kernel launch orders, plus the paper's Algorithm 1.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code, header, table or constant
 * with the product path (paper_1511_07983_b200/ and include/): it has its own
 * input structs, its own unranking, its own block-by-block placement and its
 * own Algorithm 1.
 *
 * Citations: PAPER:L = /root/reference/PAPER.md line L; SPEC:L = SPEC.md line L.
 * Readings of gaps in the paper (L1..L23) are listed in DESIGN.md §3.
 *
 * Every function here follows the paper/SPEC step by step:
 *   O1  inputs and per-block demand ............ Table 1
 *   O2  enumerate idx -> order (lexicographic) .. PAPER:254
 *   O3  block-by-block round-robin placement .... PAPER:69-81 (§2)
 *   O4  exact integer round scoring ............. SPEC:210, 232-240, 264
 *   O5  naive double cross-check ................ SPEC:210 (literal formula)
 *   O6  statistics ............................... Table 3
 *   O7  histogram ................................ Fig. 1
 *   O8  Algorithm 1 (ScoreGen/ProfileCombine) .... PAPER:110-198
 *
 * Pins (tests/test_oracle_*.py): hand-derived W4/W2 goldens (tests/golden/),
 * App. C counterexamples, std::next_permutation enumeration, closed forms
 * (single round, same-side theorem, lower bound), §3 invariances, brute-force
 * statistics by sorting, SPEC worked examples for ScoreGen/ProfileCombine.
 * Every function is pinned; none is "parity unpinned".
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

typedef unsigned __int128 u128;

/* ---- O1: inputs (Table 1) ------------------------ */
/* GPU: N_SM, N_reg_SM, N_shm_SM, N_warp_SM, N_blk_SM, R_B = rb_num / rb_den    */
struct OrGpu {
    uint32_t n_sm, regs_per_sm, shm_per_sm, warps_per_sm, blocks_per_sm, rb_num, rb_den;
    uint32_t flags; /* model-reading variants, 0 = readings L4/L5:
                       bit 0: the round-robin cursor restarts at SM 0 for every kernel (L4 alt.)
                       bit 1: strict round robin — a block goes to the SM under the cursor or
                              nowhere; no scan of the other SMs (L4 alt.)
                       bit 2: skip-ahead — a block that fits nowhere defers the rest of its
                              kernel to the next round and dispatch continues with the next
                              kernel in launch order (L5 alt., the option SPEC:262 rejects) */
};
#define OR_CURSOR_PER_KERNEL 1u
#define OR_STRICT_RR 2u
#define OR_SKIP_AHEAD 4u
/* Kernel profile.  inst_per_block A_i = N_inst_i / N_tblk_i;  mem_per_block
 * M_i = A_i / R_i = 4*mem_events_i / N_tblk_i, in
 * instruction units so that the round cost is max(I_r, R_B*M_r). */
struct OrKernel {
    uint32_t grid_blocks, threads_per_block, regs_per_thread, shm_per_block, inst_per_block,
        mem_per_block;
};

/* Per-block demand of kernel i (O1): regs = regs/thread * tpb,
 * shm = shm/block, warps = ceil(tpb/32), one block slot. */
struct Demand {
    uint64_t regs, shm, warps, slots;
};
static Demand demand_of(const OrKernel& k) {
    Demand d;
    d.regs = (uint64_t)k.regs_per_thread * k.threads_per_block;
    d.shm = k.shm_per_block;
    d.warps = (k.threads_per_block + 31) / 32;
    d.slots = 1;
    return d;
}

enum { OR_OK = 0, OR_EINVAL = 1, OR_EINFEASIBLE = 2, OR_ETOOMANY = 3, OR_EMISSINGRATIO = 4, OR_EOVERFLOW = 5 };

static int check_inputs(const OrGpu& g, const OrKernel* k, int n) {
    if (g.n_sm == 0 || g.regs_per_sm == 0 || g.shm_per_sm == 0 || g.warps_per_sm == 0 ||
        g.blocks_per_sm == 0 || g.rb_num == 0 || g.rb_den == 0)
        return OR_EINVAL;
    if (g.flags & ~(OR_CURSOR_PER_KERNEL | OR_STRICT_RR | OR_SKIP_AHEAD)) return OR_EINVAL;
    if (n < 0 || n > 20) return OR_ETOOMANY;
    for (int i = 0; i < n; i++) {
        if (k[i].grid_blocks < 1) return OR_EINVAL;
        if (k[i].threads_per_block < 1 || k[i].threads_per_block > 1024) return OR_EINVAL;
        if (k[i].inst_per_block < 1) return OR_EINVAL;
        if (k[i].mem_per_block < 1) return OR_EMISSINGRATIO;
        Demand d = demand_of(k[i]);
        if (d.regs > g.regs_per_sm || d.shm > g.shm_per_sm || d.warps > g.warps_per_sm)
            return OR_EINFEASIBLE;
    }
    return OR_OK;
}

/* ---- O2: lexicographic unrank / rank (factorial number system) ------------ */
/* idx -> order: L = [0..n-1]; for j: f = (n-1-j)!, d = idx / f, idx %= f,
 * pi_j = L.pop(d).  Ties of the sweep are broken by this order. */
static uint64_t factorial(int m) {
    uint64_t f = 1;
    for (int i = 2; i <= m; i++) f *= (uint64_t)i;
    return f;
}
static void unrank(uint64_t idx, int n, int* order) {
    std::vector<int> L;
    for (int i = 0; i < n; i++) L.push_back(i);
    for (int j = 0; j < n; j++) {
        uint64_t f = factorial(n - 1 - j);
        uint64_t d = idx / f;
        idx %= f;
        order[j] = L[(size_t)d];
        L.erase(L.begin() + (long)d);
    }
}
static uint64_t rank_of(const int* order, int n) {
    std::vector<int> L;
    for (int i = 0; i < n; i++) L.push_back(i);
    uint64_t idx = 0;
    for (int j = 0; j < n; j++) {
        size_t pos = (size_t)(std::find(L.begin(), L.end(), order[j]) - L.begin());
        idx += (uint64_t)pos * factorial(n - 1 - j);
        L.erase(L.begin() + (long)pos);
    }
    return idx;
}

/* ---- O3 + O4 + O5: simulate one launch order -------------------------------
 * PAPER:69-70 "all thread blocks from the earliest issued kernel are first
 * allocated to the SMs, followed by thread blocks from the next issued kernel";
 * PAPER:76-78 "mapped to SMs in a round-robin fashion, until any one of the SM
 * resource limitations is met"; "relegated to the next execution
 * round ... sequentially executed one after the other".
 * Reading L4: next-fit cursor = placed SM + 1, persisting across
 * kernels inside a round, reset to 0 at each new round.  L5: a block that fits
 * nowhere closes the round; no skip-ahead, no backfill. */
struct SmFree {
    uint64_t regs, shm, warps, slots;
};
static bool fits(const SmFree& s, const Demand& d) { /* inclusive <= (L8) */
    return d.regs <= s.regs && d.shm <= s.shm && d.warps <= s.warps && d.slots <= s.slots;
}

struct SimOut {
    u128 key;                          /* K = sum_r max(den*I_r, num*M_r) (O4) */
    double t_naive;                    /* SPEC:210 literal double formula (O5) */
    std::vector<std::vector<uint32_t>> rounds; /* p[r][i] blocks of kernel i in round r */
};

static void close_round(const OrGpu& g, const OrKernel* k, int n, std::vector<uint32_t>& p, SimOut& out,
                        bool keep_rounds) {
    /* O4: I_r = sum p_i*A_i, M_r = sum p_i*M_i,
     * round time max(I_r, R_B*M_r) = max(den*I_r, num*M_r) / den. */
    u128 I = 0, M = 0;
    for (int i = 0; i < n; i++) {
        I += (u128)p[i] * k[i].inst_per_block;
        M += (u128)p[i] * k[i].mem_per_block;
    }
    u128 ci = I * g.rb_den, cm = M * g.rb_num;
    out.key += (ci >= cm) ? ci : cm;
    /* O5: SPEC:210 literally, in double: inst_units = sum inst_count_i *
     * (placed / N_tblk_i); mem_units = sum (inst_count_i / R_i) * (placed / N_tblk_i);
     * time = max(inst_units, R_B * mem_units). */
    double inst_units = 0.0, mem_units = 0.0;
    for (int i = 0; i < n; i++) {
        double inst_count = (double)k[i].grid_blocks * (double)k[i].inst_per_block;
        double R_i = (double)k[i].inst_per_block / (double)k[i].mem_per_block;
        double frac = (double)p[i] / (double)k[i].grid_blocks;
        inst_units += inst_count * frac;
        mem_units += (inst_count / R_i) * frac;
    }
    double R_B = (double)g.rb_num / (double)g.rb_den;
    out.t_naive += std::max(inst_units, R_B * mem_units);
    if (keep_rounds) out.rounds.push_back(p);
    for (int i = 0; i < n; i++) p[i] = 0;
}

/* First SM, in ring order from the cursor, that can take a block of demand d
 * ("round-robin ... until any one of the SM resource limitations is
 * met"), or -1.  Strict round robin (flag bit 1) looks at the cursor's SM only. */
static int find_sm(const OrGpu& g, const std::vector<SmFree>& sm, uint32_t cursor, const Demand& d) {
    const uint32_t S = g.n_sm;
    const uint32_t steps = (g.flags & OR_STRICT_RR) ? 1u : S;
    for (uint32_t step = 0; step < steps; step++) { /* scan ring-wise from the cursor */
        uint32_t s = (cursor + step) % S;
        if (fits(sm[s], d)) return (int)s;
    }
    return -1;
}

/* Skip-ahead reading of L5 (flag bit 2; SPEC:262 names and rejects it): every
 * round offers the pending blocks kernel by kernel in launch order; a kernel
 * whose next block fits nowhere keeps the rest of its blocks for the next
 * round and dispatch moves on to the next kernel.  The round closes once every
 * kernel with pending blocks has been offered; the next round starts with all
 * SMs free and the cursor at SM 0 (as in L4/L5).  Blocks of one kernel stay in
 * order ("all thread blocks from the earliest issued kernel are
 * first allocated").  A fresh round always places at least the first pending
 * block (every kernel is feasible, O1), so the loop ends. */
static void simulate_skip_ahead(const OrGpu& g, const OrKernel* k, int n, const int* order, SimOut& out,
                                bool keep_rounds, std::vector<int32_t>* trace) {
    const uint32_t S = g.n_sm;
    SmFree caps{g.regs_per_sm, g.shm_per_sm, g.warps_per_sm, g.blocks_per_sm};
    std::vector<SmFree> sm(S, caps);
    std::vector<uint32_t> p(n, 0), pending(n, 0);
    uint64_t left = 0;
    for (int j = 0; j < n; j++) {
        pending[j] = k[order[j]].grid_blocks;
        left += pending[j];
    }
    out.key = 0;
    out.t_naive = 0.0;
    out.rounds.clear();
    int round = 0;
    while (left > 0) {
        for (uint32_t s = 0; s < S; s++) sm[s] = caps;
        uint32_t cursor = 0;
        for (int j = 0; j < n; j++) {
            if (pending[j] == 0) continue;
            int ki = order[j];
            Demand d = demand_of(k[ki]);
            if (g.flags & OR_CURSOR_PER_KERNEL) cursor = 0;
            while (pending[j] > 0) {
                int found = find_sm(g, sm, cursor, d);
                if (found < 0) break; /* the rest of kernel ki waits for the next round */
                sm[found].regs -= d.regs;
                sm[found].shm -= d.shm;
                sm[found].warps -= d.warps;
                sm[found].slots -= d.slots;
                p[ki]++;
                pending[j]--;
                left--;
                cursor = ((uint32_t)found + 1) % S;
                if (trace) {
                    trace->push_back(round);
                    trace->push_back(found);
                }
            }
        }
        close_round(g, k, n, p, out, keep_rounds);
        round++;
    }
}

/* trace (optional): for every block in dispatch order, (round, sm). */
static void simulate(const OrGpu& g, const OrKernel* k, int n, const int* order, SimOut& out, bool keep_rounds,
                     std::vector<int32_t>* trace) {
    if (g.flags & OR_SKIP_AHEAD) {
        simulate_skip_ahead(g, k, n, order, out, keep_rounds, trace);
        return;
    }
    const uint32_t S = g.n_sm;
    SmFree caps{g.regs_per_sm, g.shm_per_sm, g.warps_per_sm, g.blocks_per_sm};
    std::vector<SmFree> sm(S, caps);
    std::vector<uint32_t> p(n, 0);
    uint32_t cursor = 0;
    int round = 0;
    bool round_nonempty = false;
    out.key = 0;
    out.t_naive = 0.0;
    out.rounds.clear();
    for (int j = 0; j < n; j++) {
        int ki = order[j];
        Demand d = demand_of(k[ki]);
        if (g.flags & OR_CURSOR_PER_KERNEL) cursor = 0; /* alternative reading of L4 (f3) */
        for (uint32_t b = 0; b < k[ki].grid_blocks; b++) {
            int found = find_sm(g, sm, cursor, d);
            if (found < 0) { /* fits nowhere: close the round, start the next one */
                close_round(g, k, n, p, out, keep_rounds);
                round++;
                for (uint32_t s = 0; s < S; s++) sm[s] = caps;
                cursor = 0;
                found = 0; /* a feasible block always fits a fresh SM (O1) */
            }
            sm[found].regs -= d.regs;
            sm[found].shm -= d.shm;
            sm[found].warps -= d.warps;
            sm[found].slots -= d.slots;
            p[ki]++;
            round_nonempty = true;
            cursor = ((uint32_t)found + 1) % S;
            if (trace) {
                trace->push_back(round);
                trace->push_back(found);
            }
        }
    }
    if (round_nonempty) close_round(g, k, n, p, out, keep_rounds); /* final round */
}

/* ---- O6: statistics over an index range ---------------------------------- */
struct OrStats { /* same meaning as the SweepReport columns */
    uint64_t key_min, key_max, argmin, argmax, n_lt, n_eq, n_gt, evaluated;
};

struct ChunkResult {
    u128 kmin, kmax;
    uint64_t argmin, argmax, n_lt, n_eq, n_gt, evaluated;
    double max_rel_err;
    int err;
};

static void sweep_chunk(const OrGpu& g, const OrKernel* k, int n, uint64_t first, uint64_t count, uint64_t cand,
                        uint64_t* keys_out, ChunkResult& r) {
    r.kmin = 0;
    r.kmax = 0;
    r.argmin = r.argmax = 0;
    r.n_lt = r.n_eq = r.n_gt = r.evaluated = 0;
    r.max_rel_err = 0.0;
    r.err = 0;
    std::vector<int> order(n);
    SimOut out;
    for (uint64_t idx = first; idx < first + count; idx++) {
        unrank(idx, n, order.data());
        simulate(g, k, n, order.data(), out, false, nullptr);
        u128 K = out.key;
        if ((K >> 64) != 0) {
            r.err = OR_EOVERFLOW;
            return;
        }
        /* O5 cross-check: |T_naive - K/den| <= 1e-12 * K/den */
        double T = (double)(uint64_t)K / (double)g.rb_den;
        double rel = (T == 0.0) ? std::fabs(out.t_naive) : std::fabs(out.t_naive - T) / T;
        if (rel > r.max_rel_err) r.max_rel_err = rel;
        if (r.evaluated == 0 || K < r.kmin) { r.kmin = K; r.argmin = idx; } /* strict: smallest idx on ties (L12) */
        if (r.evaluated == 0 || K > r.kmax) { r.kmax = K; r.argmax = idx; }
        if (K < (u128)cand) r.n_lt++;
        else if (K == (u128)cand) r.n_eq++;
        else r.n_gt++;
        r.evaluated++;
        if (keys_out) keys_out[idx - first] = (uint64_t)K;
    }
}

/* ---- O8: Algorithm 1 ------------------------ */
/* Footprint (reading L2): b_i = ceil(N_tblk_i / N_SM);
 * N_warp_i = warps/blk * b_i, N_reg_i = regs/blk * b_i, N_shm_i = shm/blk * b_i,
 * slots = b_i; N_inst_i = N_tblk_i * A_i; R_i = A_i / M_i. */
struct Prof {
    uint64_t H, G, W, Bk; /* shm, regs, warps, block slots (per-SM footprint) */
    double I;             /* N_inst */
    double R;             /* inst/mem ratio */
};
static Prof footprint(const OrGpu& g, const OrKernel& k) {
    Prof p;
    uint64_t b = (k.grid_blocks + g.n_sm - 1) / g.n_sm;
    Demand d = demand_of(k);
    p.H = d.shm * b;
    p.G = d.regs * b;
    p.W = d.warps * b;
    p.Bk = b;
    p.I = (double)k.grid_blocks * (double)k.inst_per_block;
    p.R = (double)k.inst_per_block / (double)k.mem_per_block;
    return p;
}
/* ProfileCombine: sums; R_comb = (I_a+I_b)/(I_a/R_a + I_b/R_b) */
static Prof combine(const Prof& a, const Prof& b) {
    Prof c;
    c.H = a.H + b.H;
    c.G = a.G + b.G;
    c.W = a.W + b.W;
    c.Bk = a.Bk + b.Bk;
    c.I = a.I + b.I;
    c.R = (a.I + b.I) / (a.I / a.R + b.I / b.R);
    return c;
}
/* "can fit within an execution round"; SPEC:136 incl. slots */
static bool pair_fits(const OrGpu& g, const Prof& a, const Prof& b) {
    return a.H + b.H <= g.shm_per_sm && a.G + b.G <= g.regs_per_sm && a.W + b.W <= g.warps_per_sm &&
           a.Bk + b.Bk <= g.blocks_per_sm;
}
/* ScoreGen body, fixed order: shm, reg, warp, bonus. */
static double pair_score(const OrGpu& g, const Prof& a, const Prof& b) {
    double S = 0.0; /* L19: S[i][j] starts at 0 */
    S += std::max(((double)((int64_t)g.shm_per_sm - (int64_t)a.H - (int64_t)b.H)) / (double)g.shm_per_sm, 0.0);
    S += std::max(((double)((int64_t)g.regs_per_sm - (int64_t)a.G - (int64_t)b.G)) / (double)g.regs_per_sm, 0.0);
    S += std::max(((double)((int64_t)g.warps_per_sm - (int64_t)a.W - (int64_t)b.W)) / (double)g.warps_per_sm, 0.0);
    double RB = (double)g.rb_num / (double)g.rb_den;
    if ((a.R <= RB && RB <= b.R) || (b.R <= RB && RB <= a.R)) { /* PAPER:165 (inclusive, L18) */
        double Rc = (a.I + b.I) / (a.I / a.R + b.I / b.R);
        S += std::max(1.0 - std::fabs(Rc - RB) / RB, 0.0);
    }
    return S;
}

static void heuristic(const OrGpu& g, const OrKernel* k, int n, int* order_out, int* round_of_out) {
    std::vector<Prof> P;
    for (int i = 0; i < n; i++) P.push_back(footprint(g, k[i]));
    std::vector<int> remaining;
    for (int i = 0; i < n; i++) remaining.push_back(i);
    std::vector<std::vector<int>> rounds;
    while (!remaining.empty()) {
        if (remaining.size() == 1) { /* a lone kernel is a singleton round */
            rounds.push_back({remaining[0]});
            remaining.clear();
            break;
        }
        /* line 5: highest-scoring feasible pair; strict > in scan order
         * a<b ascending so the lexicographically first pair wins ties. */
        int ba = -1, bb = -1;
        double bs = 0.0;
        for (size_t x = 0; x < remaining.size(); x++)
            for (size_t y = x + 1; y < remaining.size(); y++) {
                int a = remaining[x], b = remaining[y];
                if (!pair_fits(g, P[a], P[b])) continue; /* infeasible never chosen */
                double s = pair_score(g, P[a], P[b]);
                if (ba < 0 || s > bs) { ba = a; bb = b; bs = s; }
            }
        if (ba < 0) { /* no feasible pair -> singletons by decreasing shm */
            std::vector<int> rest = remaining;
            std::stable_sort(rest.begin(), rest.end(), [&](int x, int y) { return P[x].H > P[y].H; });
            for (int x : rest) rounds.push_back({x});
            remaining.clear();
            break;
        }
        /* line 6: push pair in decreasing N_shm; tie -> lower index first */
        std::vector<int> rd;
        if (P[bb].H > P[ba].H) rd = {bb, ba};
        else rd = {ba, bb};
        remaining.erase(std::find(remaining.begin(), remaining.end(), ba));
        remaining.erase(std::find(remaining.begin(), remaining.end(), bb));
        Prof comb = combine(P[ba], P[bb]); /* line 7 */
        while (true) {                     /* lines 8-12 */
            int bc = -1;
            double cs = 0.0;
            for (int c : remaining) {
                if (!pair_fits(g, comb, P[c])) continue;
                double s = pair_score(g, comb, P[c]);
                if (bc < 0 || s > cs) { bc = c; cs = s; }
            }
            if (bc < 0) break;
            /* line 10 "(Sort by N_shm_c, N_shm_comb)" — reading L17: stable
             * insertion keeping the round in non-increasing member N_shm. */
            size_t pos = 0;
            while (pos < rd.size() && P[rd[pos]].H >= P[bc].H) pos++;
            rd.insert(rd.begin() + (long)pos, bc);
            comb = combine(comb, P[bc]); /* line 11 */
            remaining.erase(std::find(remaining.begin(), remaining.end(), bc));
        }
        rounds.push_back(rd);
    }
    /* Output: launch order Rd_1 .. Rd_r */
    int j = 0;
    for (size_t r = 0; r < rounds.size(); r++)
        for (int x : rounds[r]) {
            order_out[j] = x;
            if (round_of_out) round_of_out[j] = (int)r;
            j++;
        }
}

/* ===================== C ABI for the Python test harness =================== */
extern "C" {

int or_check_inputs(const uint32_t* gpu8, const uint32_t* kern, int n) {
    return check_inputs(*(const OrGpu*)gpu8, (const OrKernel*)kern, n);
}

void or_unrank(uint64_t idx, int n, int* order) { unrank(idx, n, order); }
uint64_t or_rank(const int* order, int n) { return rank_of(order, n); }
uint64_t or_factorial(int n) { return factorial(n); }

/* rounds_out: max_rounds x n row-major (p[r][i]); trace_out: 2*sum(T) int32
 * (round, sm) per block in dispatch order.  Both nullable. */
int or_simulate(const uint32_t* gpu8, const uint32_t* kern, int n, const int* order, uint32_t* rounds_out,
                int max_rounds, int* n_rounds, uint64_t* key_lo, uint64_t* key_hi, double* t_naive,
                int32_t* trace_out) {
    const OrGpu& g = *(const OrGpu*)gpu8;
    const OrKernel* k = (const OrKernel*)kern;
    int e = check_inputs(g, k, n);
    if (e) return e;
    SimOut out;
    std::vector<int32_t> trace;
    simulate(g, k, n, order, out, true, trace_out ? &trace : nullptr);
    if (n_rounds) *n_rounds = (int)out.rounds.size();
    if (rounds_out) {
        if ((int)out.rounds.size() > max_rounds) return OR_EINVAL;
        for (size_t r = 0; r < out.rounds.size(); r++)
            for (int i = 0; i < n; i++) rounds_out[r * n + i] = out.rounds[r][i];
    }
    if (trace_out) std::memcpy(trace_out, trace.data(), trace.size() * sizeof(int32_t));
    *key_lo = (uint64_t)out.key;
    *key_hi = (uint64_t)(out.key >> 64);
    *t_naive = out.t_naive;
    return OR_OK;
}

/* Sweep [first, first+count) with `threads` contiguous chunks merged in order. */
int or_sweep(const uint32_t* gpu8, const uint32_t* kern, int n, uint64_t first, uint64_t count, uint64_t cand_key,
             int threads, uint64_t* stats8, uint64_t* keys_out, double* max_rel_err) {
    const OrGpu& g = *(const OrGpu*)gpu8;
    const OrKernel* k = (const OrKernel*)kern;
    int e = check_inputs(g, k, n);
    if (e) return e;
    if (n < 1 || first + count > factorial(n)) return OR_EINVAL;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > count) threads = count ? (int)count : 1;
    std::vector<ChunkResult> res((size_t)threads);
    std::vector<std::thread> th;
    uint64_t base = count / threads, extra = count % threads, off = first;
    for (int t = 0; t < threads; t++) {
        uint64_t c = base + ((uint64_t)t < extra ? 1 : 0);
        uint64_t* ko = keys_out ? keys_out + (off - first) : nullptr;
        th.emplace_back(sweep_chunk, std::cref(g), k, n, off, c, cand_key, ko, std::ref(res[(size_t)t]));
        off += c;
    }
    for (auto& t : th) t.join();
    ChunkResult m{};
    bool any = false;
    double err = 0.0;
    for (auto& r : res) { /* in-order merge: earlier chunk wins ties (smallest idx) */
        if (r.err) return r.err;
        if (r.evaluated == 0) continue;
        if (!any || r.kmin < m.kmin) { m.kmin = r.kmin; m.argmin = r.argmin; }
        if (!any || r.kmax > m.kmax) { m.kmax = r.kmax; m.argmax = r.argmax; }
        m.n_lt += r.n_lt;
        m.n_eq += r.n_eq;
        m.n_gt += r.n_gt;
        m.evaluated += r.evaluated;
        err = std::max(err, r.max_rel_err);
        any = true;
    }
    stats8[0] = (uint64_t)m.kmin;
    stats8[1] = (uint64_t)m.kmax;
    stats8[2] = m.argmin;
    stats8[3] = m.argmax;
    stats8[4] = m.n_lt;
    stats8[5] = m.n_eq;
    stats8[6] = m.n_gt;
    stats8[7] = m.evaluated;
    if (max_rel_err) *max_rel_err = err;
    return OR_OK;
}

/* Keys of explicit indices (parity samples): keys_out[i] = K(unrank(idx[i])),
 * the same O2 + O3 + O4 as or_sweep, split over `threads` contiguous chunks. */
static void keys_chunk(const OrGpu& g, const OrKernel* k, int n, const uint64_t* idx, uint64_t count,
                       uint64_t* keys_out, int* err) {
    std::vector<int> order(n);
    SimOut out;
    for (uint64_t i = 0; i < count; i++) {
        unrank(idx[i], n, order.data());
        simulate(g, k, n, order.data(), out, false, nullptr);
        if ((out.key >> 64) != 0) {
            *err = OR_EOVERFLOW;
            return;
        }
        keys_out[i] = (uint64_t)out.key;
    }
}

int or_keys_of(const uint32_t* gpu8, const uint32_t* kern, int n, const uint64_t* idx, uint64_t count, int threads,
               uint64_t* keys_out) {
    const OrGpu& g = *(const OrGpu*)gpu8;
    const OrKernel* k = (const OrKernel*)kern;
    int e = check_inputs(g, k, n);
    if (e) return e;
    const uint64_t N = factorial(n);
    for (uint64_t i = 0; i < count; i++)
        if (idx[i] >= N) return OR_EINVAL;
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > count) threads = count ? (int)count : 1;
    std::vector<int> errs((size_t)threads, 0);
    std::vector<std::thread> th;
    uint64_t base = count / threads, extra = count % threads, off = 0;
    for (int t = 0; t < threads; t++) {
        uint64_t c = base + ((uint64_t)t < extra ? 1 : 0);
        th.emplace_back(keys_chunk, std::cref(g), k, n, idx + off, c, keys_out + off, &errs[(size_t)t]);
        off += c;
    }
    for (auto& t : th) t.join();
    for (int x : errs)
        if (x) return x;
    return OR_OK;
}

/* O7: equal-width bins over [kmin, kmax]; if kmax == kmin all in
 * bin 0; else bin = min(B-1, floor((K-kmin)*B/(kmax-kmin))) in 128-bit ints.
 * hist is accumulated (+=). */
int or_histogram(const uint64_t* keys, uint64_t count, uint64_t kmin, uint64_t kmax, int bins, uint64_t* hist) {
    if (bins < 1 || kmax < kmin) return OR_EINVAL;
    for (uint64_t i = 0; i < count; i++) {
        uint64_t K = keys[i];
        if (K < kmin || K > kmax) return OR_EINVAL;
        uint64_t b;
        if (kmax == kmin) b = 0;
        else {
            u128 num = (u128)(K - kmin) * (u128)(uint64_t)bins;
            b = (uint64_t)(num / (u128)(kmax - kmin));
            if (b > (uint64_t)(bins - 1)) b = (uint64_t)(bins - 1);
        }
        hist[b]++;
    }
    return OR_OK;
}

int or_heuristic(const uint32_t* gpu8, const uint32_t* kern, int n, int* order_out, int* round_of_out) {
    const OrGpu& g = *(const OrGpu*)gpu8;
    const OrKernel* k = (const OrKernel*)kern;
    int e = check_inputs(g, k, n);
    if (e) return e;
    heuristic(g, k, n, order_out, round_of_out);
    return OR_OK;
}

/* ScoreGen / ProfileCombine on two single kernels (for SPEC example pins). */
int or_pair_score(const uint32_t* gpu8, const uint32_t* kern, int i, int j, int* feasible, double* score,
                  double* r_comb) {
    const OrGpu& g = *(const OrGpu*)gpu8;
    const OrKernel* k = (const OrKernel*)kern;
    Prof a = footprint(g, k[i]), b = footprint(g, k[j]);
    *feasible = pair_fits(g, a, b) ? 1 : 0;
    *score = *feasible ? pair_score(g, a, b) : 0.0;
    *r_comb = combine(a, b).R;
    return OR_OK;
}

/* C5-style batch: for each set, Algorithm 1 order -> its key -> full sweep.
 * Sets are distributed over threads; each set is evaluated single-threaded.
 * out per set: stats8 (8 u64) + cand_index + cand_key (10 u64 total). */
int or_sweep_sets(const uint32_t* gpu8, const uint32_t* kern, int n, int n_sets, int threads, uint64_t* out10) {
    const OrGpu& g = *(const OrGpu*)gpu8;
    const OrKernel* all = (const OrKernel*)kern;
    for (int s = 0; s < n_sets; s++) {
        int e = check_inputs(g, all + (size_t)s * n, n);
        if (e) return e;
    }
    if (threads < 1) threads = 1;
    std::vector<int> errs((size_t)threads, 0);
    auto work = [&](int t) {
        std::vector<int> order(n);
        for (int s = t; s < n_sets; s += threads) {
            const OrKernel* k = all + (size_t)s * n;
            heuristic(g, k, n, order.data(), nullptr);
            SimOut so;
            simulate(g, k, n, order.data(), so, false, nullptr);
            if ((so.key >> 64) != 0) { errs[(size_t)t] = OR_EOVERFLOW; return; }
            ChunkResult r;
            sweep_chunk(g, k, n, 0, factorial(n), (uint64_t)so.key, nullptr, r);
            if (r.err) { errs[(size_t)t] = r.err; return; }
            uint64_t* o = out10 + (size_t)s * 10;
            o[0] = (uint64_t)r.kmin; o[1] = (uint64_t)r.kmax; o[2] = r.argmin; o[3] = r.argmax;
            o[4] = r.n_lt; o[5] = r.n_eq; o[6] = r.n_gt; o[7] = r.evaluated;
            o[8] = rank_of(order.data(), n);
            o[9] = (uint64_t)so.key;
        }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < threads; t++) th.emplace_back(work, t);
    for (auto& t : th) t.join();
    for (int e : errs)
        if (e) return e;
    return OR_OK;
}

} /* extern "C" */
