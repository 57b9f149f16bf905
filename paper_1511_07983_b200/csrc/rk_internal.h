/* rk_internal.h — tables and launchers shared by rk_host.cpp and rk_kernels.cu
 * (product path only; the oracle never includes this).
 *
 * Device state layout: each SM's free resources are packed in
 * two u32 words, every field stored as 2*x+1 (odd encoding) so that
 * floor(x/d) = floor((2x+1)/(2d)) is one IMAD.HI with a host-verified magic:
 *   fa = (2*regs+1)  | (2*shm+1)   << 16
 *   fb = (2*warps+1) | (2*slots+1) << 16
 * A block of kernel k subtracts dA = 2*dr | 2*ds << 16 and dB = 2*dw | 2 << 16.
 * Register and shared-memory quantities are divided by their gcd over the GPU
 * capacity and all kernel demands first (exact: fit tests are scale-free).
 *
 * Symmetry reduction: with g = gcd(N_SM, N_tblk_1..n), every run of equal SMs
 * in ring order from the cursor has a length that is a multiple of g, so the
 * model on (N_SM, N_tblk_i, A_i, M_i) is the model on (N_SM/g, N_tblk_i/g,
 * g*A_i, g*M_i) with identical exact keys.
 */
#ifndef RK_INTERNAL_H
#define RK_INTERNAL_H

#include <stdint.h>
#include <vector_types.h>
#include "rk.h"

#define RK_MAX_N 16
#define RK_SMAX 32

struct RkKTab {        /* one kernel; 72 B */
    uint32_t T;        /* N_tblk */
    uint32_t mr, ms, mw;   /* magic multipliers for floor((2x+1)/(2d)); 0xFFFFFFFF if d == 0 */
    uint32_t zr;           /* regs numerator OR-mask: 0, or 0x7FFF0000 if d == 0 (quotient >> any cap) */
    uint32_t zs;           /* shm numerator high word for the funnel shift: 0, or 0x7FFF if d == 0 */
    uint32_t scm;          /* magic for floor(x / SC), exact for x < T; 0 = use a division */
    uint32_t dA, dB;       /* per-block decrement of fa / fb */
    uint32_t C;            /* blocks per fresh SM */
    uint32_t SC;           /* S * C: blocks per full single-kernel round */
    uint32_t pad;
    uint64_t cA, cM;       /* den * A_i and num * M_i (scaled per-block work, exact) */
    uint64_t fullkey;      /* max(SC*cA, SC*cM): key of one full round */
};

struct RkGTab {
    uint32_t S;            /* super-SMs: N_SM / blkscale (DESIGN.md §5 symmetry reduction) */
    uint32_t blkscale;     /* g = gcd(N_SM, all N_tblk): SMs per super-SM, blocks per super-block */
    uint32_t num, den;     /* R_B = num / den */
    uint32_t freshA, freshB;   /* packed words of a fresh SM */
    uint32_t smagic;       /* ceil(2^32 / S) */
    uint32_t tbits;        /* highest power of two <= max_blocks_per_sm (binary search) */
    uint32_t n;            /* number of kernels */
    uint32_t flags;        /* RK_FLAG_* model-reading policy */
    uint64_t fact[RK_MAX_N + 1];
};

struct RkTables {
    RkGTab g;
    RkKTab k[RK_MAX_N];
};

/* Variant selector bit on the S argument of the launchers: the model-reading
 * policy kernels (RK_FLAG_STRICT_RR / RK_FLAG_SKIP_AHEAD; per-order
 * simulation on the register state, S' <= 32). */
constexpr uint32_t RK_S_POLICY = 0x40000000u;

/* ---- launchers (rk_kernels.cu); return cudaError_t as int -------------- */
int rk_launch_eval(const RkTables* tab_dev, uint32_t n, uint32_t S, uint64_t first, uint64_t count,
                   const uint64_t* cand_key_dev, uint64_t cand_key_imm, rk_stats* stats_dev, uint64_t* keys_dev,
                   rk_stats* scratch_recs, uint32_t* scratch_counter, uint32_t max_ctas, void* stream,
                   uint32_t* launches, uint32_t* keys32_dev = nullptr, uint64_t key_base = 0,
                   uint32_t* ovf_dev = nullptr, const rk_stats* hist_range = nullptr, uint32_t bins = 0,
                   uint64_t* hist_dev = nullptr);
int rk_launch_range_histogram32(const uint32_t* keys_dev, uint64_t count, uint64_t key_base, uint64_t lo,
                                uint64_t span, uint32_t bins, uint64_t* hist_dev, void* stream, uint32_t* launches);
int rk_launch_histogram32(const uint32_t* keys_dev, uint64_t count, uint64_t key_base, const rk_stats* range_dev,
                          uint32_t bins, uint64_t* hist_dev, void* stream, uint32_t* launches);
int rk_launch_merge(const rk_stats* in_dev, uint32_t n_records, rk_stats* out_dev, void* stream, uint32_t* launches);
int rk_launch_histogram(const uint64_t* keys_dev, uint64_t count, uint64_t kmin, uint64_t kmax,
                        const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, void* stream,
                        uint32_t* launches);
int rk_launch_range_histogram(const uint64_t* keys_dev, uint64_t count, uint64_t lo, uint64_t span, uint32_t bins,
                              uint64_t* hist_dev, void* stream, uint32_t* launches);
/* keys of explicit indices (1 thread each): out_dev[i] = key(idx_dev[i]) of set (set_dev ? set_dev[i] : 0) */
int rk_launch_keys_of(const RkTables* tabs_dev, uint32_t n, uint32_t S, const uint64_t* idx_dev,
                      uint32_t m, uint64_t* out_dev, void* stream, uint32_t* launches);
int rk_launch_keys_of_same(const RkTables* tab_dev, uint32_t S, const uint64_t* idx_dev, uint32_t m,
                           uint64_t* out_dev, void* stream, uint32_t* launches);
int rk_launch_key_of_index(const RkTables* tab_dev, uint32_t S, uint64_t index, uint64_t* out_dev, void* stream,
                           uint32_t* launches);
/* one order -> rounds partition (1 thread) */
int rk_launch_simulate(const RkTables* tab_dev, uint32_t n, uint32_t S, const int32_t* order_dev,
                       uint32_t* rounds_dev, uint32_t max_rounds, uint32_t* n_rounds_dev, uint64_t* key_dev,
                       void* stream, uint32_t* launches);
/* batch: tabs_dev[n_sets]; per-set candidate keys (device); per-set records out */
int rk_launch_batch(const RkTables* tabs_dev, uint32_t n, uint32_t S, uint32_t n_sets, const uint64_t* cand_keys_dev,
                    rk_stats* out_dev, rk_stats* scratch_recs, uint32_t chunks_per_set, void* stream,
                    uint32_t* launches);
/* Algorithm 1 on the device, one thread per set */
int rk_launch_heuristic(const rk_kernel* sets_dev, uint32_t n, uint32_t n_sets, const rk_gpu_params* p,
                        int32_t* orders_dev, uint64_t* index_dev, void* stream, uint32_t* launches);
int rk_batch_chunks_per_set(uint32_t n, uint32_t S);
/* memoised batch: 6 <= n <= 9 on S' <= 2 (one CTA per set, persistent grid;
 * scratch = rk_batch_memo_scratch(S, grid) bytes of device memory) */
bool rk_batch_memo_ok(uint32_t n, uint32_t S);
int rk_batch_memo_grid(uint32_t S, uint32_t n_sets);
size_t rk_batch_memo_scratch(uint32_t n, uint32_t S, uint32_t grid);
int rk_launch_batch_memo(const RkTables* tabs_dev, uint32_t n, uint32_t S, uint32_t n_sets,
                         const uint64_t* cand_keys_dev, rk_stats* out_dev, void* scratch, uint32_t grid, void* stream,
                         uint32_t* launches);
int rk_eval_max_ctas(uint32_t S, int device);
/* branch-and-bound exact optimum: gb_dev = 48-B BnbGlobal (best seeded, rest 0),
 * recs_dev = 2*rk_bnb_ctas() u64 */
int rk_bnb_ctas();

/* Suffix memoisation: device tables of one plan */
struct DPView {
    const uint32_t* tid[RK_MAX_N]; /* level j transition: node id of level j+1, per (u, k) = u*n + k */
    const uint64_t* dk[RK_MAX_N];  /* closed-round key increment of that transition */
    const uint8_t* code;           /* level-P suffix keys as D! one-byte ranks into dv, per node */
    const void* dvc;               /* per node: sorted distinct suffix keys with multiplicities, 16 B each (D! slots) */
    const uint2* dvp;              /* the same distinct keys as {offset from the row minimum (exact unless nd bit 31), count} */
    const uint32_t* offs;          /* per node: the low 32 bits of the D! suffix keys (offset from the row minimum =
                                      offs - low32(min) mod 2^32, exact unless nd bit 31) */
    const uint32_t* nd;            /* per node: number of distinct suffix keys */
    const uint64_t* fst;           /* per node: min, max, argmin sigma, argmax sigma */
    uint32_t P, D, Dfact;
};
constexpr uint32_t RK_DP_D = 5; /* suffix depth: 120 keys per level-P node */
uint32_t rk_dp_node_bytes(uint32_t S);
/* one prefix-expansion level (entries {node, mask, K lo, hi} as uint4) */
struct RkExpand {
    const void* Rj;
    uint64_t aj;
    void* Rn;
    uint64_t an, cnt;
    uint32_t j;
    const uint32_t* tid;
    const uint64_t* dk;
};
/* one level of the table build: level j's nodes (Uj, *cnt_j; nullptr = the fresh root) x their nrem
 * unused kernels into level j+1 (Un, *cnt_n, capacity cap_n, hash table table/tmask, transitions tid/dk,
 * overflow flag ovf); work = items for grid sizing; ex = the range's level j-1 -> j expansion (nullable) */
struct RkLevel {
    const void* Uj;
    const uint32_t* cnt_j;
    void* Un;
    uint32_t* cnt_n;
    uint32_t cap_n;
    uint32_t* table;
    uint32_t tmask;
    uint32_t* tid;
    uint64_t* dk;
    uint32_t* ovf;
    const RkExpand* ex;
    uint32_t nrem;
    uint64_t work;
};
/* nl consecutive levels: one launch for nl == 1, one cooperative launch (grid barriers between levels)
 * for 1 < nl <= 8 */
int rk_dp_levels(const RkTables* tab, uint32_t S, const RkLevel* lv, uint32_t nl, void* stream, uint32_t* launches);
/* the first nl (<= 4) levels in one CTA (shared-memory dedup, deterministic ids); each level's live children
 * must number <= items_max = rk_dp_small_items_max(S) (0: not available for S) */
uint32_t rk_dp_small_items_max(uint32_t S);
int rk_dp_small_levels(const RkTables* tab, uint32_t S, const RkLevel* lv, uint32_t nl, uint32_t items_max,
                       void* stream, uint32_t* launches);
/* the 24 suffix keys of every level-(P+1) node (row24: nodes x 24 u64) */
int rk_dp_row24(const RkTables* tab, uint32_t S, const void* U, const uint32_t* cnt, uint64_t* row24, uint64_t nodes,
                void* stream, uint32_t* launches);
/* the level-P suffix rows from the level-P transitions and row24 */
int rk_dp_suffix(const RkTables* tab, uint32_t S, const void* UP, const uint32_t* cnt_P, const uint32_t* tidP,
                 const uint64_t* dkP, const uint64_t* row24, uint8_t* code, void* dvc, void* dvp, uint32_t* nd,
                 uint64_t* fst, uint32_t* offs, uint64_t nodes, void* stream, uint32_t* launches);
uint32_t rk_dp_max_fused_bins();
/* race audit of level (U, cnt) and its hash table + the previous level's
 * transitions; bad = 6 zeroed u64 counters (rk_dp_audit_kernel) */
int rk_dp_audit(uint32_t S, const void* U, const uint32_t* cnt, uint32_t cap, const uint32_t* table, uint32_t tmask,
                const uint32_t* tid_prev, uint64_t work_prev, const void* Uprev, uint32_t n, unsigned long long* bad,
                void* stream);
/* a range's row multiset: 16-B open-addressing slots of the
 * distinct rows (node | wide << 31, Kb) with 8 multiplicity counters each;
 * slot (nullptr: none) and mult must be zeroed and *nlist = 0 before pass 1;
 * list (>= runs entries) takes the runs that are not in a slot (range edges,
 * probe overflow); list_hint = an upper bound of *nlist for grid sizing */
struct RkRows {
    void* slot;
    uint32_t* mult;
    uint32_t mask;
    uint32_t* list;
    uint32_t* nlist;
    uint64_t list_hint;
    uint32_t* minrun; /* per slot: smallest run offset of the row (0xFFFFFFFF before pass 1) */
    void* wlist;       /* weighted rows that found no slot: uint4 {node, m, K_closed lo, hi} */
    uint32_t* wminrun; /* their smallest run offsets */
    uint32_t* nwlist;  /* device counter (zeroed before pass 1) */
};
/* the row multiset from the range's last stored expansion level (lastexp: level P-1 -> P, its Rj = the level-(P-1)
 * prefixes): parents multiset, then the children into rows (both zeroed before; minrun 0xFF) */
int rk_dp_multiset(uint32_t n, uint64_t first, uint64_t count, const RkExpand* lastexp, const RkRows& parents,
                   const RkRows& rows, void* stream, uint32_t* launches);
/* pass 1's run pass: per run of the range its (node, K_closed) into meta_u /
 * meta_K, and the row multiset (rows.slot nullable); last = the range's level
 * P-1 -> P expansion (nullptr: walk).  Needs the levels only (runs beside the
 * suffix rows). */
int rk_dp_runs(const RkTables* tab, const DPView& v, uint64_t first, uint64_t count, uint32_t* meta_u,
               uint64_t* meta_K, const RkRows& rows, const RkExpand* last, void* stream, uint32_t* launches);
/* pass 1's extremes (after the run pass and the suffix rows) from the row
 * multiset + run list (or every run without a multiset): the range's record
 * (counts: n_gt = evaluated = count) */
int rk_dp_ext(const DPView& v, uint64_t first, uint64_t count, const RkRows& rows, const uint32_t* meta_u,
              const uint64_t* meta_K, rk_stats* out, rk_stats* recs, uint32_t* counter, uint32_t max_ctas,
              void* stream, uint32_t* launches);
/* pass 2's counts (into rec, nullable) and histogram (nullable) from the row multiset */
int rk_dp_rows(const RkTables* tab, const DPView& v, uint64_t first, uint64_t count, const uint64_t* cand_dev,
               const rk_stats* range, uint32_t bins, uint64_t* hist, const RkRows& rows, const uint32_t* meta_u,
               const uint64_t* meta_K, rk_stats* rec, uint32_t max_ctas, void* stream, uint32_t* launches);
/* pass 2's compact key stream: u32 offsets from key_base; *ovf |= 1 (and no key written) when
 * range->key_max - key_base >= 2^32 */
int rk_dp_keys32(const DPView& v, uint64_t first, uint64_t count, const uint32_t* meta_u, const uint64_t* meta_K,
                 uint32_t* keys32, uint64_t key_base, uint32_t* ovf, const rk_stats* range, void* stream,
                 uint32_t* launches);
/* pass 2's key stream from the run metadata (one-shot grid) */
int rk_dp_keys(const DPView& v, uint64_t first, uint64_t count, const uint32_t* meta_u, const uint64_t* meta_K,
               uint64_t* keys, void* stream, uint32_t* launches);
int rk_launch_bnb(const RkTables* tab_dev, uint32_t S, uint32_t P, uint64_t n_units, void* gb_dev,
                  unsigned long long* recs_dev, void* stream, uint32_t* launches);

#endif
