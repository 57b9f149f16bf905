/*
 * rk.h — C ABI of librk, the B200-native (sm_100a) exhaustive evaluator of
 * kernel launch orders under the execution-round model of Li, Narayana &
 * El-Ghazawi, "Reordering GPU Kernel Launches to Enable Efficient Concurrent
 * Execution" (arXiv 1511.07983).
 *
 * Citations: PAPER:L = reference PAPER.md line L (section/table/algorithm
 * named); SPEC:L = reference SPEC.md line L.  The model readings (L1..L23)
 * are listed in DESIGN.md §3.
 *
 * Conventions (every entry point):
 *   - Returns rk_status; no exception or abort crosses the ABI.  On error the
 *     outputs are left untouched and rk_last_error(ctx) holds a message
 *     (owned by ctx, valid until the next call on that ctx).
 *   - The caller owns every host array; the library copies what it keeps.
 *     Device buffers (*_dev) are allocated by the caller (e.g. torch tensors)
 *     on the ctx's device; the library never frees them.
 *   - One ctx per host thread (no global mutable state).  The ctx owns its
 *     device tables and scratch; rk_destroy frees them.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  *_async
 *     calls only enqueue work; the synchronous calls return after the
 *     results are on the host.
 *   - There is no CPU fallback: every call that evaluates the model runs on
 *     the GPU and returns RK_ENODEVICE on a host-only ctx.
 */
#ifndef RK_H
#define RK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RK_OK = 0,
    RK_EINVAL = 1,         /* invalid argument / profile (SPEC:359 ValidationError)           */
    RK_EINFEASIBLE = 2,    /* a single block exceeds an SM limit      */
    RK_ETOOMANY = 3,       /* n > 16 (indices are u64, kernel ids 4-bit)       */
    RK_EMISSINGRATIO = 4,  /* mem_per_block == 0: R_i undefined                 */
    RK_EOVERFLOW = 5,      /* exact key bound sum_i T_i(den*A_i + num*M_i) >= 2^63            */
    RK_ESTATE = 6,         /* call order (params/kernels not set)                              */
    RK_ECUDA = 7,          /* CUDA runtime error (message in rk_last_error)                   */
    RK_ENODEVICE = 8,      /* compute call on a host-only ctx (rk_create(..., -1))            */
    RK_EUNSUPPORTED = 9    /* input outside the device fast path's packing     */
} rk_status;

typedef struct rk_ctx rk_ctx;

/* Create a context bound to CUDA device `cuda_device` (>= 0), or a host-only
 * context (cuda_device = -1) that can validate inputs and run Algorithm 1 but
 * returns RK_ENODEVICE for every model evaluation.  Testing switches, read once
 * here from the environment (every path computes the same exact keys):
 * RK_NO_REDUCE=1 (no SM-symmetry reduction), RK_FORCE_RUNS=1 (run-length SM
 * state for every S), RK_NO_MEMO=1 (direct per-order evaluation),
 * RK_FORCE_MEMO=1 (suffix memoisation even where it does not pay),
 * RK_ROW_DEDUP=0 (pass 2 counts every run instead of the distinct rows),
 * RK_OVERLAP=0 (the memoised step's side-stream work runs on the caller's
 * stream), RK_ROWS_CTAS=k (CTAs per SM of the side-stream counts/histogram),
 * RK_SIDE_PRIO=0|1 (both side streams at the default | high priority; by
 * default pass 1's is at the default and pass 2's at high priority).
 * RK_BATCH_TRACE=1 prints rk_eval_batch's host phase times on stderr. */
rk_status rk_create(rk_ctx** out, int cuda_device);
void rk_destroy(rk_ctx* ctx);
const char* rk_last_error(const rk_ctx* ctx);

/* GPU parameters, Table 1 top half: N_SM, N_reg_SM, N_shm_SM,
 * N_warp_SM, N_blk_SM, and the balanced inst/mem ratio R_B
 * as the exact rational rb_num / rb_den (reading L10; GTX580 preset
 * {16, 32768, 49152, 48, 8, 411, 100}).  All fields > 0
 * (SPEC:30-32); n_sm <= 65535, max_blocks_per_sm <= 255.  A reduced SM count
 * S' = n_sm / gcd(n_sm, grids) <= 32 runs on per-SM register state, a larger one
 * (e.g. the 148-SM B200 preset) on a run-length SM state.
 * Invalidates previously set kernels.  Errors: RK_EINVAL. */
typedef struct {
    uint32_t n_sm, regs_per_sm, shm_bytes_per_sm, max_warps_per_sm, max_blocks_per_sm;
    uint32_t rb_num, rb_den;
    uint32_t flags; /* model-reading policy, 0 = the readings of DESIGN.md §3 */
} rk_gpu_params;
/* flags bit: the round-robin cursor restarts at SM 0 for every kernel (the
 * alternative reading of L4; PAPER:76 only says "round-robin fashion"). */
#define RK_FLAG_CURSOR_PER_KERNEL 1u
/* flags bit: strict round robin — a block is offered to the SM under the
 * cursor only; if it does not fit there the round closes (L4 read literally:
 * PAPER:76 "mapped to SMs in a round-robin fashion, until any one of the SM
 * resource limitations is met"). */
#define RK_FLAG_STRICT_RR 2u
/* flags bit: skip-ahead — a kernel whose next block fits nowhere keeps its
 * remaining blocks for the next round while dispatch continues with the later
 * kernels in launch order; a round closes once every kernel with pending
 * blocks has been offered (the alternative of L5 that SPEC:262 rejects;
 * PAPER:80 "relegated to the next execution round").
 * STRICT_RR keeps the prefix state of L4 (only the placement rule differs) and
 * runs on every path of the register state (memoised step, direct kernel,
 * branch and bound, batch).  SKIP_AHEAD (with or without the other two) runs
 * on the per-order policy kernels: stats, keys, round partitions, candidates,
 * batches and the two-pass step; memoisation, branch and bound, compact keys
 * and the fused histogram return RK_EUNSUPPORTED.  STRICT_RR or SKIP_AHEAD
 * with a reduced SM count S' > 32 (run-length state) returns RK_EUNSUPPORTED
 * at rk_set_kernels (DESIGN.md §5 "Model-reading policies"). */
#define RK_FLAG_SKIP_AHEAD 4u
#define RK_FLAGS_POLICY (RK_FLAG_STRICT_RR | RK_FLAG_SKIP_AHEAD)
rk_status rk_set_gpu_params(rk_ctx* ctx, const rk_gpu_params* p);

/* Kernel profile, Table 1 bottom half:
 *   grid_blocks         N_tblk_i >= 1
 *   threads_per_block   1..1024; warps/block = ceil(tpb/32) (reading L7)
 *   regs_per_thread     registers/block = regs_per_thread * tpb (reading L6)
 *   shm_bytes_per_block
 *   inst_per_block      A_i = N_inst_i / N_tblk_i >= 1
 *   mem_per_block       M_i = A_i / R_i = 4*mem_events_i / N_tblk_i >= 1,
 *                       in instruction units
 * Per-block demand is used by the simulator, the per-SM footprint
 * (demand * ceil(N_tblk/N_SM)) by Algorithm 1 (reading L2). */
typedef struct {
    uint32_t grid_blocks, threads_per_block, regs_per_thread, shm_bytes_per_block;
    uint32_t inst_per_block, mem_per_block;
} rk_kernel;

/* Copy and validate n kernels (1 <= n <= 16) and upload the device tables.
 * Errors: RK_ESTATE (no gpu params), RK_EINVAL, RK_EINFEASIBLE,
 * RK_ETOOMANY, RK_EMISSINGRATIO, RK_EOVERFLOW, RK_EUNSUPPORTED, RK_ECUDA. */
rk_status rk_set_kernels(rk_ctx* ctx, const rk_kernel* k, uint32_t n);

/* Reduction record over an index range (Table 3 columns, PAPER:236;
 * SPEC:281-286).  Keys are exact: K = sum_r max(rb_den*I_r, rb_num*M_r) =
 * rb_den * T (O4), so T = K / rb_den.  argmin/argmax = smallest lexicographic
 * index attaining the extreme (reading L12).  n_lt/n_eq/n_gt count keys
 * below/equal/above the candidate key.  64 bytes, no padding. */
typedef struct {
    uint64_t key_min, key_max;
    uint64_t argmin, argmax;
    uint64_t n_lt, n_eq, n_gt;
    uint64_t evaluated;
} rk_stats;

/* Evaluate every launch order with lexicographic index in [first, first+count)
 * ("all possible kernel orderings (all permutations)"; order <->
 * index is the Lehmer code, reading L11): unrank, place all blocks
 * round-robin into execution rounds, score the rounds
 * and reduce.  first + count <= n!.
 *   candidate_key  key the counts compare against (e.g. from rk_heuristic_order)
 *   out_host       host rk_stats (synchronous call)
 *   keys_dev       nullable device u64[count]: key of index first+j at [j]
 * Errors: RK_ESTATE, RK_EINVAL, RK_ENODEVICE, RK_ECUDA. */
rk_status rk_eval_range(rk_ctx* ctx, uint64_t first, uint64_t count, uint64_t candidate_key,
                        rk_stats* out_host, uint64_t* keys_dev, void* stream);

/* Stream-ordered variant: the candidate key is read from device memory
 * (cand_key_dev, nullable = 0) and the record written to stats_dev (device).
 * Only enqueues. */
rk_status rk_eval_range_async(rk_ctx* ctx, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                              rk_stats* stats_dev, uint64_t* keys_dev, void* stream);

/* Second pass for spaces too large to keep keys (n >= 13: 13! keys = 50 GB):
 * re-evaluates [first, first+count) and bins every key straight into `bins`
 * Fig. 1 bins over [range_dev->key_min, key_max] (the first pass's global
 * record) in shared memory; hist_dev (device u64[bins]) is accumulated.  Also
 * writes the range's record to stats_dev (nullable).  1 <= bins <= 32768.
 * Only enqueues. */
rk_status rk_eval_range_hist_async(rk_ctx* ctx, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                                   rk_stats* stats_dev, const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev,
                                   void* stream);

/* Exact key of the single launch order with lexicographic index `index`,
 * written to key_dev (device u64).  Stream-ordered, no host sync (used for the
 * candidate order inside a device pipeline).  index < n!. */
rk_status rk_eval_index_async(rk_ctx* ctx, uint64_t index, uint64_t* key_dev, void* stream);

/* Compact-key variant: keys32_dev[j] = K(first+j) - key_base as
 * u32, halving the key traffic.  key_base must not exceed any key of the range
 * (e.g. rk_key_lower_bound).  If some K - key_base >= 2^32 the kernel ORs 1
 * into *ovf_dev (caller-zeroed u32) and that entry is truncated: re-run with
 * rk_eval_range_async.  Stats are exact either way.  Only enqueues. */
rk_status rk_eval_range32_async(rk_ctx* ctx, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                                rk_stats* stats_dev, uint32_t* keys32_dev, uint64_t key_base, uint32_t* ovf_dev,
                                void* stream);

/* Exact lower bound of every order's key for the current kernel set:
 * max(den*sum_i T_i A_i, num*sum_i T_i M_i) ("sum of maxima >= maximum
 * of sums").  Host only. */
rk_status rk_key_lower_bound(rk_ctx* ctx, uint64_t* lb_out);

/* Deterministic merge of n_records device records (e.g. all-gathered per-rank
 * records) into out_dev: min/max with smallest-index ties, counts summed.
 * The result is independent of record order.  Only enqueues. */
rk_status rk_merge_stats_async(rk_ctx* ctx, const rk_stats* in_dev, uint32_t n_records, rk_stats* out_dev,
                               void* stream);

/* Time histogram (Fig. 1): `bins` equal-width bins
 * over [kmin, kmax]; bin = min(bins-1, floor((K-kmin)*bins/(kmax-kmin))) in
 * exact integers; all keys in bin 0 when kmax == kmin.  hist_dev (device u64
 * [bins]) is ACCUMULATED (+=), so shards can be summed in place.  Keys outside
 * [kmin,kmax] are an error of the caller (counted in the nearest end bin).
 * Stream-ordered (returns after enqueueing).  1 <= bins <= 65536. */
rk_status rk_histogram(rk_ctx* ctx, const uint64_t* keys_dev, uint64_t count, uint64_t kmin, uint64_t kmax,
                       uint32_t bins, uint64_t* hist_dev, void* stream);
/* Same, with [kmin,kmax] read from a device record (range_dev->key_min/max). */
rk_status rk_histogram_async(rk_ctx* ctx, const uint64_t* keys_dev, uint64_t count, const rk_stats* range_dev,
                             uint32_t bins, uint64_t* hist_dev, void* stream);

/* rk_histogram_async over compact keys: K = key_base + keys32_dev[j]. */
rk_status rk_histogram32_async(rk_ctx* ctx, const uint32_t* keys32_dev, uint64_t count, uint64_t key_base,
                               const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, void* stream);

/* Order statistics over device keys (SPEC:299-302 SweepReport median = the
 * lower-middle element, rank (N-1)/2; Fig. 1 PAPER:204 "ranking" curve = keys
 * at chosen ranks).  keys_out[j] = the ranks[j]-th smallest (0-based) of
 * keys_dev[0..count); every key must lie in [kmin, kmax] (e.g. a record's
 * key_min/key_max).  Exact: iterated integer histograms over shrinking key
 * ranges.  Synchronous.  RK_EINVAL if a rank >= count. */
rk_status rk_select_keys(rk_ctx* ctx, const uint64_t* keys_dev, uint64_t count, uint64_t kmin, uint64_t kmax,
                         const uint64_t* ranks, uint32_t m, uint64_t* keys_out, void* stream);
/* Building block of sharded selection: hist_dev[b] += #{keys in [lo, lo+span) with
 * floor((K-lo)*bins/span) = b} (half-open equal bins, keys outside ignored).
 * span >= 1, 1 <= bins <= 65536.  Stream-ordered. */
rk_status rk_range_histogram(rk_ctx* ctx, const uint64_t* keys_dev, uint64_t count, uint64_t lo, uint64_t span,
                             uint32_t bins, uint64_t* hist_dev, void* stream);

/* The same two calls over compact keys K = key_base + keys32_dev[j]. */
rk_status rk_select_keys32(rk_ctx* ctx, const uint32_t* keys32_dev, uint64_t key_base, uint64_t count, uint64_t kmin,
                           uint64_t kmax, const uint64_t* ranks, uint32_t m, uint64_t* keys_out, void* stream);
rk_status rk_range_histogram32(rk_ctx* ctx, const uint32_t* keys32_dev, uint64_t key_base, uint64_t count,
                               uint64_t lo, uint64_t span, uint32_t bins, uint64_t* hist_dev, void* stream);

/* Algorithm 1 (readings L2, L16-L19), on the
 * host (sequential by nature).  order_out[n] = launch order Rd_1..Rd_r
 * (PAPER:134); round_of_out[n] (nullable) = round of each position;
 * index_out (nullable) = its lexicographic index; key_out (nullable) = its
 * exact key, evaluated on the device (RK_ENODEVICE on a host-only ctx). */
rk_status rk_heuristic_order(rk_ctx* ctx, int32_t* order_out, int32_t* round_of_out, uint64_t* index_out,
                             uint64_t* key_out);

/* Algorithm 1 for n_sets independent kernel sets on the device (SURVEY §8(f)
 * f4), one thread per set, bit-identical to rk_heuristic_order (same readings,
 * same explicitly rounded double operations).  orders_out (nullable host
 * int32[n_sets*n]) and index_out (host u64[n_sets]: lexicographic index).
 * Uses the ctx's gpu params.  Synchronous. */
rk_status rk_heuristic_batch(rk_ctx* ctx, const rk_kernel* sets, uint32_t n, uint32_t n_sets, int32_t* orders_out,
                             uint64_t* index_out, void* stream);

/* Percentile support (Table 3 "Percentile rank"):
 * key of `order` and the number of indices in [first, first+count) whose key
 * is >= it (ties count for the candidate, reading L13).  Shard-aware: sum
 * n_ge over shards and divide by n!.  Synchronous. */
rk_status rk_percentile(rk_ctx* ctx, const int32_t* order, uint64_t first, uint64_t count, uint64_t* n_ge_out,
                        uint64_t* key_out);

/* Batch mode (config C5): n_sets independent kernel sets of equal size n,
 * sets[s*n + i]; per set the full n! space is evaluated against that set's
 * candidate.  cand_index (nullable host u64[n_sets]): candidate indices; if
 * NULL, Algorithm 1 runs for each set on the device (as rk_heuristic_batch,
 * bit-identical to the host's).  out_host[n_sets] per-set records;
 * cand_key_out (nullable host u64[n_sets]).  Synchronous.  Every set is
 * validated as by rk_set_kernels (on up to 16 host threads); the lowest
 * failing set is reported as "set q: ...".  Sets with 6 <= n <= 9 on at most
 * two super-SMs run the memoised batch kernel (one CTA per set; runs whose
 * (n-5)-prefix states are equal share one 120-key suffix row, PAPER:79-80 /
 * SPEC:210), the others the direct one (RK_NO_MEMO=1: always direct); the
 * memoised kernel keeps a grow-only device scratch in the ctx of about
 * 1.1 KB x n!/120 per resident CTA (1.0 GB for n = 9 on a B200), freed by
 * rk_destroy.  Uses the ctx's gpu params; does not change the ctx's kernel
 * set. */
rk_status rk_eval_batch(rk_ctx* ctx, const rk_kernel* sets, uint32_t n, uint32_t n_sets, const uint64_t* cand_index,
                        rk_stats* out_host, uint64_t* cand_key_out, void* stream);

/* Round partition of one order (SPEC:209-219 PlacedRound), computed by the
 * device path: rounds_out (host u32[max_rounds*n], row-major p[r][i] = blocks
 * of kernel i placed in round r), n_rounds_out, key_out.  RK_EINVAL if the
 * order has more than max_rounds rounds (n_rounds_out still set). */
rk_status rk_simulate_order(rk_ctx* ctx, const int32_t* order, uint32_t* rounds_out, uint32_t max_rounds,
                            uint32_t* n_rounds_out, uint64_t* key_out);

/* The step of the hot path in two passes, so that N ranks can agree on the
 * histogram range in between.
 * Pass 1, rec_dev (64 B, device) <- the extremes of [first, first+count):
 * {key_min, key_max, argmin, argmax (smallest index on ties, reading L12),
 * n_lt = 0, n_eq = 0, n_gt = count, evaluated = count}.  With suffix
 * memoisation on (rk_memo_info) pass 1 rebuilds the memo tables
 * from scratch and takes the extremes from the rows' extremes run by run;
 * otherwise it is rk_eval_range_async (complete record, every key to
 * keys_dev).  N ranks all-gather their records and merge them
 * (rk_merge_stats_async) into the global record between the passes.
 * Pass 2 over the same range: adds the counts against *cand_key_dev (reading
 * L13) to rec_dev (n_lt, n_eq += ..., n_gt -= their sum; a zeroed record
 * collects them alone, to be merged with the extremes record), writes every
 * exact key to keys_dev (u64[count] index-major, nullable, 16-byte alignment
 * not required), and accumulates (+=) into hist_dev (u64[bins], nullable,
 * zeroed by the caller) the Fig. 1 histogram over [range_dev->key_min,
 * range_dev->key_max] (reading L14; range_dev = this rank's
 * record for one rank, the merged global record for N ranks).  Memoised: from
 * the tables of the preceding pass 1; otherwise, or for more than 32768 bins,
 * from keys_dev (then required).  Memoised, pass 2 streams pass 1's run
 * metadata: it must follow pass 1 over the same [first, first+count) on the
 * same ctx (else RK_ESTATE).  Pass 1 also builds the range's multiset of
 * distinct rows (node, K_closed) with multiplicities, from which pass 2
 * counts and bins (C4: 217,659 distinct rows for 3,991,680 runs).  Scratch:
 * ~36 B per run of D! = 120 indices (run metadata, multiset, lists), ctx-owned
 * and grow-only; rk_eval_range splits ranges of more than 2^26 runs itself,
 * callers of the two-pass API split theirs.
 * Errors: RK_EINVAL (range, missing pointers), RK_ESTATE, RK_ENODEVICE,
 * RK_ECUDA. */
rk_status rk_sweep_pass1_async(rk_ctx* ctx, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                               rk_stats* rec_dev, uint64_t* keys_dev, void* stream);
rk_status rk_sweep_pass2_async(rk_ctx* ctx, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                               const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, uint64_t* keys_dev,
                               rk_stats* rec_dev, void* stream);
/* Pass 2 with compact keys (memoised only): as rk_sweep_pass2_async, but every
 * key goes to keys32_dev (u32[count], index-major, caller-owned) as the exact
 * offset key - key_base, with key_base <= every key of the range (normally
 * rk_key_lower_bound: the exact lower bound of SPEC:255) — half the HBM bytes
 * of u64 keys, no information lost.  range_dev is required: when
 * range_dev->key_max >= key_base + 2^32 (some key would not fit), *ovf_dev (u32,
 * caller-zeroed) is set to 1 and no key is written: re-run pass 1 and pass 2
 * with u64 keys.  bins <= 32768.  Errors: as rk_sweep_pass2_async,
 * plus RK_EUNSUPPORTED without memoisation (rk_eval_range32_async is the
 * direct path's compact form). */
rk_status rk_sweep_pass2_32_async(rk_ctx* ctx, uint64_t first, uint64_t count, const uint64_t* cand_key_dev,
                                  const rk_stats* range_dev, uint32_t bins, uint64_t* hist_dev, uint32_t* keys32_dev,
                                  uint64_t key_base, uint32_t* ovf_dev, rk_stats* rec_dev, void* stream);

/* Per-phase device timing of the step (measurement support):
 * while on, every phase the library enqueues records a CUDA event pair on its
 * launching stream — RK_PHASE_TABLES (pass 1 memoised: levels + suffix rows
 * rebuilt, main stream), RK_PHASE_RUNS (pass 1 memoised: each run's node and
 * closed key + the row multiset, on the ctx's side stream beside the suffix
 * rows), RK_PHASE_EXTREMES (pass 1 memoised: the key stream's run metadata and
 * the range's extremes), RK_PHASE_STREAM (pass 2's key stream), RK_PHASE_HIST
 * (pass 2's counts and histogram from the row multiset), RK_PHASE_DIRECT (the
 * direct evaluation kernel of pass 1).
 * rk_timing_read synchronises on the recorded events and returns per phase the
 * summed milliseconds (ms_sum[p]) and the number of marks (counts[p]) since
 * the last read or rk_set_timing, for p < n_phases; then clears the marks.
 * Event objects are owned by the ctx (grow-only).  Errors: RK_EINVAL,
 * RK_ENODEVICE, RK_ECUDA. */
enum { RK_PHASE_TABLES = 0, RK_PHASE_STREAM = 1, RK_PHASE_HIST = 2, RK_PHASE_DIRECT = 3, RK_PHASE_EXTREMES = 4,
       RK_PHASE_RUNS = 5, RK_N_PHASES = 6 };
rk_status rk_set_timing(rk_ctx* ctx, int on);
rk_status rk_timing_read(rk_ctx* ctx, double* ms_sum, uint32_t* counts, uint32_t n_phases);

/* Suffix memoisation of the current kernel set: on_out = 1 when
 * the device path evaluates orders as K(prefix) + f(state, suffix) from
 * deduplicated prefix states (planned at rk_set_kernels; off for n < 6, for
 * more than 32 super-SMs, with RK_NO_MEMO=1, or when it would not pay).
 * levels_out = P (prefix length); nodes_out[j] (j <= P, up to max_levels) =
 * distinct (remaining set, state) pairs after j kernels. */
rk_status rk_memo_info(rk_ctx* ctx, uint32_t* on_out, uint32_t* levels_out, uint32_t* nodes_out, uint32_t max_levels);

/* Race audit of the memo tables built by the most recent pass 1 (diagnostic;
 * DESIGN.md §5 "lock-free hash tables"): checks every level's open-addressing
 * table and transitions on the device and returns 8 counters in out[8]:
 * [0] levels over capacity, [1] slots left BUSY, [2] published ids >= count,
 * [3] nodes not found first from their own hash (lost publish or duplicate
 * state), [4] transitions neither EMPTY nor a valid id, [5] levels whose
 * published slots != count, [6] levels whose count != the plan's count,
 * [7] nodes audited.  [0..6] are all 0 for a race-free build.  Synchronous.
 * Errors: RK_ESTATE (memoisation off or no pass 1 yet), RK_ENODEVICE, RK_ECUDA. */
rk_status rk_memo_audit(rk_ctx* ctx, uint64_t* out);

/* Exact optimum by branch and bound (the same (key_min,
 * argmin) as a full rk_eval_range over [0, n!) — SPEC:300, ties -> smallest
 * index — without enumerating n!).  Bound of a prefix (PAPER:79-81 round
 * time): K_closed + max(den*(I_open + sum_rem T*A), num*(M_open +
 * sum_rem T*M)); pruning is strict (bound > best) so every order with the
 * minimum key is visited.  seed_index: an order whose key seeds the bound
 * (e.g. Algorithm 1's rank), or UINT64_MAX for none.  Outputs (host, each
 * optional): order_out int32[n] (the argmin order), index_out, key_out (exact
 * scaled key K = den*T), nodes_out (placements performed; n! * n would be the
 * exhaustive count).  Synchronous on `stream`.  Run time depends on how tight
 * the bound is: worst case is the full tree. */
rk_status rk_best_order(rk_ctx* ctx, uint64_t seed_index, int32_t* order_out, uint64_t* index_out, uint64_t* key_out,
                        uint64_t* nodes_out, void* stream);

/* Lexicographic rank/unrank (factorial number system; reading L11). Pure host
 * helpers, no ctx.  1 <= n <= 20. RK_EINVAL on a non-permutation / idx >= n!. */
rk_status rk_rank(const int32_t* order, uint32_t n, uint64_t* idx_out);
rk_status rk_unrank(uint64_t idx, uint32_t n, int32_t* order_out);

/* Bytes of the packed device tables rk_set_kernels uploads (host -> device). */
uint32_t rk_table_bytes(void);

/* Number of kernel launches the last synchronous/async call enqueued on the
 * device (for the bench's gpu_launches count). */
uint32_t rk_last_launch_count(const rk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* RK_H */
