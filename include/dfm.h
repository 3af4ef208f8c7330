/*
 * dfm.h — C-ABI of the B200-native DFA-minimization engine (libdfm.so).
 *
 * The drop-in boundary for the reference's minimize path (arxiv 2410.22764,
 * `dfamin` headers).  Each entry point replaces one reference interface, cited
 * below as proj/include/dfamin/<file>:<line>.  Plain pointers and sizes only:
 * no torch/CUDA types appear in a signature (device pointers are `void*`).
 *
 * Conventions
 *  - Return value: DFM_OK or a dfm_err code for INFRASTRUCTURE faults (bad
 *    argument, CUDA/NCCL error, out of device memory); the message is in
 *    dfm_last_error(ctx).  ALGORITHMIC outcomes are reported like the
 *    reference, as a run status in dfm_stats.status (core.hpp:58):
 *    timeout / capacity_exceeded leave block_out untouched and set
 *    *num_blocks_out = 0 (the reference returns an empty partition,
 *    min_sort.hpp:94-99, min_transpr.hpp:95-101, min_trans.hpp:89-95).
 *    A CUDA error is never reported as a timeout.
 *  - dfm_expand_alphabet alone reports over-limit as DFM_ERR_CAPACITY with
 *    *required_bytes_out set: it mirrors the CapacityError the reference throws
 *    (min_transpr.hpp:63-67).
 *  - block_out receives the canonical partition (core.hpp:123-136: label b
 *    first occurs before label b+1), n entries, caller-owned.
 *  - Calls are synchronous from the caller's view.  One dfm_ctx per host
 *    thread (a ctx serialises its own calls with an internal mutex).
 *  - Host DFA rows are the reference's SoA layout: delta[a] points at the n
 *    successors on letter a (Dfa::delta[a].data(), core.hpp:24-33) — zero-copy.
 */
#ifndef DFM_H
#define DFM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFM_ABI_VERSION 2  /* 2: dfm_stats.executed_passes, sharded driver, LTS ingestion */

typedef enum {
  DFM_OK = 0,
  DFM_ERR_INVALID = 1,  /* malformed argument (the reference would throw invalid_argument) */
  DFM_ERR_CUDA = 2,     /* CUDA runtime / launch failure */
  DFM_ERR_CAPACITY = 3, /* dfm_expand_alphabet over max_memory_bytes (CapacityError) */
  DFM_ERR_NO_MEMORY = 4,/* device allocation failed */
  DFM_ERR_NO_DEVICE = 5,/* no sm_100 device / extension unusable: never silently falls back */
  DFM_ERR_PARSE = 6,    /* dfm_lts_parse: the reference's ParseError (ingest.hpp:20-28) */
  DFM_ERR_BUDGET = 7    /* dfm_determinize: SubsetBudgetExceeded (ingest.hpp:31-39) */
} dfm_err;

/* RunStatus, core.hpp:58 */
typedef enum { DFM_STATUS_OK = 0, DFM_STATUS_TIMEOUT = 1, DFM_STATUS_CAPACITY_EXCEEDED = 2 } dfm_run_status;

/* substrate::RacePolicy, substrate.hpp:24 */
typedef enum { DFM_POLICY_ARBITRARY = 0, DFM_POLICY_MIN = 1, DFM_POLICY_MAX = 2 } dfm_policy;

/* Algo, bench.hpp:23 (DFM_ALGO_ORACLE is the CPU Moore oracle: not provided by the
 * GPU engine, dfm_run_algorithm returns DFM_ERR_INVALID for it) */
typedef enum {
  DFM_ALGO_TRANS = 0,
  DFM_ALGO_NAIVE = 1,
  DFM_ALGO_NAIVE_CAS = 2,
  DFM_ALGO_SORT = 3,
  DFM_ALGO_TRANSPR = 4,
  DFM_ALGO_ORACLE = 5
} dfm_algo;

typedef struct dfm_ctx dfm_ctx;   /* device, stream, scratch arena */
typedef struct dfm_ddfa dfm_ddfa; /* a DFA resident in device memory */

/* Dfa, core.hpp:24-33 (host memory, borrowed) */
typedef struct {
  uint32_t num_states;
  uint32_t alphabet_size;
  const uint32_t* const* delta; /* alphabet_size row pointers, num_states entries each */
  const uint8_t* accepting;     /* num_states indicators */
  uint32_t initial;
} dfm_dfa;

/* RunStats, core.hpp:71-77 */
typedef struct {
  uint64_t iterations;     /* passes including the final no-change pass */
  uint64_t closure_steps;  /* alphabet-doubling rounds (transPR), else 0 */
  double elapsed_ms;       /* host steady clock around the whole call */
  uint64_t peak_memory_estimate; /* the reference's estimate formula */
  int32_t status;          /* dfm_run_status */
  /* passes whose kernels actually ran (<= iterations): a pass that starts with
   * every block a singleton can only confirm the fixpoint; it is counted, as the
   * reference counts it (min_sort.hpp:110), without being run */
  uint64_t executed_passes;
} dfm_stats;

/* Limits, core.hpp:81-84.  timeout_ms <= 0 disables the deadline. */
typedef struct {
  uint64_t max_memory_bytes; /* reference default 16 GiB */
  int64_t timeout_ms;        /* reference default 300000 */
} dfm_limits;

/* Per-pass trace (SortTrace min_sort.hpp:21-24, PrTrace min_partref.hpp:21-24):
 * called on the host after every pass with the engine's RAW labels for the
 * pass (block ids for sortPR, leader ids for naivePR) and the block count. */
typedef void (*dfm_pass_fn)(void* user, uint64_t pass, const uint32_t* raw_block, uint32_t n,
                            uint32_t num_blocks);
typedef struct {
  dfm_pass_fn on_pass;
  void* user;
} dfm_trace;

/* ---------------------------------------------------------------- context */
const char* dfm_version(void);
int dfm_ctx_create(int device, dfm_ctx** out);
void dfm_ctx_destroy(dfm_ctx* ctx);
const char* dfm_last_error(const dfm_ctx* ctx);
/* Use an external CUDA stream (cudaStream_t as void*); NULL restores the ctx's own.
 * The legacy default stream is passed as cudaStreamLegacy ((void*)0x1). */
int dfm_ctx_set_stream(dfm_ctx* ctx, void* stream);
/* sortPR grouping engine: both give the reference's partitions and pass
 * counts.  HASH (default): active states grouped through an open-addressing table;
 * RADIX: the paper's sort — onesweep LSD radix sort + look-back scans.  The
 * DFM_SORTPR_ENGINE=radix|hash environment variable sets the default per context. */
#define DFM_SORTPR_HASH 0
#define DFM_SORTPR_RADIX 1
int dfm_ctx_set_sortpr_engine(dfm_ctx* ctx, int engine);
/* Cho–Huynh squaring engine: AUTO (tensor cores for |V| >= 1024), BIT (packed 64-bit
 * rows on CUDA cores) or TENSOR (tcgen05 kind::i8 GEMM).  Same results. */
#define DFM_TRANS_AUTO 0
#define DFM_TRANS_BIT 1
#define DFM_TRANS_TENSOR 2
int dfm_ctx_set_trans_engine(dfm_ctx* ctx, int engine);
/* Output-ready hook for the NEXT host-buffer minimize call on this context (that call
 * consumes it; NULL clears it): the library calls ready(user) once — from one of its
 * threads, possibly while the GPU still works — before it first writes the caller's
 * partition buffer (block_out), and waits for it to return.  A caller can thus prepare
 * a fresh output buffer (fault its pages in) concurrently with the minimization; the
 * C++ layer (dfamin_b200.hpp) does this for the MinResult partition vector.  Not a
 * reference interface: the reference returns a freshly built std::vector. */
typedef void (*dfm_out_ready_fn)(void* user);
int dfm_ctx_set_out_ready_hook(dfm_ctx* ctx, dfm_out_ready_fn ready, void* user);
/* Record per-kernel CUDA-event timings for subsequent calls (bench/roofline). */
int dfm_ctx_set_profiling(dfm_ctx* ctx, int enabled);
/* Read back timing for a kernel family ("sig", "sort", "scan", "relabel", "elect",
 * "split", "double", "gemm", "propagate", "canon", ...): timed scopes, total ms and
 * total ALGORITHMIC bytes since the last reset; returns
 * DFM_ERR_INVALID for an unknown name. */
int dfm_profile_get(dfm_ctx* ctx, const char* name, uint64_t* scopes, double* total_ms,
                    uint64_t* algo_bytes);
/* Comma-separated list of the kernel families recorded so far. */
const char* dfm_profile_names(dfm_ctx* ctx);
int dfm_profile_reset(dfm_ctx* ctx);
/* Process-wide count of libdfm kernel launches so far (all contexts). */
uint64_t dfm_kernel_launches(void);
/* Bytes of device memory currently held by the ctx's scratch arena. */
uint64_t dfm_ctx_device_bytes(const dfm_ctx* ctx);

/* ---------------------------------------------------------------- host-buffer API */
/* sort_pr, min_sort.hpp:72 / :128 */
int dfm_sort_pr(dfm_ctx* ctx, const dfm_dfa* d, int64_t timeout_ms, const dfm_trace* trace,
                uint32_t* block_out, uint32_t* num_blocks_out, dfm_stats* stats);
/* naive_pr, min_partref.hpp:156 / :160 (policy = dfm_policy) */
int dfm_naive_pr(dfm_ctx* ctx, const dfm_dfa* d, int32_t policy, int64_t timeout_ms,
                 const dfm_trace* trace, uint32_t* block_out, uint32_t* num_blocks_out,
                 dfm_stats* stats);
/* naive_pr_cas, min_partref.hpp:170 */
int dfm_naive_pr_cas(dfm_ctx* ctx, const dfm_dfa* d, int64_t timeout_ms, const dfm_trace* trace,
                     uint32_t* block_out, uint32_t* num_blocks_out, dfm_stats* stats);
/* power_levels / expand_required_bytes, min_transpr.hpp:21-27 */
uint32_t dfm_power_levels(uint32_t n);
uint64_t dfm_expand_required_bytes(uint32_t n, uint32_t k);
/* expand_alphabet, min_transpr.hpp:59.  rows_out: levels*k*n u32 (row lvl*k+a holds
 * a^(2^lvl)); may be NULL to query *levels_out / *required_bytes_out only. */
int dfm_expand_alphabet(dfm_ctx* ctx, const dfm_dfa* d, uint64_t max_memory_bytes,
                        uint32_t* rows_out, uint32_t* levels_out, uint64_t* required_bytes_out);
/* trans_pr, min_transpr.hpp:90 / :114 */
int dfm_trans_pr(dfm_ctx* ctx, const dfm_dfa* d, int32_t policy, const dfm_limits* limits,
                 uint32_t* block_out, uint32_t* num_blocks_out, dfm_stats* stats);
/* trans_required_bytes, min_trans.hpp:24-27 (saturates at UINT64_MAX) */
uint64_t dfm_trans_required_bytes(uint64_t n);
/* trans_minimize, min_trans.hpp:81.  TransInspect (min_trans.hpp:41-44) when
 * apart_out (n*n u8) and/or popcounts_out (one u64 per pass, up to cap) are non-NULL. */
int dfm_trans_minimize(dfm_ctx* ctx, const dfm_dfa* d, const dfm_limits* limits,
                       uint8_t* apart_out, uint64_t* popcounts_out, uint32_t popcounts_cap,
                       uint32_t* block_out, uint32_t* num_blocks_out, dfm_stats* stats);
/* run_algorithm, bench.hpp:83 (AlgoRunConfig = policy + limits) */
int dfm_run_algorithm(dfm_ctx* ctx, int32_t algo, const dfm_dfa* d, int32_t policy,
                      const dfm_limits* limits, uint32_t* block_out, uint32_t* num_blocks_out,
                      dfm_stats* stats);

/* ---------------------------------------------------------------- device-resident API */
/* Upload a host DFA once (pinned staging, SoA rows of length n). */
int dfm_ddfa_upload(dfm_ctx* ctx, const dfm_dfa* d, dfm_ddfa** out);
/* Bit-exact device-side random_dfa (generators.hpp:130-145, counter-based SplitMix64). */
int dfm_ddfa_random(dfm_ctx* ctx, uint32_t n, uint32_t k, uint64_t seed, double accept_prob,
                    dfm_ddfa** out);
/* Copy a device DFA back (rows: k*n u32 flat, acc: n u8); either may be NULL. */
int dfm_ddfa_download(dfm_ctx* ctx, const dfm_ddfa* dd, uint32_t* delta_flat, uint8_t* accepting);
int dfm_ddfa_shape(const dfm_ddfa* dd, uint32_t* num_states, uint32_t* alphabet_size);
void dfm_ddfa_free(dfm_ddfa* dd);
/* Same algorithms on a resident DFA.  block_out_dev: device pointer (n u32) or NULL
 * to keep the canonical labels inside the ctx only; *num_blocks_out and stats are host. */
int dfm_run_algorithm_dev(dfm_ctx* ctx, int32_t algo, const dfm_ddfa* dd, int32_t policy,
                          const dfm_limits* limits, void* block_out_dev, uint32_t* num_blocks_out,
                          dfm_stats* stats);

/* ---------------------------------------------------------------- post-/pre-processing */
/* quotient, core.hpp:256-290: the automaton induced on the blocks of a CANONICAL
 * partition (block: n labels, e.g. a minimizer's block_out).  delta_out: k*num_blocks
 * u32 (row a at a*num_blocks), acc_out: num_blocks u8; either may be NULL.  Returns
 * DFM_ERR_INVALID with the reference's std::invalid_argument message in
 * dfm_last_error ("partition is not in canonical form", "inconsistent partition:
 * block B mixes accepting and rejecting states" / "... splits on letter A"). */
int dfm_quotient(dfm_ctx* ctx, const dfm_dfa* d, const uint32_t* block, uint32_t num_blocks,
                 uint32_t* delta_out, uint8_t* acc_out, uint32_t* initial_out);
/* Same on the device: block_dev = device canonical labels (dfm_run_algorithm_dev's
 * block_out_dev); *out is a new device DFA (free with dfm_ddfa_free). */
int dfm_ddfa_quotient(dfm_ctx* ctx, const dfm_ddfa* dd, const void* block_dev,
                      uint32_t num_blocks, dfm_ddfa** out);
/* remove_unreachable, core.hpp:152-187: keeps the states reachable from the initial
 * state, renumbered densely in ascending original order.  delta_out/acc_out need room
 * for the input's k*n / n entries; *num_states_out = kept states. */
int dfm_remove_unreachable(dfm_ctx* ctx, const dfm_dfa* d, uint32_t* num_states_out,
                           uint32_t* delta_out, uint8_t* acc_out, uint32_t* initial_out);
int dfm_ddfa_remove_unreachable(dfm_ctx* ctx, const dfm_ddfa* dd, dfm_ddfa** out);
int dfm_ddfa_initial(const dfm_ddfa* dd, uint32_t* initial);

/* ---------------------------------------------------------------- bulk input path */
/* Binary DFA file beside the reference's text format (ingest.hpp:286-369):
 * "DFMBIN01" | u32 n | u32 k | u32 initial | u32 0 | acc[n] u8 | pad to 4 | delta[k][n]
 * u32 (the reference's SoA rows).  Host write; device load through double-buffered
 * pinned staging (file reads overlap the H2D copies) and device save. */
int dfm_write_dfa_bin(const char* path, const dfm_dfa* d);
int dfm_ddfa_load_bin(dfm_ctx* ctx, const char* path, dfm_ddfa** out);
int dfm_ddfa_save_bin(dfm_ctx* ctx, const dfm_ddfa* dd, const char* path);

/* ---------------------------------------------------------------- host generators */
/* Multi-threaded, bit-exact with generators.hpp (SplitMix64 draw j = mix(seed+(j+1)*gamma)). */
int dfm_gen_random_dfa(uint32_t n, uint32_t k, uint64_t seed, double accept_prob,
                       uint32_t* delta_flat, uint8_t* accepting);

/* ---------------------------------------------------------------- sharded sortPR primitives */
/* State-sharded sortPR: one process per GPU; the host driver
 * (paper_2410_22764_b200/sharded.py) owns the collectives (torch.distributed over
 * NCCL) and calls these on device pointers (ctx's device and stream).  A rank owns
 * states [lo, lo+n_local); delta_local is k rows of n_local GLOBAL target ids. */
/* keys_out (u64[n_local]): 64-bit hash (never 0) of the signature row
 * (block_full[lo+i], block_full[delta_a(i)] for a < k) under `seed`; sig_out
 * (u32[n_local*(k+1)]): the rows themselves; dest_out (u32[n_local]): the rank in
 * [0, ranks) that groups this key. */
int dfm_shard_signature(dfm_ctx* ctx, const void* delta_local, uint64_t n_local, uint32_t k,
                        const void* block_full, uint64_t lo, uint64_t seed, uint32_t ranks,
                        void* keys_out, void* sig_out, void* dest_out);
/* Same with the block vector at id_bytes = 1/2/4 per state (all-gathered at the
 * narrowest width that holds B ids) and, when pack_bits > 0 ((k+1)*pack_bits <= 63),
 * EXACT packed keys (block, successor ids) + 1 instead of hashes: sig_out is then
 * not written (may be NULL) and the grouping needs no verification (words = 0). */
int dfm_shard_signature_ex(dfm_ctx* ctx, const void* delta_local, uint64_t n_local, uint32_t k,
                           const void* block_full, uint32_t id_bytes, uint64_t lo, uint64_t seed,
                           uint32_t ranks, uint32_t pack_bits, void* keys_out, void* sig_out,
                           void* dest_out);
/* Exact grouping of `count` received (key, signature-row) pairs: label_out[i] = dense
 * local group id in [0, *groups_out).  Equal-hash members are verified word by word
 * against the group's first member (words = 0: exact keys, no rows, sig may be NULL);
 * *collision_out = 1 when two different rows share a key (the driver then redoes the
 * pass under another seed). */
int dfm_shard_group(dfm_ctx* ctx, const void* keys, const void* sig, uint32_t words,
                    uint64_t count, void* label_out, uint64_t* groups_out, int* collision_out);
/* In-place stable LSD radix sort of (u64 key, u32 value) pairs on the low `bits` bits. */
int dfm_sort_pairs(dfm_ctx* ctx, void* keys, void* values, uint64_t count, uint32_t bits);
/* Canonical relabel (core.hpp:123-136) of raw labels < n: device in, device out. */
int dfm_canonicalize_dev(dfm_ctx* ctx, const void* raw_dev, uint64_t n, void* out_dev,
                         uint32_t* num_blocks_out);
/* Bit-exact random_dfa (generators.hpp:130-145) rows for states [lo, lo+count) of an
 * n_total-state automaton: delta_out k rows of `count` u32, accepting_out count u8. */
int dfm_random_dfa_slice_dev(dfm_ctx* ctx, uint64_t n_total, uint32_t k, uint64_t seed,
                             double accept_prob, uint64_t lo, uint64_t count, void* delta_out,
                             void* accepting_out);

/* ---------------------------------------------------------------- LTS ingestion (host) */
/* The VLTS front-end of the reference, host-side: parse_lts
 * (ingest.hpp:130-175), determinize (ingest.hpp:187-245), complete
 * (ingest.hpp:253-284).  No context (no GPU) needed.  Same automaton, same numbering,
 * same errors as the reference; the parser is multi-threaded. */
typedef struct dfm_lts dfm_lts;
typedef struct dfm_pdfa dfm_pdfa;
/* DFM_ERR_PARSE: err receives "line <n>: <what>" (ParseError::what()), *err_line = n */
int dfm_lts_parse(const char* text, uint64_t len, dfm_lts** out, uint64_t* err_line, char* err,
                  uint32_t err_cap);
int dfm_lts_info(const dfm_lts* lts, uint32_t* num_states, uint32_t* initial,
                 uint32_t* num_labels, uint64_t* num_transitions);
/* label i (interned in first-appearance order): pointer valid until dfm_lts_free */
int dfm_lts_label(const dfm_lts* lts, uint32_t i, const char** data, uint64_t* len);
/* the transitions in file order (each array num_transitions entries; NULL skips) */
int dfm_lts_transitions(const dfm_lts* lts, uint32_t* src, uint32_t* label, uint32_t* dst);
void dfm_lts_free(dfm_lts* lts);
/* an LTS from arrays (labels NULL: named "0", "1", ...) */
int dfm_lts_build(uint32_t num_states, uint32_t initial, uint32_t num_labels,
                  const char* const* labels, const uint64_t* label_lens, uint64_t m,
                  const uint32_t* src, const uint32_t* label, const uint32_t* dst, dfm_lts** out);
/* subset construction from {initial}; DFM_ERR_BUDGET (and *budget_out) when more than
 * max_subset_states subsets appear (reference default 1 << 22) */
int dfm_determinize(const dfm_lts* lts, uint64_t max_subset_states, dfm_pdfa** out,
                    uint64_t* budget_out);
int dfm_pdfa_shape(const dfm_pdfa* p, uint32_t* num_states, uint32_t* alphabet_size,
                   uint32_t* initial);
/* k rows of n targets, 0xFFFFFFFF = missing (PartialDfa::kMissing) */
int dfm_pdfa_rows(const dfm_pdfa* p, uint32_t* delta_flat);
/* complete with one rejecting sink iff a transition is missing: *num_states_out = n or
 * n + 1; delta_flat k * (*num_states_out) and accepting (*num_states_out) may be NULL
 * (query the size first) */
int dfm_complete(const dfm_pdfa* p, uint32_t* num_states_out, uint32_t* delta_flat,
                 uint8_t* accepting);
void dfm_pdfa_free(dfm_pdfa* p);
int dfm_pdfa_build(uint32_t num_states, uint32_t alphabet_size, uint32_t initial,
                   const uint32_t* delta_flat, dfm_pdfa** out);

/* ---------------------------------------------------------------- sharded sortPR driver */
/* The C++ driver of the state-sharded sortPR: a context
 * that owns one rank of a communicator runs the whole protocol (narrow-width
 * all-gather of block ids, keys, routed exact grouping, dense ids back, fixpoint,
 * canonical labels) — the drop-in for min_sort.hpp:72 sort_pr on DFAs too large
 * for one GPU.  Rank r owns the contiguous states [r*S, min(n, (r+1)*S)),
 * S = ceil(n/world) rounded up to a multiple of 32 (dfm_shard_bounds); its rows
 * hold GLOBAL target ids.
 * Result: the same canonical partition, block count and pass count as the
 * reference's sort_pr for every world size. */
#define DFM_NCCL_ID_BYTES 128
/* rank 0 calls this; the host distributes the 128 bytes to every rank */
int dfm_nccl_get_unique_id(uint8_t* id_out /* DFM_NCCL_ID_BYTES */);
/* one process per GPU: a context owning rank `rank` of an NCCL communicator */
int dfm_ctx_create_sharded(int device, int rank, int world, const uint8_t* nccl_id,
                           dfm_ctx** out);
/* test transport: `world` ranks as host threads of ONE process on one device,
 * meeting in the named group (each thread creates its own context) */
int dfm_ctx_create_sharded_local(int device, int rank, int world, const char* group,
                                 dfm_ctx** out);
int dfm_ctx_shard_info(const dfm_ctx* ctx, int* rank, int* world, const char** transport);
void dfm_shard_bounds(uint64_t n_total, int world, int rank, uint64_t* lo, uint64_t* hi);
/* Collective calls: an infrastructure fault on one rank (e.g. out of device memory)
 * leaves the other ranks waiting in the next collective, as with NCCL itself — abort
 * the job.  Algorithmic outcomes (timeout, an out-of-range target) are agreed on by
 * all ranks and returned everywhere. */
/* Host rows of the owned states (local->num_states = hi - lo, targets < n_total;
 * pageable or pinned).  block_out: the owned states' canonical labels (hi - lo
 * entries), or with gather_all the whole canonical partition (n_total entries) on
 * every rank.  Collective: every rank calls it. */
int dfm_sort_pr_sharded(dfm_ctx* ctx, uint64_t n_total, const dfm_dfa* local, int gather_all,
                        uint32_t* block_out, uint32_t* num_blocks_out, int64_t timeout_ms,
                        dfm_stats* stats);
/* Device-resident shard: delta_dev k rows of n_local u32, acc_dev n_local u8,
 * block_out_dev n_local u32 (canonical labels of the owned states).  Targets are
 * trusted (< n_total), like dfm_run_algorithm_dev; the host entry checks them. */
int dfm_sort_pr_sharded_dev(dfm_ctx* ctx, uint64_t n_total, uint32_t n_local, uint32_t k,
                            const void* delta_dev, const void* acc_dev, void* block_out_dev,
                            uint32_t* num_blocks_out, int64_t timeout_ms, dfm_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* DFM_H */
