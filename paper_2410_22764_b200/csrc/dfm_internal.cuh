// Internal runtime of libdfm.so: context, error model, stream-ordered scratch
// arena and per-kernel-family CUDA-event profiling.  sm_100a only.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "dfm.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libdfm is written for sm_100a only (compile with -gencode arch=compute_100a,code=sm_100a)"
#endif

namespace dfm {

constexpr uint32_t kNoLeader = 0xFFFFFFFFu;  // substrate.hpp:95

// Infrastructure faults travel as exceptions inside the library and become
// dfm_err codes at the C-ABI boundary (capi.cu).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? DFM_ERR_NO_MEMORY : DFM_ERR_CUDA;
    throw Error(code, std::string(what) + " failed at " + file + ":" + std::to_string(line) +
                          ": " + cudaGetErrorString(e));
  }
}
#define DFM_CUDA(x) ::dfm::cuda_check((x), #x, __FILE__, __LINE__)
// every kernel launch site calls DFM_LAUNCH_CHECK(): it also counts launches
// (dfm_kernel_launches(), the bench's gpu_launches evidence)
uint64_t note_launch();
uint64_t launch_count();
#define DFM_LAUNCH_CHECK() \
  (::dfm::note_launch(), ::dfm::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__))

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Per-device, thread-safe memo for kernel attributes and occupancy queries:
// cudaFuncSetAttribute applies to the CURRENT device only, so an opt-in made for
// one context must be repeated for a context on another device.  `key` names the
// kernel (its address); `f` runs once per (key, device) under a mutex and its
// result is cached.
int per_device_memo(const void* key, int device, int (*f)(const void* key));

// A growable device buffer from the ctx arena (stream-ordered allocator with
// an unbounded release threshold, so repeated calls reuse the same HBM).
struct Buf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

struct Ctx;
struct Comm;  // comm.cuh: collectives of a sharded context

// Times one kernel family with events on the launching stream when profiling
// is enabled.  Usage: { ProfScope p(ctx, "sig"); kernel<<<..., ctx.stream>>>(); }
// `bytes` is the ALGORITHMIC byte count of the scoped work,
// accumulated next to the measured time for the roofline.
struct ProfScope {
  Ctx& ctx;
  const char* name;
  uint64_t bytes;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool stopped = false;
  ProfScope(Ctx& c, const char* n, uint64_t algo_bytes = 0);
  // end the timed region early; `bytes` may still be set before destruction (work
  // counts known only after a device read-back, e.g. persistent-kernel passes)
  void stop();
  ~ProfScope();
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  std::string last_error;
  // named scratch slots: each algorithm asks for a slot by name and size
  std::map<std::string, Buf> slots;
  uint64_t held_bytes = 0;
  // pinned host staging
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // sortPR grouping engine: DFM_SORTPR_HASH (default) or DFM_SORTPR_RADIX
  int sortpr_engine = 0;
  // Cho–Huynh squaring engine: DFM_TRANS_AUTO (default) / DFM_TRANS_BIT / DFM_TRANS_TENSOR
  int trans_engine = 0;
  // sharded contexts (dfm_ctx_create_sharded[_local]): this rank's communicator
  Comm* comm = nullptr;
  // dfm_ctx_set_out_ready_hook: armed for the next host-buffer call
  void (*out_ready)(void*) = nullptr;
  void* out_user = nullptr;
  // profiling
  bool profiling = false;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
    uint64_t bytes;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> free_events;
  struct Acc {
    uint64_t launches = 0;
    double ms = 0;
    uint64_t bytes = 0;
  };
  std::map<std::string, Acc> prof;
  std::string prof_names;
  // small device scalars for host read-back (pinned host mirror)
  uint64_t* d_scalars = nullptr;  // device, 64 slots
  uint64_t* h_scalars = nullptr;  // pinned host, 64 slots
  // second stream for pipelined host->device uploads, and its chunk events
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> chunk_events;
  cudaStream_t copy();
  const cudaEvent_t* chunk_event_pool(uint32_t count);

  explicit Ctx(int dev);
  ~Ctx();

  void* slot(const std::string& name, size_t bytes);
  template <class T>
  T* slot_t(const std::string& name, size_t count) {
    return static_cast<T*>(slot(name, count * sizeof(T)));
  }
  void release_slot(const std::string& name);
  void* host_pinned(size_t bytes);
  void sync() { DFM_CUDA(cudaStreamSynchronize(stream)); }
  // fold completed profiling events into the accumulators
  void harvest();
  cudaEvent_t take_event();
};

inline double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// Deadline bookkeeping shared by all algorithms (core.hpp:190-199).
struct Deadline {
  double start;
  double limit;  // <= 0: none
  Deadline(int64_t timeout_ms) : start(now_ms()), limit(timeout_ms > 0 ? (double)timeout_ms : 0) {}
  bool expired() const { return limit > 0 && now_ms() - start > limit; }
  double elapsed() const { return now_ms() - start; }
};

// Host side of a pipelined upload whose chunk events are recorded by a staging
// thread (pageable rows copied through a pinned ring): a consumer must not enqueue
// cudaStreamWaitEvent(ready[c]) before the event is recorded, so it blocks here
// until chunk c's copy has been enqueued.
struct ChunkGate {
  virtual void wait_recorded(uint32_t c) = 0;
  virtual ~ChunkGate() = default;
};

// Device-resident DFA: SoA rows packed as one [k][n] allocation.
struct DevDfa {
  uint32_t n = 0, k = 0, initial = 0;
  uint32_t* delta = nullptr;  // k*n
  uint8_t* acc = nullptr;     // n
  bool owns = true;
  // pipelined upload (sortPR from host buffers): the rows of states
  // [c*chunk_states, (c+1)*chunk_states) are in HBM once ready[c] has fired on the
  // copy stream; their targets are not yet validated (`bad` flags an out-of-range
  // one, which the consumer zeroes).  acc is complete.  nready == 0: all resident.
  const cudaEvent_t* ready = nullptr;
  uint32_t nready = 0;
  uint64_t chunk_states = 0;
  unsigned long long* bad = nullptr;
  ChunkGate* gate = nullptr;  // pageable source: chunk events recorded by a stager thread
};

struct AlgoOut {
  uint32_t num_blocks = 0;
  uint64_t iterations = 0, closure_steps = 0, peak_memory_estimate = 0;
  uint64_t skipped_passes = 0;  // counted fixpoint passes that did not run
  int32_t status = DFM_STATUS_OK;
  uint32_t* canon_dev = nullptr;  // canonical labels on device (ctx slot "canon")
  bool canon_identity = false;    // every block a singleton: canonical labels = 0..n-1
};

// ---- algorithm drivers (device-resident input, results on device) ----
AlgoOut run_sort_pr(Ctx& ctx, const DevDfa& d, const Deadline& dl, const dfm_trace* trace);
AlgoOut run_sort_pr_hash(Ctx& ctx, const DevDfa& d, const Deadline& dl, const dfm_trace* trace);
// states per chunk of a pipelined sortPR upload (whole layout windows, ~64 MB of
// rows), or 0 when sortPR would not consume the rows chunk by chunk
uint64_t sortpr_upload_chunk(uint64_t n, uint32_t k);
AlgoOut run_leader_election(Ctx& ctx, const DevDfa& d, const uint32_t* rows, uint64_t letters,
                            int policy, bool fused_cas, const Deadline& dl,
                            const dfm_trace* trace);
uint32_t* expand_alphabet_dev(Ctx& ctx, const DevDfa& d, uint32_t levels);
AlgoOut run_trans_pr(Ctx& ctx, const DevDfa& d, int policy, const dfm_limits& lim,
                     const Deadline& dl);
AlgoOut run_trans_minimize(Ctx& ctx, const DevDfa& d, const dfm_limits& lim, const Deadline& dl,
                           uint8_t* apart_host, uint64_t* popcounts, uint32_t pop_cap);
// canonical relabel of raw labels (< n) into ctx slot "canon"; returns block count
uint32_t canonicalize_dev(Ctx& ctx, const uint32_t* raw, uint64_t n, uint32_t* out);
// quotient (core.hpp:256-290) of a canonical device partition; throws Error
// (DFM_ERR_INVALID) with the reference's invalid_argument messages
DevDfa quotient_dev(Ctx& ctx, const DevDfa& d, const uint32_t* block, uint32_t num_blocks);
// remove_unreachable (core.hpp:152-187)
DevDfa remove_unreachable_dev(Ctx& ctx, const DevDfa& d);
// binary DFA files (csrc/io.cu): host write, device load / save
void write_dfa_bin(const char* path, uint32_t n, uint32_t k, uint32_t initial,
                   const uint32_t* const* rows, const uint8_t* acc);
DevDfa load_dfa_bin(Ctx& ctx, const char* path);
void save_dfa_bin(Ctx& ctx, const DevDfa& dd, const char* path);
// host -> device copy on ctx.stream of a possibly pageable host buffer (pageable:
// staged by several host threads through a pinned ring, synchronous for the host)
void h2d_rows(Ctx& ctx, void* dst, const void* src, uint64_t bytes);
struct H2DPiece {
  void* dst;
  const void* src;
  uint64_t bytes;
};
void h2d_batch(Ctx& ctx, const std::vector<H2DPiece>& pieces);
// sharded sortPR primitives (shard.cu) and the C++ driver (shard_driver.cu)
void shard_signature(Ctx& ctx, const void* delta_local, uint64_t n_local, uint32_t k,
                     const void* block_full, uint32_t id_bits, uint64_t lo, uint64_t seed,
                     uint32_t ranks, uint32_t pack_bits, void* keys_out, void* sig_out,
                     void* dest_out);
void shard_group(Ctx& ctx, const void* keys, const void* sig, uint32_t words, uint64_t count,
                 void* label_out, uint64_t* groups_out, int* collision_out);
// exact packed keys (+1) from a key space of 2^key_bits: presence bitmap + rank
void shard_group_direct(Ctx& ctx, const void* keys, uint64_t count, uint32_t key_bits,
                        void* label_out, uint64_t* groups_out);
// the blocked signature builder over a shard's rows (sortpr_hash.cu): null when the
// shard is too small or n_total exceeds the layout's range limit (~2e8 states)
struct ShardLayout;
ShardLayout* shard_layout_build(Ctx& ctx, const DevDfa& loc, uint64_t n_total);
void shard_layout_free(ShardLayout* s);
// keys (exact packed, or the shard kernels' hash chain + rows of `row` words) of the
// m = loc.n owned states from the all-gathered ids at id_bits in {1, 4, 8, 16, 32}
void shard_layout_keys(Ctx& ctx, ShardLayout* s, int id_bits, const uint32_t* full,
                       const uint32_t* own, uint64_t m, int w, bool hashed, uint64_t seed,
                       unsigned long long* keys, uint32_t* sig, uint32_t row);
// the same builder for the radix engine (sort_pr.cu) over the whole DFA: keys of the
// m active states (ascending act, or all states) in active order
ShardLayout* radix_layout_build(Ctx& ctx, const DevDfa& d);
// DFM_SORTPR_WEAK_HASH (tests): truncated hashed keys under the first seed
void sortpr_weak_hash_setup();
void radix_layout_keys(Ctx& ctx, ShardLayout* s, int id_bits, const uint32_t* ids,
                       const uint32_t* act, uint64_t m, const uint32_t* block, int w, bool hashed,
                       uint64_t seed, unsigned long long* keys, uint32_t* sig, uint32_t row);
// contiguous shards of S = ceil(n/world) rounded up to a multiple of 32 states (a
// rank's slice of a bit-packed id vector is whole words): rank r owns
// [r*S, min(n, (r+1)*S))
inline uint64_t shard_size(uint64_t n, int world) {
  return ceil_div(ceil_div(n, (uint64_t)world), 32) * 32;
}
// `loc` = the owned rows (n = owned states, GLOBAL targets); canonical labels of the
// owned states into canon_dev (device, loc.n entries)
AlgoOut run_sort_pr_sharded(Ctx& ctx, uint64_t n_total, const DevDfa& loc, const Deadline& dl,
                            uint32_t* canon_dev, bool force_protocol, bool validate = true);
// device random_dfa
void random_dfa_dev(Ctx& ctx, DevDfa& d, uint32_t n, uint32_t k, uint64_t seed, double p);

}  // namespace dfm
