// C-ABI entry points of libdfm.so (include/dfm.h).  Converts infrastructure
// exceptions into dfm_err codes, uploads host DFAs, dispatches algorithms and
// copies canonical partitions back.
#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "dfm_internal.cuh"
#include "prims.cuh"

struct dfm_ctx {};   // opaque: really dfm::Ctx
struct dfm_ddfa {};  // opaque: really dfm::DevDfa

namespace dfm {
namespace {

thread_local std::string g_create_error;

Ctx* as_ctx(dfm_ctx* c) { return reinterpret_cast<Ctx*>(c); }
const Ctx* as_ctx(const dfm_ctx* c) { return reinterpret_cast<const Ctx*>(c); }
DevDfa* as_dd(dfm_ddfa* d) { return reinterpret_cast<DevDfa*>(d); }
const DevDfa* as_dd(const dfm_ddfa* d) { return reinterpret_cast<const DevDfa*>(d); }

template <class F>
int guarded(dfm_ctx* c, F&& f) {
  Ctx* ctx = as_ctx(c);
  if (ctx == nullptr) return DFM_ERR_INVALID;
  std::lock_guard<std::mutex> lk(ctx->mu);
  try {
    DFM_CUDA(cudaSetDevice(ctx->device));
    f(*ctx);
    ctx->harvest();
    return DFM_OK;
  } catch (const Error& e) {
    ctx->last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    ctx->last_error = "host allocation failed";
    return DFM_ERR_NO_MEMORY;
  } catch (const std::exception& e) {
    ctx->last_error = e.what();
    return DFM_ERR_INVALID;
  }
}

__global__ void validate_kernel(const uint32_t* __restrict__ delta, uint64_t total, uint32_t n,
                                unsigned long long* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  bool b = false;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
    b |= delta[i] >= n;
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1ull);
}

void check_host_dfa(const dfm_dfa* d) {
  if (d == nullptr) throw Error(DFM_ERR_INVALID, "null dfa");
  if (d->num_states < 1) throw Error(DFM_ERR_INVALID, "automaton needs at least one state");
  if (d->alphabet_size > 0 && d->delta == nullptr)
    throw Error(DFM_ERR_INVALID, "transition table has wrong number of letter rows");
  for (uint32_t a = 0; a < d->alphabet_size; ++a)
    if (d->delta[a] == nullptr)
      throw Error(DFM_ERR_INVALID, "transition row " + std::to_string(a) + " is null");
  if (d->accepting == nullptr) throw Error(DFM_ERR_INVALID, "accepting indicator is null");
  if (d->initial >= d->num_states) throw Error(DFM_ERR_INVALID, "initial state out of range");
}

// every target < n (the engine would fault otherwise; core.hpp:104-119)
void validate_targets(Ctx& ctx, const DevDfa& dd) {
  const uint64_t total = (uint64_t)dd.n * dd.k;
  if (total == 0) return;
  auto* bad = reinterpret_cast<unsigned long long*>(ctx.d_scalars + 40);
  DFM_CUDA(cudaMemsetAsync(bad, 0, 8, ctx.stream));
  const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(total, 256), ctx.num_sms * 16ull);
  validate_kernel<<<grid, 256, 0, ctx.stream>>>(dd.delta, total, dd.n, bad);
  DFM_LAUNCH_CHECK();
  DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 40, bad, 8, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  if (ctx.h_scalars[40]) throw Error(DFM_ERR_INVALID, "transition target out of range");
}

// ---- host input in pageable memory (the reference's Dfa: std::vector rows).
// cudaMemcpyAsync from pageable memory is staged by the driver through its own
// small pinned buffer, synchronously and single-threaded; instead the rows are
// copied by several host threads into a pinned ring and DMA'd from there.
bool host_pinned_ptr(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // clear
    return false;
  }
  return at.type == cudaMemoryTypeHost;  // cudaMallocHost or cudaHostRegister
}

unsigned stage_threads() {
  if (const char* e = getenv("DFM_STAGE_THREADS")) return std::max(1, atoi(e));
  // measured on the 16-core B200 hosts (tools/e2e_stage.py), e2e of random_dfa(1e8, 4)
  // from pageable rows: threads spawned per copy (profiles/r02h) 4 / 8 / 12 / 16 ->
  // 84 / 69 / 66 / 69 ms; the persistent pool (profiles/r04/r04g) 8 / 12 / 16 -> 66.7 /
  // 60.8 / 58.1 ms (pinned rows: 41 ms)
  return std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
}

// Persistent host workers for the staging copies.  Spawning the copy threads per
// memcpy call (one fork-join per letter segment of every chunk) cost a third of the
// staging throughput: copying random_dfa(1e8, 4)'s rows into a pinned ring took 83 ms
// with 8 spawned threads per call and 56 ms with 8 persistent workers, one fork-join
// per chunk (8-core container).  One pool per process;
// concurrent uploads take turns (they share the host's memory bandwidth anyway).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool(stage_threads());
    return pool;
  }
  unsigned size() const { return T_; }
  // f(t) for t in [0, size()): t = 0 on the calling thread
  void run(const std::function<void(unsigned)>& f) {
    std::lock_guard<std::mutex> turn(run_mu_);
    if (T_ == 1) {
      f(0);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      left_ = T_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return left_ == 0; });
    job_ = nullptr;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }

 private:
  explicit HostPool(unsigned T) : T_(std::max(1u, T)) {
    for (unsigned t = 1; t < T_; ++t)
      th_.emplace_back([this, t] {
        uint64_t seen = 0;
        while (true) {
          const std::function<void(unsigned)>* f;
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            f = job_;
          }
          (*f)(t);
          std::lock_guard<std::mutex> lk(mu_);
          if (--left_ == 0) done_.notify_one();
        }
      });
  }
  unsigned T_;
  std::vector<std::thread> th_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(unsigned)>* job_ = nullptr;
  uint64_t gen_ = 0;
  unsigned left_ = 0;
  bool stop_ = false;
};

// dst[0 .. nseg*seg) = the segments srcs[0..nseg) (seg bytes each) back to back,
// split evenly over the pool (a worker's share may cross segment boundaries)
void par_memcpy_segs(char* dst, const char* const* srcs, size_t seg, size_t nseg) {
  const size_t total = seg * nseg;
  HostPool& pool = HostPool::get();
  const unsigned T = total < (8u << 20) ? 1u : pool.size();
  auto part = [&](unsigned t) {
    size_t lo = (total * t / T) & ~size_t(63);
    const size_t hi = t + 1 == T ? total : (total * (t + 1) / T) & ~size_t(63);
    while (lo < hi) {
      const size_t a = lo / seg, o = lo - a * seg, e = std::min(hi, (a + 1) * seg);
      std::memcpy(dst + lo, srcs[a] + o, e - lo);
      lo = e;
    }
  };
  if (T == 1) part(0);
  else pool.run(part);
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  const char* s = static_cast<const char*>(src);
  par_memcpy_segs(static_cast<char*>(dst), &s, bytes, 1);
}

constexpr uint32_t kRing = 3;  // pinned ring slots of one upload chunk each

// Copies the rows of a pageable host DFA chunk by chunk (all k letter segments of
// states [q0, q0+len)) through a pinned ring on its own host thread, issuing each
// chunk's DMA on the copy stream and recording ready[c]; consumers gate on
// wait_recorded(c) before waiting for the event on the device.
class PageableStager final : public ChunkGate {
 public:
  PageableStager(Ctx& ctx, const dfm_dfa* d, uint32_t* delta_dev, uint64_t chunk,
                 const cudaEvent_t* ready, uint32_t nc, char* ring, uint64_t slot_bytes,
                 cudaEvent_t* slot_ev, bool* slot_used)
      : ctx_(ctx), d_(d), dev_(delta_dev), chunk_(chunk), ready_(ready), nc_(nc), ring_(ring),
        slot_bytes_(slot_bytes), slot_ev_(slot_ev), slot_used_(slot_used) {
    th_ = std::thread([this] { run(); });
  }
  ~PageableStager() override { join_quiet(); }
  void wait_recorded(uint32_t c) override {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return recorded_ > c || !err_.empty(); });
    if (!err_.empty()) throw Error(DFM_ERR_CUDA, err_);
  }
  void join() {
    join_quiet();
    if (!err_.empty()) throw Error(DFM_ERR_CUDA, err_);
  }

 private:
  void join_quiet() {
    if (th_.joinable()) th_.join();
  }
  void run() {
    try {
      DFM_CUDA(cudaSetDevice(ctx_.device));
      const uint64_t n = d_->num_states, k = d_->alphabet_size;
      cudaStream_t cs = ctx_.copy();
      std::vector<const char*> srcs(k);
      for (uint32_t c = 0; c < nc_; ++c) {
        const uint32_t s = c % kRing;
        if (slot_used_[s]) DFM_CUDA(cudaEventSynchronize(slot_ev_[s]));
        char* slot = ring_ + (uint64_t)s * slot_bytes_;
        const uint64_t q0 = (uint64_t)c * chunk_, len = std::min(n, q0 + chunk_) - q0;
        for (uint64_t a = 0; a < k; ++a)
          srcs[a] = reinterpret_cast<const char*>(d_->delta[a] + q0);
        par_memcpy_segs(slot, srcs.data(), len * 4, k);
        for (uint64_t a = 0; a < k; ++a)
          DFM_CUDA(cudaMemcpyAsync(dev_ + a * n + q0, slot + a * len * 4, len * 4,
                                   cudaMemcpyHostToDevice, cs));
        DFM_CUDA(cudaEventRecord(ready_[c], cs));
        DFM_CUDA(cudaEventRecord(slot_ev_[s], cs));
        slot_used_[s] = true;
        {
          std::lock_guard<std::mutex> lk(mu_);
          recorded_ = c + 1;
        }
        cv_.notify_all();
      }
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lk(mu_);
      err_ = std::string("pageable upload: ") + e.what();
      cv_.notify_all();
    }
  }
  Ctx& ctx_;
  const dfm_dfa* d_;
  uint32_t* dev_;
  uint64_t chunk_;
  const cudaEvent_t* ready_;
  uint32_t nc_;
  char* ring_;
  uint64_t slot_bytes_;
  cudaEvent_t* slot_ev_;
  bool* slot_used_;
  std::thread th_;
  std::mutex mu_;
  std::condition_variable cv_;
  uint32_t recorded_ = 0;
  std::string err_;
};

// per-upload staging resources (events created once per upload; the ring is the
// ctx's cached pinned buffer)
struct StageRes {
  cudaEvent_t ev[kRing] = {};
  bool used[kRing] = {};
  uint32_t next = 0;
  std::unique_ptr<PageableStager> stager;
  ~StageRes() {
    stager.reset();
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
};

// copy `bytes` of pageable host memory to the device through the ring slots
// (synchronous for the caller; the DMA runs on `stream`)
void staged_h2d(Ctx& ctx, void* dst, const void* src, uint64_t bytes, cudaStream_t stream,
                char* ring, uint64_t slot_bytes, StageRes& res) {
  uint32_t& s = res.next;  // ring cursor continues across pieces
  for (uint64_t off = 0; off < bytes; off += slot_bytes, s = (s + 1) % kRing) {
    const uint64_t len = std::min(slot_bytes, bytes - off);
    if (res.used[s]) DFM_CUDA(cudaEventSynchronize(res.ev[s]));
    char* slot = ring + (uint64_t)s * slot_bytes;
    par_memcpy(slot, static_cast<const char*>(src) + off, len);
    DFM_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, slot, len, cudaMemcpyHostToDevice,
                             stream));
    DFM_CUDA(cudaEventRecord(res.ev[s], stream));
    res.used[s] = true;
  }
}

StageRes& new_stage_res(std::unique_ptr<StageRes>& holder) {
  holder.reset(new StageRes);
  for (auto& e : holder->ev) DFM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return *holder;
}

// stage a host DFA into device memory (slot names under `prefix`)
DevDfa upload(Ctx& ctx, const dfm_dfa* d, const std::string& prefix, bool own_alloc) {
  check_host_dfa(d);
  DevDfa dd;
  dd.n = d->num_states;
  dd.k = d->alphabet_size;
  dd.initial = d->initial;
  const uint64_t n = dd.n, k = dd.k;
  if (own_alloc) {
    DFM_CUDA(cudaMalloc(&dd.delta, std::max<uint64_t>(n * k, 1) * 4));
    DFM_CUDA(cudaMalloc(&dd.acc, n));
    dd.owns = true;
  } else {
    dd.delta = ctx.slot_t<uint32_t>(prefix + ".delta", std::max<uint64_t>(n * k, 1));
    dd.acc = ctx.slot_t<uint8_t>(prefix + ".acc", n);
    dd.owns = false;
  }
  std::vector<H2DPiece> pieces;
  for (uint64_t a = 0; a < k; ++a) pieces.push_back({dd.delta + a * n, d->delta[a], n * 4});
  pieces.push_back({dd.acc, d->accepting, n});
  h2d_batch(ctx, pieces);
  validate_targets(ctx, dd);
  return dd;
}

// sortPR from host buffers: accepting flags first, then the rows chunk by chunk on
// the copy stream; sortPR's first pass and the layout build consume each chunk as
// it lands (validation included), so only the tail of the copy is exposed
DevDfa upload_progressive(Ctx& ctx, const dfm_dfa* d, uint64_t chunk,
                          std::unique_ptr<StageRes>& stage) {
  check_host_dfa(d);
  DevDfa dd;
  dd.n = d->num_states;
  dd.k = d->alphabet_size;
  dd.initial = d->initial;
  const uint64_t n = dd.n, k = dd.k;
  dd.delta = ctx.slot_t<uint32_t>("in.delta", std::max<uint64_t>(n * k, 1));
  dd.acc = ctx.slot_t<uint8_t>("in.acc", n);
  dd.owns = false;
  const bool pageable = k > 0 && !host_pinned_ptr(d->delta[0]);
  const uint32_t nc = (uint32_t)ceil_div(n, chunk);
  const cudaEvent_t* ev = ctx.chunk_event_pool(nc);
  cudaStream_t cs = ctx.copy();
  if (pageable) {
    // rows through a pinned ring on a stager thread; acc first, from the caller thread
    const uint64_t slot_bytes = chunk * k * 4;
    char* ring = static_cast<char*>(ctx.host_pinned(kRing * slot_bytes));
    StageRes& res = new_stage_res(stage);
    if (host_pinned_ptr(d->accepting))
      DFM_CUDA(cudaMemcpyAsync(dd.acc, d->accepting, n, cudaMemcpyHostToDevice, ctx.stream));
    else
      staged_h2d(ctx, dd.acc, d->accepting, n, ctx.stream, ring, slot_bytes, res);
    DFM_CUDA(cudaEventRecord(ev[0], ctx.stream));
    DFM_CUDA(cudaStreamWaitEvent(cs, ev[0], 0));
    res.stager.reset(new PageableStager(ctx, d, dd.delta, chunk, ev, nc, ring, slot_bytes, res.ev,
                                        res.used));
    dd.gate = res.stager.get();
  } else {
    DFM_CUDA(cudaMemcpyAsync(dd.acc, d->accepting, n, cudaMemcpyHostToDevice, ctx.stream));
    // the copy stream starts after everything queued so far (slot allocations)
    DFM_CUDA(cudaEventRecord(ev[0], ctx.stream));
    DFM_CUDA(cudaStreamWaitEvent(cs, ev[0], 0));
  }
  for (uint32_t c = 0; c < nc && !pageable; ++c) {
    const uint64_t q0 = c * chunk, len = std::min(n, q0 + chunk) - q0;
    for (uint64_t a = 0; a < k; ++a)
      DFM_CUDA(cudaMemcpyAsync(dd.delta + a * n + q0, d->delta[a] + q0, len * 4,
                               cudaMemcpyHostToDevice, cs));
    DFM_CUDA(cudaEventRecord(ev[c], cs));
  }
  dd.ready = ev;
  dd.nready = nc;
  dd.chunk_states = chunk;
  dd.bad = reinterpret_cast<unsigned long long*>(ctx.d_scalars + 40);
  DFM_CUDA(cudaMemsetAsync(dd.bad, 0, 8, ctx.stream));
  return dd;
}

dfm_limits limits_or_default(const dfm_limits* l) {
  dfm_limits r;
  r.max_memory_bytes = l ? l->max_memory_bytes : (16ull << 30);
  r.timeout_ms = l ? l->timeout_ms : 300000;
  return r;
}

AlgoOut dispatch(Ctx& ctx, int32_t algo, const DevDfa& dd, int32_t policy, const dfm_limits& lim,
                 const dfm_trace* trace, uint8_t* apart, uint64_t* pops, uint32_t pop_cap) {
  if (policy < DFM_POLICY_ARBITRARY || policy > DFM_POLICY_MAX)
    throw Error(DFM_ERR_INVALID, "unknown race policy");
  const Deadline dl(lim.timeout_ms);
  switch (algo) {
    case DFM_ALGO_TRANS:
      return run_trans_minimize(ctx, dd, lim, dl, apart, pops, pop_cap);
    case DFM_ALGO_NAIVE:
      return run_leader_election(ctx, dd, dd.delta, dd.k, policy, false, dl, trace);
    case DFM_ALGO_NAIVE_CAS:
      return run_leader_election(ctx, dd, dd.delta, dd.k, DFM_POLICY_ARBITRARY, true, dl, trace);
    case DFM_ALGO_SORT:
      return ctx.sortpr_engine == DFM_SORTPR_RADIX ? run_sort_pr(ctx, dd, dl, trace)
                                                   : run_sort_pr_hash(ctx, dd, dl, trace);
    case DFM_ALGO_TRANSPR:
      return run_trans_pr(ctx, dd, policy, lim, dl);
    case DFM_ALGO_ORACLE:
      throw Error(DFM_ERR_INVALID, "the Moore oracle is a CPU reference, not a GPU algorithm");
    default:
      throw Error(DFM_ERR_INVALID, "unknown algorithm");
  }
}

// host buffer = 0..n-1 with a few threads (faster than reading the identity back
// over PCIe: 400 MB at 1e8 states)
void host_iota(uint32_t* out, uint64_t n) {
  const unsigned T = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>(std::max(1u, std::thread::hardware_concurrency()), n >> 22));
  auto work = [&](unsigned t) {
    const uint64_t lo = n * t / T, hi = n * (t + 1) / T;
    for (uint64_t q = lo; q < hi; ++q) out[q] = (uint32_t)q;
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

// the caller's out-ready hook (dfm_ctx_set_out_ready_hook): run once before the first
// write into the caller's partition buffer, from whichever thread writes first
struct OutGate {
  void (*fn)(void*) = nullptr;
  void* user = nullptr;
  std::once_flag once;
  void wait() {
    if (fn) std::call_once(once, [this] { fn(user); });
  }
};

// sortPR on a large automaton usually ends all singletons (random DFAs): the identity
// labels are written into the caller's buffer by a host thread WHILE the GPU runs;
// joined before anything else touches the buffer (a non-identity result overwrites it)
struct SpeculativeIota {
  std::thread th;
  bool started = false;
  void start(uint32_t* out, uint64_t n, OutGate* gate) {
    th = std::thread([out, n, gate] {
      gate->wait();
      host_iota(out, n);
    });
    started = true;
  }
  void join() {
    if (th.joinable()) th.join();
  }
  ~SpeculativeIota() { join(); }
};

void finish(Ctx& ctx, const AlgoOut& o, uint64_t n, const Deadline& dl, uint32_t* block_out,
            uint32_t* nb_out, dfm_stats* st, bool iota_written = false, OutGate* gate = nullptr) {
  const bool identity = o.status == DFM_STATUS_OK && block_out != nullptr && o.canon_identity;
  if (gate && o.status == DFM_STATUS_OK && block_out != nullptr) gate->wait();
  if (o.status == DFM_STATUS_OK && block_out != nullptr && !identity)
    DFM_CUDA(cudaMemcpyAsync(block_out, o.canon_dev, n * 4, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  if (identity && !iota_written) host_iota(block_out, n);
  if (nb_out) *nb_out = o.status == DFM_STATUS_OK ? o.num_blocks : 0;
  if (st) {
    st->iterations = o.iterations;
    st->executed_passes = o.iterations - o.skipped_passes;
    st->closure_steps = o.closure_steps;
    st->peak_memory_estimate = o.peak_memory_estimate;
    st->status = o.status;
    st->elapsed_ms = dl.elapsed();
  }
}

int run_host(dfm_ctx* c, int32_t algo, const dfm_dfa* d, int32_t policy, const dfm_limits* l,
             const dfm_trace* trace, uint8_t* apart, uint64_t* pops, uint32_t pop_cap,
             uint32_t* block_out, uint32_t* nb_out, dfm_stats* st) {
  return guarded(c, [&](Ctx& ctx) {
    const Deadline whole(0);
    const dfm_limits lim = limits_or_default(l);
    OutGate gate;  // consumes the armed out-ready hook
    gate.fn = ctx.out_ready;
    gate.user = ctx.out_user;
    ctx.out_ready = nullptr;
    ctx.out_user = nullptr;
    SpeculativeIota spec;  // (declared after the gate: joined before it goes away)
    if (algo == DFM_ALGO_SORT && block_out != nullptr && d != nullptr &&
        d->num_states >= (1u << 22))
      spec.start(block_out, d->num_states, &gate);
    const uint64_t chunk =
        (algo == DFM_ALGO_SORT && ctx.sortpr_engine != DFM_SORTPR_RADIX && d != nullptr &&
         !(trace && trace->on_pass))
            ? sortpr_upload_chunk(d->num_states, d->alphabet_size)
            : 0;
    std::unique_ptr<StageRes> stage;
    const DevDfa dd =
        chunk ? upload_progressive(ctx, d, chunk, stage) : upload(ctx, d, "in", false);
    AlgoOut o;
    try {
      o = dispatch(ctx, algo, dd, policy, lim, trace, apart, pops, pop_cap);
    } catch (...) {
      stage.reset();  // joins the stager thread
      if (dd.nready) cudaStreamSynchronize(ctx.copy());
      throw;
    }
    if (stage && stage->stager) stage->stager->join();
    if (dd.nready) DFM_CUDA(cudaStreamSynchronize(ctx.copy()));
    spec.join();
    finish(ctx, o, dd.n, whole, block_out, nb_out, st, spec.started, &gate);
  });
}

uint64_t sm_draw(uint64_t seed, uint64_t j) {
  uint64_t z = seed + (j + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

// host -> device copy of a possibly pageable buffer (synchronous for the host when
// pageable; asynchronous on `stream` when pinned)
void h2d_rows(Ctx& ctx, void* dst, const void* src, uint64_t bytes) {
  h2d_batch(ctx, {H2DPiece{dst, src, bytes}});
}

// several host pieces in one go: pinned ones are DMA'd directly, pageable ones go
// through ONE pinned ring back to back (the copy of slot s+1 overlaps the DMA of
// slot s across piece boundaries), one synchronisation at the end
void h2d_batch(Ctx& ctx, const std::vector<H2DPiece>& pieces) {
  cudaStream_t stream = ctx.stream;
  const uint64_t slot = 64ull << 20;
  char* ring = nullptr;
  std::unique_ptr<StageRes> holder;
  StageRes* res = nullptr;
  for (const H2DPiece& p : pieces) {
    if (p.bytes == 0) continue;
    if (p.bytes < (16u << 20) || host_pinned_ptr(p.src)) {
      DFM_CUDA(cudaMemcpyAsync(p.dst, p.src, p.bytes, cudaMemcpyHostToDevice, stream));
      continue;
    }
    if (ring == nullptr) {
      ring = static_cast<char*>(ctx.host_pinned(kRing * slot));
      res = &new_stage_res(holder);
    }
    staged_h2d(ctx, p.dst, p.src, p.bytes, stream, ring, slot, *res);
  }
  if (ring) DFM_CUDA(cudaStreamSynchronize(stream));  // the ring is reused by the next call
}

}  // namespace dfm

using namespace dfm;

extern "C" {

const char* dfm_version(void) { return "libdfm 2 (B200 sm_100a)"; }

int dfm_ctx_create(int device, dfm_ctx** out) {
  if (out == nullptr) return DFM_ERR_INVALID;
  try {
    Ctx* ctx = new Ctx(device);
    if (const char* e = std::getenv("DFM_SORTPR_ENGINE"))
      ctx->sortpr_engine = std::strcmp(e, "radix") == 0 ? DFM_SORTPR_RADIX : DFM_SORTPR_HASH;
    *out = reinterpret_cast<dfm_ctx*>(ctx);
    return DFM_OK;
  } catch (const Error& e) {
    g_create_error = e.what();
    *out = nullptr;
    return e.code;
  }
}

void dfm_ctx_destroy(dfm_ctx* c) { delete as_ctx(c); }

const char* dfm_last_error(const dfm_ctx* c) {
  if (c == nullptr) return g_create_error.c_str();
  return as_ctx(c)->last_error.c_str();
}

int dfm_ctx_set_stream(dfm_ctx* c, void* stream) {
  return guarded(c, [&](Ctx& ctx) {
    ctx.sync();
    ctx.stream = stream ? static_cast<cudaStream_t>(stream) : ctx.own_stream;
  });
}

int dfm_ctx_set_sortpr_engine(dfm_ctx* c, int engine) {
  return guarded(c, [&](Ctx& ctx) {
    if (engine != DFM_SORTPR_HASH && engine != DFM_SORTPR_RADIX)
      throw Error(DFM_ERR_INVALID, "unknown sortPR engine");
    ctx.sortpr_engine = engine;
  });
}

int dfm_ctx_set_out_ready_hook(dfm_ctx* c, dfm_out_ready_fn ready, void* user) {
  return guarded(c, [&](Ctx& ctx) {
    ctx.out_ready = ready;
    ctx.out_user = ready ? user : nullptr;
  });
}

int dfm_ctx_set_trans_engine(dfm_ctx* c, int engine) {
  return guarded(c, [&](Ctx& ctx) {
    if (engine < DFM_TRANS_AUTO || engine > DFM_TRANS_TENSOR)
      throw Error(DFM_ERR_INVALID, "unknown Cho-Huynh engine");
    ctx.trans_engine = engine;
  });
}

int dfm_ctx_set_profiling(dfm_ctx* c, int enabled) {
  return guarded(c, [&](Ctx& ctx) { ctx.profiling = enabled != 0; });
}

int dfm_profile_get(dfm_ctx* c, const char* name, uint64_t* launches, double* total_ms,
                    uint64_t* algo_bytes) {
  int found = 0;
  const int rc = guarded(c, [&](Ctx& ctx) {
    auto it = ctx.prof.find(name ? name : "");
    if (it == ctx.prof.end()) return;
    found = 1;
    if (launches) *launches = it->second.launches;
    if (total_ms) *total_ms = it->second.ms;
    if (algo_bytes) *algo_bytes = it->second.bytes;
  });
  if (rc != DFM_OK) return rc;
  return found ? DFM_OK : DFM_ERR_INVALID;
}

const char* dfm_profile_names(dfm_ctx* c) {
  if (c == nullptr) return "";
  return as_ctx(c)->prof_names.c_str();
}

int dfm_profile_reset(dfm_ctx* c) {
  return guarded(c, [&](Ctx& ctx) {
    ctx.harvest();
    ctx.prof.clear();
    ctx.prof_names.clear();
  });
}

uint64_t dfm_kernel_launches(void) { return launch_count(); }

uint64_t dfm_ctx_device_bytes(const dfm_ctx* c) { return c ? as_ctx(c)->held_bytes : 0; }

int dfm_sort_pr(dfm_ctx* c, const dfm_dfa* d, int64_t timeout_ms, const dfm_trace* trace,
                uint32_t* block_out, uint32_t* nb, dfm_stats* st) {
  const dfm_limits lim{16ull << 30, timeout_ms};
  return run_host(c, DFM_ALGO_SORT, d, DFM_POLICY_ARBITRARY, &lim, trace, nullptr, nullptr, 0,
                  block_out, nb, st);
}

int dfm_naive_pr(dfm_ctx* c, const dfm_dfa* d, int32_t policy, int64_t timeout_ms,
                 const dfm_trace* trace, uint32_t* block_out, uint32_t* nb, dfm_stats* st) {
  const dfm_limits lim{16ull << 30, timeout_ms};
  return run_host(c, DFM_ALGO_NAIVE, d, policy, &lim, trace, nullptr, nullptr, 0, block_out, nb,
                  st);
}

int dfm_naive_pr_cas(dfm_ctx* c, const dfm_dfa* d, int64_t timeout_ms, const dfm_trace* trace,
                     uint32_t* block_out, uint32_t* nb, dfm_stats* st) {
  const dfm_limits lim{16ull << 30, timeout_ms};
  return run_host(c, DFM_ALGO_NAIVE_CAS, d, DFM_POLICY_ARBITRARY, &lim, trace, nullptr, nullptr,
                  0, block_out, nb, st);
}

uint32_t dfm_power_levels(uint32_t n) { return n == 0 ? 0 : 32 - __builtin_clz(n); }

uint64_t dfm_expand_required_bytes(uint32_t n, uint32_t k) {
  return (uint64_t)dfm_power_levels(n) * k * n * 4;
}

int dfm_expand_alphabet(dfm_ctx* c, const dfm_dfa* d, uint64_t max_memory_bytes,
                        uint32_t* rows_out, uint32_t* levels_out, uint64_t* required_out) {
  int capacity = 0;
  const int rc = guarded(c, [&](Ctx& ctx) {
    check_host_dfa(d);
    const uint64_t required = dfm_expand_required_bytes(d->num_states, d->alphabet_size);
    if (required_out) *required_out = required;
    if (required > max_memory_bytes) {  // CapacityError, min_transpr.hpp:63-67
      capacity = 1;
      ctx.last_error = "alphabet expansion needs " + std::to_string(required) +
                       " bytes, limit is " + std::to_string(max_memory_bytes);
      return;
    }
    const uint32_t levels = dfm_power_levels(d->num_states);
    if (levels_out) *levels_out = levels;
    if (rows_out == nullptr) return;
    const DevDfa dd = upload(ctx, d, "in", false);
    const uint32_t* rows = expand_alphabet_dev(ctx, dd, levels);
    DFM_CUDA(cudaMemcpyAsync(rows_out, rows, required, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
  });
  if (rc != DFM_OK) return rc;
  return capacity ? DFM_ERR_CAPACITY : DFM_OK;
}

int dfm_trans_pr(dfm_ctx* c, const dfm_dfa* d, int32_t policy, const dfm_limits* l,
                 uint32_t* block_out, uint32_t* nb, dfm_stats* st) {
  return run_host(c, DFM_ALGO_TRANSPR, d, policy, l, nullptr, nullptr, nullptr, 0, block_out, nb,
                  st);
}

uint64_t dfm_trans_required_bytes(uint64_t n) {
  const unsigned __int128 bits = (unsigned __int128)n * n * n * n;
  const unsigned __int128 bytes = (bits + 7) / 8;
  return bytes > (unsigned __int128)UINT64_MAX ? UINT64_MAX : (uint64_t)bytes;
}

int dfm_trans_minimize(dfm_ctx* c, const dfm_dfa* d, const dfm_limits* l, uint8_t* apart_out,
                       uint64_t* popcounts_out, uint32_t popcounts_cap, uint32_t* block_out,
                       uint32_t* nb, dfm_stats* st) {
  return run_host(c, DFM_ALGO_TRANS, d, DFM_POLICY_ARBITRARY, l, nullptr, apart_out,
                  popcounts_out, popcounts_cap, block_out, nb, st);
}

int dfm_run_algorithm(dfm_ctx* c, int32_t algo, const dfm_dfa* d, int32_t policy,
                      const dfm_limits* l, uint32_t* block_out, uint32_t* nb, dfm_stats* st) {
  return run_host(c, algo, d, policy, l, nullptr, nullptr, nullptr, 0, block_out, nb, st);
}

int dfm_ddfa_upload(dfm_ctx* c, const dfm_dfa* d, dfm_ddfa** out) {
  if (out == nullptr) return DFM_ERR_INVALID;
  *out = nullptr;
  return guarded(c, [&](Ctx& ctx) {
    DevDfa* dd = new DevDfa(upload(ctx, d, "", true));
    ctx.sync();
    *out = reinterpret_cast<dfm_ddfa*>(dd);
  });
}

int dfm_ddfa_random(dfm_ctx* c, uint32_t n, uint32_t k, uint64_t seed, double p, dfm_ddfa** out) {
  if (out == nullptr) return DFM_ERR_INVALID;
  *out = nullptr;
  return guarded(c, [&](Ctx& ctx) {
    if (n < 1 || k < 1) throw Error(DFM_ERR_INVALID, "random_dfa needs n >= 1 and k >= 1");
    DevDfa* dd = new DevDfa();
    dd->n = n;
    dd->k = k;
    dd->owns = true;
    try {
      DFM_CUDA(cudaMalloc(&dd->delta, (uint64_t)n * k * 4));
      DFM_CUDA(cudaMalloc(&dd->acc, n));
      random_dfa_dev(ctx, *dd, n, k, seed, p);
      ctx.sync();
    } catch (...) {
      cudaFree(dd->delta);
      cudaFree(dd->acc);
      delete dd;
      throw;
    }
    *out = reinterpret_cast<dfm_ddfa*>(dd);
  });
}

int dfm_ddfa_download(dfm_ctx* c, const dfm_ddfa* d, uint32_t* delta_flat, uint8_t* accepting) {
  return guarded(c, [&](Ctx& ctx) {
    const DevDfa* dd = as_dd(d);
    if (dd == nullptr) throw Error(DFM_ERR_INVALID, "null device dfa");
    if (delta_flat)
      DFM_CUDA(cudaMemcpyAsync(delta_flat, dd->delta, (uint64_t)dd->n * dd->k * 4,
                               cudaMemcpyDeviceToHost, ctx.stream));
    if (accepting)
      DFM_CUDA(cudaMemcpyAsync(accepting, dd->acc, dd->n, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
  });
}

int dfm_ddfa_shape(const dfm_ddfa* d, uint32_t* n, uint32_t* k) {
  const DevDfa* dd = as_dd(d);
  if (dd == nullptr) return DFM_ERR_INVALID;
  if (n) *n = dd->n;
  if (k) *k = dd->k;
  return DFM_OK;
}

void dfm_ddfa_free(dfm_ddfa* d) {
  DevDfa* dd = as_dd(d);
  if (dd == nullptr) return;
  if (dd->owns) {
    cudaFree(dd->delta);
    cudaFree(dd->acc);
  }
  delete dd;
}

int dfm_run_algorithm_dev(dfm_ctx* c, int32_t algo, const dfm_ddfa* d, int32_t policy,
                          const dfm_limits* l, void* block_out_dev, uint32_t* nb, dfm_stats* st) {
  return guarded(c, [&](Ctx& ctx) {
    const DevDfa* dd = as_dd(d);
    if (dd == nullptr) throw Error(DFM_ERR_INVALID, "null device dfa");
    const Deadline whole(0);
    const dfm_limits lim = limits_or_default(l);
    const AlgoOut o = dispatch(ctx, algo, *dd, policy, lim, nullptr, nullptr, nullptr, 0);
    if (o.status == DFM_STATUS_OK && block_out_dev != nullptr)
      DFM_CUDA(cudaMemcpyAsync(block_out_dev, o.canon_dev, (uint64_t)dd->n * 4,
                               cudaMemcpyDeviceToDevice, ctx.stream));
    finish(ctx, o, dd->n, whole, nullptr, nb, st);
  });
}

int dfm_quotient(dfm_ctx* c, const dfm_dfa* d, const uint32_t* block, uint32_t num_blocks,
                 uint32_t* delta_out, uint8_t* acc_out, uint32_t* initial_out) {
  return guarded(c, [&](Ctx& ctx) {
    if (block == nullptr) throw Error(DFM_ERR_INVALID, "null partition");
    const DevDfa dd = upload(ctx, d, "qt.in", false);
    uint32_t* blk = ctx.slot_t<uint32_t>("qt.block", dd.n);
    DFM_CUDA(cudaMemcpyAsync(blk, block, (uint64_t)dd.n * 4, cudaMemcpyHostToDevice, ctx.stream));
    DevDfa q = quotient_dev(ctx, dd, blk, num_blocks);
    if (delta_out)
      DFM_CUDA(cudaMemcpyAsync(delta_out, q.delta, (uint64_t)q.n * q.k * 4, cudaMemcpyDeviceToHost,
                               ctx.stream));
    if (acc_out)
      DFM_CUDA(cudaMemcpyAsync(acc_out, q.acc, q.n, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    if (initial_out) *initial_out = q.initial;
    cudaFree(q.delta);
    cudaFree(q.acc);
  });
}

int dfm_ddfa_quotient(dfm_ctx* c, const dfm_ddfa* d, const void* block_dev, uint32_t num_blocks,
                      dfm_ddfa** out) {
  if (out == nullptr) return DFM_ERR_INVALID;
  *out = nullptr;
  return guarded(c, [&](Ctx& ctx) {
    const DevDfa* dd = as_dd(d);
    if (dd == nullptr || block_dev == nullptr) throw Error(DFM_ERR_INVALID, "null input");
    DevDfa* q = new DevDfa(quotient_dev(ctx, *dd, static_cast<const uint32_t*>(block_dev),
                                        num_blocks));
    *out = reinterpret_cast<dfm_ddfa*>(q);
  });
}

int dfm_remove_unreachable(dfm_ctx* c, const dfm_dfa* d, uint32_t* num_states_out,
                           uint32_t* delta_out, uint8_t* acc_out, uint32_t* initial_out) {
  return guarded(c, [&](Ctx& ctx) {
    const DevDfa dd = upload(ctx, d, "ur.in", false);
    DevDfa r = remove_unreachable_dev(ctx, dd);
    if (delta_out)
      DFM_CUDA(cudaMemcpyAsync(delta_out, r.delta, (uint64_t)r.n * r.k * 4, cudaMemcpyDeviceToHost,
                               ctx.stream));
    if (acc_out)
      DFM_CUDA(cudaMemcpyAsync(acc_out, r.acc, r.n, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    if (num_states_out) *num_states_out = r.n;
    if (initial_out) *initial_out = r.initial;
    cudaFree(r.delta);
    cudaFree(r.acc);
  });
}

int dfm_ddfa_remove_unreachable(dfm_ctx* c, const dfm_ddfa* d, dfm_ddfa** out) {
  if (out == nullptr) return DFM_ERR_INVALID;
  *out = nullptr;
  return guarded(c, [&](Ctx& ctx) {
    const DevDfa* dd = as_dd(d);
    if (dd == nullptr) throw Error(DFM_ERR_INVALID, "null device dfa");
    DevDfa* r = new DevDfa(remove_unreachable_dev(ctx, *dd));
    *out = reinterpret_cast<dfm_ddfa*>(r);
  });
}

int dfm_write_dfa_bin(const char* path, const dfm_dfa* d) {
  if (path == nullptr) return DFM_ERR_INVALID;
  try {
    check_host_dfa(d);
    write_dfa_bin(path, d->num_states, d->alphabet_size, d->initial, d->delta, d->accepting);
    return DFM_OK;
  } catch (const Error& e) {
    g_create_error = e.what();
    return e.code;
  }
}

int dfm_ddfa_load_bin(dfm_ctx* c, const char* path, dfm_ddfa** out) {
  if (out == nullptr || path == nullptr) return DFM_ERR_INVALID;
  *out = nullptr;
  return guarded(c, [&](Ctx& ctx) {
    DevDfa* dd = new DevDfa(load_dfa_bin(ctx, path));
    try {
      validate_targets(ctx, *dd);
    } catch (...) {
      cudaFree(dd->delta);
      cudaFree(dd->acc);
      delete dd;
      throw;
    }
    *out = reinterpret_cast<dfm_ddfa*>(dd);
  });
}

int dfm_ddfa_save_bin(dfm_ctx* c, const dfm_ddfa* d, const char* path) {
  if (path == nullptr) return DFM_ERR_INVALID;
  return guarded(c, [&](Ctx& ctx) {
    const DevDfa* dd = as_dd(d);
    if (dd == nullptr) throw Error(DFM_ERR_INVALID, "null device dfa");
    save_dfa_bin(ctx, *dd, path);
  });
}

int dfm_ddfa_initial(const dfm_ddfa* d, uint32_t* initial) {
  const DevDfa* dd = as_dd(d);
  if (dd == nullptr || initial == nullptr) return DFM_ERR_INVALID;
  *initial = dd->initial;
  return DFM_OK;
}

int dfm_gen_random_dfa(uint32_t n, uint32_t k, uint64_t seed, double p, uint32_t* delta,
                       uint8_t* acc) {
  if (n < 1 || k < 1 || delta == nullptr || acc == nullptr) return DFM_ERR_INVALID;
  const uint64_t total = (uint64_t)n * k;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned T = (unsigned)std::min<uint64_t>(hw, std::max<uint64_t>(1, (total + n) >> 16));
  auto work = [&](unsigned t) {
    const uint64_t lo = total * t / T, hi = total * (t + 1) / T;
    for (uint64_t j = lo; j < hi; ++j) delta[j] = (uint32_t)(sm_draw(seed, j) % n);
    const uint64_t alo = (uint64_t)n * t / T, ahi = (uint64_t)n * (t + 1) / T;
    for (uint64_t q = alo; q < ahi; ++q)
      acc[q] = ((double)(sm_draw(seed, total + q) >> 11) * 0x1.0p-53) < p ? 1 : 0;
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  return DFM_OK;
}

}  // extern "C"
