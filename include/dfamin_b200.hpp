// dfamin_b200.hpp — header-only C++ host layer over the libdfm C-ABI (dfm.h).
//
// Mirrors the reference minimize entry points (proj/include/dfamin) with the
// same names, signatures, argument meaning and error behaviour, so the
// reference's callers switch by namespace:
//
//   dfamin::sort_pr(d, opt)          -> dfamin::b200::sort_pr(d, opt)        min_sort.hpp:72,:128
//   dfamin::naive_pr(d, opt|policy)  -> dfamin::b200::naive_pr(...)          min_partref.hpp:156,:160
//   dfamin::naive_pr_cas(d, t, tr)   -> dfamin::b200::naive_pr_cas(...)      min_partref.hpp:170
//   dfamin::expand_alphabet(d, lim)  -> dfamin::b200::expand_alphabet(...)   min_transpr.hpp:59 (throws CapacityError)
//   dfamin::trans_pr(...)            -> dfamin::b200::trans_pr(...)          min_transpr.hpp:90,:114
//   dfamin::trans_minimize(d,l,ins)  -> dfamin::b200::trans_minimize(...)    min_trans.hpp:81
//   dfamin::run_algorithm(a, d, cfg) -> dfamin::b200::run_algorithm(...)     bench.hpp:83
//   dfamin::sort_pr(d, opt)          -> dfamin::b200::sort_pr(d, sharded, opt) state-sharded over
//                                       the GPUs of one box (dfm_sort_pr_sharded)
//
// Types: with DFAMIN_B200_USE_REFERENCE_TYPES defined (and the reference
// headers dfamin/bench.hpp etc. included first) the functions take and return
// the reference's own Dfa/MinResult/... types — a true drop-in.  Otherwise
// this header provides structurally identical mirror types.
//
// Algorithmic outcomes (timeout, capacity) come back in RunStats.status with
// an empty partition, exactly like the reference.  Infrastructure faults
// (no GPU, CUDA error) throw dfamin::b200::EngineError: the engine never falls
// back to a CPU path.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#if defined(__linux__)
#include <sys/mman.h>
#endif

#include "dfm.h"

#ifdef DFAMIN_B200_USE_REFERENCE_TYPES
namespace dfamin::b200 {
using ::dfamin::Algo;
using ::dfamin::AlgoRunConfig;
using ::dfamin::CapacityError;
using ::dfamin::Dfa;
using ::dfamin::ExpandedDfa;
using ::dfamin::Limits;
using ::dfamin::MinResult;
using ::dfamin::Partition;
using ::dfamin::PrOptions;
using ::dfamin::PrTrace;
using ::dfamin::RunStats;
using ::dfamin::RunStatus;
using ::dfamin::SortOptions;
using ::dfamin::SortTrace;
using ::dfamin::State;
using ::dfamin::TransInspect;
using RacePolicy = ::dfamin::substrate::RacePolicy;
inline Partition canonicalize(const std::vector<std::uint32_t>& raw) {
  return ::dfamin::canonicalize(raw);
}
}  // namespace dfamin::b200
#else
namespace dfamin::b200 {
using State = std::uint32_t;
struct Dfa {  // core.hpp:24-33
  std::uint32_t num_states = 0;
  std::uint32_t alphabet_size = 0;
  std::vector<std::vector<State>> delta;
  std::vector<std::uint8_t> accepting;
  State initial = 0;
  bool is_accepting(State q) const { return accepting[q] != 0; }
};
struct Partition {  // core.hpp:52-56
  std::vector<std::uint32_t> block;
  std::uint32_t num_blocks = 0;
  bool operator==(const Partition&) const = default;
};
enum class RunStatus { ok, timeout, capacity_exceeded };  // core.hpp:58
struct RunStats {                                          // core.hpp:71-77
  std::uint64_t iterations = 0;
  std::uint64_t closure_steps = 0;
  double elapsed_ms = 0.0;
  std::uint64_t peak_memory_estimate = 0;
  RunStatus status = RunStatus::ok;
};
struct Limits {  // core.hpp:81-84
  std::uint64_t max_memory_bytes = std::uint64_t{16} << 30;
  std::int64_t timeout_ms = 300'000;
};
struct MinResult {  // core.hpp:87-90
  Partition partition;
  RunStats stats;
};
class CapacityError : public std::runtime_error {  // core.hpp:93-101
 public:
  CapacityError(const std::string& what, std::uint64_t required)
      : std::runtime_error(what), required_(required) {}
  std::uint64_t required_bytes() const { return required_; }

 private:
  std::uint64_t required_;
};
enum class RacePolicy { arbitrary_winner, deterministic_min, deterministic_max };  // substrate.hpp:24
struct SortTrace {                                                                // min_sort.hpp:21-24
  std::vector<Partition> partitions;
  std::vector<std::uint32_t> block_counts;
};
struct SortOptions {  // min_sort.hpp:26-29
  std::int64_t timeout_ms = 300'000;
  SortTrace* trace = nullptr;
};
struct PrTrace {  // min_partref.hpp:21-24
  std::vector<std::vector<std::uint32_t>> leader_arrays;
  std::vector<Partition> partitions;
};
struct PrOptions {  // min_partref.hpp:26-30
  RacePolicy policy = RacePolicy::arbitrary_winner;
  std::int64_t timeout_ms = 300'000;
  PrTrace* trace = nullptr;
};
struct TransInspect {  // min_trans.hpp:41-44
  std::vector<std::uint8_t> apart;
  std::vector<std::uint64_t> apart_popcounts;
};
struct ExpandedDfa {  // min_transpr.hpp:31-53
  std::uint32_t num_states = 0;
  std::uint32_t base_alphabet = 0;
  std::uint32_t levels = 0;
  std::vector<std::vector<State>> delta;
  std::vector<std::uint8_t> accepting;
  State initial = 0;
  const std::vector<State>& row(std::uint32_t letter, std::uint32_t level) const {
    return delta[static_cast<std::size_t>(level) * base_alphabet + letter];
  }
  Dfa as_dfa() const {
    return Dfa{num_states, static_cast<std::uint32_t>(delta.size()), delta, accepting, initial};
  }
};
enum class Algo { trans, naive, naive_cas, sort, transpr, oracle };  // bench.hpp:23
struct AlgoRunConfig {                                                // bench.hpp:78-81
  RacePolicy policy = RacePolicy::arbitrary_winner;
  Limits limits;
};
inline Partition canonicalize(const std::vector<std::uint32_t>& raw) {  // core.hpp:123-136
  Partition p;
  p.block.resize(raw.size());
  std::unordered_map<std::uint32_t, std::uint32_t> relabel;
  for (std::size_t i = 0; i < raw.size(); ++i) {
    auto [it, fresh] = relabel.try_emplace(raw[i], static_cast<std::uint32_t>(relabel.size()));
    (void)fresh;
    p.block[i] = it->second;
  }
  p.num_blocks = static_cast<std::uint32_t>(relabel.size());
  return p;
}
}  // namespace dfamin::b200
#endif

namespace dfamin::b200 {

class EngineError : public std::runtime_error {
 public:
  EngineError(int code, const std::string& what)
      : std::runtime_error("libdfm error " + std::to_string(code) + ": " + what), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

// One libdfm context per thread (the reference functions are re-entrant; a
// ctx serialises its own calls).  DFM_DEVICE selects the GPU (default 0).
class Engine {
 public:
  explicit Engine(int device = 0) {
    const int rc = dfm_ctx_create(device, &ctx_);
    if (rc != DFM_OK) throw EngineError(rc, dfm_last_error(nullptr));
  }
  ~Engine() { dfm_ctx_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  dfm_ctx* get() const { return ctx_; }
  void check(int rc) const {
    if (rc != DFM_OK) throw EngineError(rc, dfm_last_error(ctx_));
  }
  static Engine& thread_default() {
    thread_local std::unique_ptr<Engine> e;
    if (!e) {
      const char* s = std::getenv("DFM_DEVICE");
      e = std::make_unique<Engine>(s ? std::atoi(s) : 0);
    }
    return *e;
  }

 private:
  dfm_ctx* ctx_ = nullptr;
};

namespace detail {

struct View {
  std::vector<const std::uint32_t*> rows;
  dfm_dfa c{};
  explicit View(const Dfa& d) : rows(d.alphabet_size) {
    for (std::uint32_t a = 0; a < d.alphabet_size; ++a) rows[a] = d.delta[a].data();
    c.num_states = d.num_states;
    c.alphabet_size = d.alphabet_size;
    c.delta = rows.empty() ? nullptr : rows.data();
    c.accepting = d.accepting.data();
    c.initial = d.initial;
  }
};

// The partition vector a MinResult returns (core.hpp: Partition::block).  A value-
// initialised std::vector of 1e8 labels page-faults 400 MB of fresh mmap'd memory on
// one thread (~200 ms, more than the whole GPU minimization).  For large partitions
// the vector is reserved, its pages advised as huge pages and faulted in by several
// threads, and only then resized (the memset runs over resident memory) — all on a
// helper thread WHILE the library works: the library calls ready() (through the
// context's out-ready hook, dfm.h) before it first writes the buffer.
class OutPartition {
 public:
  explicit OutPartition(std::size_t n) {
    constexpr std::size_t kParallelBytes = std::size_t(64) << 20;
    if (n * sizeof(std::uint32_t) < kParallelBytes) {
      v_.resize(n);
      p_ = v_.data();
      return;
    }
    v_.reserve(n);
    p_ = v_.data();  // stable: resize() within the capacity does not reallocate
    th_ = std::thread([this, n] {
      prefault(p_, n);
      v_.resize(n);
    });
  }
  OutPartition(const OutPartition&) = delete;
  OutPartition& operator=(const OutPartition&) = delete;
  ~OutPartition() { ready(); }
  std::uint32_t* data() const { return p_; }
  void ready() {
    std::call_once(once_, [this] {
      if (th_.joinable()) th_.join();
    });
  }
  static void hook(void* self) { static_cast<OutPartition*>(self)->ready(); }
  std::vector<std::uint32_t> take() {
    ready();
    return std::move(v_);
  }

 private:
  static void prefault(std::uint32_t* p, std::size_t n) {
    const std::uintptr_t b = reinterpret_cast<std::uintptr_t>(p);
    const std::uintptr_t e = b + n * sizeof(std::uint32_t);
#if defined(__linux__) && defined(MADV_HUGEPAGE)
    const std::uintptr_t kHuge = std::uintptr_t(2) << 20;
    const std::uintptr_t hb = (b + kHuge - 1) & ~(kHuge - 1), he = e & ~(kHuge - 1);
    if (he > hb) madvise(reinterpret_cast<void*>(hb), he - hb, MADV_HUGEPAGE);
#endif
    const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    auto touch = [b, e, T](unsigned t) {
      const std::uintptr_t span = e - b;
      std::uintptr_t lo = b + (span * t / T + 4095) / 4096 * 4096;
      const std::uintptr_t hi = b + span * (t + 1) / T;
      for (; lo < hi; lo += 4096) *reinterpret_cast<volatile char*>(lo) = 0;
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back(touch, t);
    touch(0);
    for (auto& x : th) x.join();
  }
  std::vector<std::uint32_t> v_;
  std::uint32_t* p_ = nullptr;
  std::thread th_;
  std::once_flag once_;
};

// Arms the context's out-ready hook for one host-buffer call and disarms it after
// (the library consumes it at the start of the call; this covers a call that fails
// before reaching it).
struct OutHook {
  dfm_ctx* ctx;
  OutHook(dfm_ctx* c, OutPartition& out) : ctx(c) {
    dfm_ctx_set_out_ready_hook(ctx, &OutPartition::hook, &out);
  }
  ~OutHook() { dfm_ctx_set_out_ready_hook(ctx, nullptr, nullptr); }
};

inline MinResult result(std::vector<std::uint32_t>&& block, std::uint32_t nb, const dfm_stats& s) {
  MinResult r;
  r.stats.iterations = s.iterations;
  r.stats.closure_steps = s.closure_steps;
  r.stats.elapsed_ms = s.elapsed_ms;
  r.stats.peak_memory_estimate = s.peak_memory_estimate;
  r.stats.status = static_cast<RunStatus>(s.status);
  if (r.stats.status == RunStatus::ok) {
    r.partition.block = std::move(block);
    r.partition.num_blocks = nb;
  }
  return r;
}

inline std::int32_t policy_of(RacePolicy p) {
  switch (p) {
    case RacePolicy::deterministic_min: return DFM_POLICY_MIN;
    case RacePolicy::deterministic_max: return DFM_POLICY_MAX;
    default: return DFM_POLICY_ARBITRARY;
  }
}

inline void on_sort_pass(void* user, std::uint64_t, const std::uint32_t* raw, std::uint32_t n,
                         std::uint32_t count) {
  auto* t = static_cast<SortTrace*>(user);
  t->partitions.push_back(canonicalize(std::vector<std::uint32_t>(raw, raw + n)));
  t->block_counts.push_back(count);
}

inline void on_pr_pass(void* user, std::uint64_t, const std::uint32_t* raw, std::uint32_t n,
                       std::uint32_t) {
  auto* t = static_cast<PrTrace*>(user);
  t->leader_arrays.emplace_back(raw, raw + n);
  t->partitions.push_back(canonicalize(t->leader_arrays.back()));
}

}  // namespace detail

inline MinResult sort_pr(const Dfa& d, const SortOptions& opt = {}) {
  Engine& e = Engine::thread_default();
  detail::View v(d);
  detail::OutPartition block(d.num_states);
  std::uint32_t nb = 0;
  dfm_stats st{};
  dfm_trace tr{&detail::on_sort_pass, opt.trace};
  {
    detail::OutHook hook(e.get(), block);
    e.check(dfm_sort_pr(e.get(), &v.c, opt.timeout_ms, opt.trace ? &tr : nullptr, block.data(),
                        &nb, &st));
  }
  return detail::result(block.take(), nb, st);
}

inline MinResult sort_pr(const Dfa& d, std::int64_t timeout_ms) {
  SortOptions opt;
  opt.timeout_ms = timeout_ms;
  return ::dfamin::b200::sort_pr(d, opt);
}

inline MinResult naive_pr(const Dfa& d, const PrOptions& opt = {}) {
  Engine& e = Engine::thread_default();
  detail::View v(d);
  detail::OutPartition block(d.num_states);
  std::uint32_t nb = 0;
  dfm_stats st{};
  dfm_trace tr{&detail::on_pr_pass, opt.trace};
  {
    detail::OutHook hook(e.get(), block);
    e.check(dfm_naive_pr(e.get(), &v.c, detail::policy_of(opt.policy), opt.timeout_ms,
                         opt.trace ? &tr : nullptr, block.data(), &nb, &st));
  }
  return detail::result(block.take(), nb, st);
}

inline MinResult naive_pr(const Dfa& d, RacePolicy policy, std::int64_t timeout_ms = 300'000) {
  PrOptions opt;
  opt.policy = policy;
  opt.timeout_ms = timeout_ms;
  return ::dfamin::b200::naive_pr(d, opt);
}

inline MinResult naive_pr_cas(const Dfa& d, std::int64_t timeout_ms = 300'000,
                              PrTrace* trace = nullptr) {
  Engine& e = Engine::thread_default();
  detail::View v(d);
  detail::OutPartition block(d.num_states);
  std::uint32_t nb = 0;
  dfm_stats st{};
  dfm_trace tr{&detail::on_pr_pass, trace};
  {
    detail::OutHook hook(e.get(), block);
    e.check(dfm_naive_pr_cas(e.get(), &v.c, timeout_ms, trace ? &tr : nullptr, block.data(),
                             &nb, &st));
  }
  return detail::result(block.take(), nb, st);
}

inline std::uint32_t power_levels(std::uint32_t n) { return dfm_power_levels(n); }
inline std::uint64_t expand_required_bytes(std::uint32_t n, std::uint32_t k) {
  return dfm_expand_required_bytes(n, k);
}

inline ExpandedDfa expand_alphabet(const Dfa& d, const Limits& limits = {}) {
  Engine& e = Engine::thread_default();
  detail::View v(d);
  const std::uint64_t required = expand_required_bytes(d.num_states, d.alphabet_size);
  if (required > limits.max_memory_bytes)  // min_transpr.hpp:63-67
    throw CapacityError("alphabet expansion needs " + std::to_string(required) +
                            " bytes, limit is " + std::to_string(limits.max_memory_bytes),
                        required);
  std::vector<std::uint32_t> flat(required / 4);
  std::uint32_t levels = 0;
  std::uint64_t req = 0;
  const int rc = dfm_expand_alphabet(e.get(), &v.c, limits.max_memory_bytes, flat.data(), &levels,
                                     &req);
  if (rc == DFM_ERR_CAPACITY) throw CapacityError(dfm_last_error(e.get()), req);
  e.check(rc);
  ExpandedDfa x;
  x.num_states = d.num_states;
  x.base_alphabet = d.alphabet_size;
  x.levels = levels;
  x.accepting = d.accepting;
  x.initial = d.initial;
  x.delta.resize(static_cast<std::size_t>(levels) * d.alphabet_size);
  for (std::size_t r = 0; r < x.delta.size(); ++r)
    x.delta[r].assign(flat.begin() + r * d.num_states, flat.begin() + (r + 1) * d.num_states);
  return x;
}

inline MinResult trans_pr(const Dfa& d, const PrOptions& opt = {}, const Limits& limits = {}) {
  Engine& e = Engine::thread_default();
  detail::View v(d);
  detail::OutPartition block(d.num_states);
  std::uint32_t nb = 0;
  dfm_stats st{};
  const dfm_limits lim{limits.max_memory_bytes, opt.timeout_ms};
  {
    detail::OutHook hook(e.get(), block);
    e.check(dfm_trans_pr(e.get(), &v.c, detail::policy_of(opt.policy), &lim, block.data(), &nb,
                         &st));
  }
  return detail::result(block.take(), nb, st);
}

inline MinResult trans_pr(const Dfa& d, RacePolicy policy, std::int64_t timeout_ms = 300'000,
                          const Limits& limits = {}) {
  PrOptions opt;
  opt.policy = policy;
  opt.timeout_ms = timeout_ms;
  Limits lim = limits;
  lim.timeout_ms = timeout_ms;
  return ::dfamin::b200::trans_pr(d, opt, lim);
}

inline std::uint64_t trans_required_bytes_u64(std::uint64_t n) { return dfm_trans_required_bytes(n); }

inline MinResult trans_minimize(const Dfa& d, const Limits& limits = {},
                                TransInspect* inspect = nullptr) {
  Engine& e = Engine::thread_default();
  detail::View v(d);
  const std::size_t n = d.num_states;
  detail::OutPartition block(n);
  std::uint32_t nb = 0;
  dfm_stats st{};
  const dfm_limits lim{limits.max_memory_bytes, limits.timeout_ms};
  std::vector<std::uint8_t> apart;
  std::vector<std::uint64_t> pops;
  if (inspect) {
    apart.resize(n * n);
    pops.resize(4096);
  }
  {
    detail::OutHook hook(e.get(), block);
    e.check(dfm_trans_minimize(e.get(), &v.c, &lim, inspect ? apart.data() : nullptr,
                               inspect ? pops.data() : nullptr, inspect ? 4096u : 0u,
                               block.data(), &nb, &st));
  }
  MinResult r = detail::result(block.take(), nb, st);
  if (inspect && r.stats.status == RunStatus::ok) {
    inspect->apart = std::move(apart);
    inspect->apart_popcounts.assign(pops.begin(), pops.begin() + r.stats.iterations);
  }
  return r;
}

// quotient, core.hpp:256-290: throws std::invalid_argument with the reference's
// message for a non-canonical or inconsistent partition
inline Dfa quotient(const Dfa& d, const Partition& p) {
  if (p.block.size() != d.num_states)
    throw std::invalid_argument("partition covers a different state count");
  Engine& e = Engine::thread_default();
  detail::View v(d);
  const std::uint32_t nb = p.num_blocks;
  std::vector<std::uint32_t> flat((std::size_t)d.alphabet_size * nb);
  Dfa out;
  out.num_states = nb;
  out.alphabet_size = d.alphabet_size;
  out.accepting.assign(nb, 0);
  std::uint32_t init = 0;
  const int rc = dfm_quotient(e.get(), &v.c, p.block.data(), nb, flat.data(), out.accepting.data(),
                              &init);
  if (rc == DFM_ERR_INVALID) throw std::invalid_argument(dfm_last_error(e.get()));
  e.check(rc);
  out.delta.assign(d.alphabet_size, std::vector<State>(nb));
  for (std::uint32_t a = 0; a < d.alphabet_size; ++a)
    std::copy(flat.begin() + (std::size_t)a * nb, flat.begin() + (std::size_t)(a + 1) * nb,
              out.delta[a].begin());
  out.initial = init;
  return out;
}

// remove_unreachable, core.hpp:152-187
inline Dfa remove_unreachable(const Dfa& d) {
  Engine& e = Engine::thread_default();
  detail::View v(d);
  std::vector<std::uint32_t> flat((std::size_t)d.alphabet_size * d.num_states);
  std::vector<std::uint8_t> acc(d.num_states);
  std::uint32_t kept = 0, init = 0;
  e.check(dfm_remove_unreachable(e.get(), &v.c, &kept, flat.data(), acc.data(), &init));
  Dfa out;
  out.num_states = kept;
  out.alphabet_size = d.alphabet_size;
  out.delta.assign(d.alphabet_size, std::vector<State>(kept));
  for (std::uint32_t a = 0; a < d.alphabet_size; ++a)
    std::copy(flat.begin() + (std::size_t)a * kept, flat.begin() + (std::size_t)(a + 1) * kept,
              out.delta[a].begin());
  out.accepting.assign(acc.begin(), acc.begin() + kept);
  out.initial = init;
  return out;
}

inline MinResult run_algorithm(Algo algo, const Dfa& d, const AlgoRunConfig& cfg = {}) {
  switch (algo) {  // bench.hpp:83-112
    case Algo::trans: return ::dfamin::b200::trans_minimize(d, cfg.limits);
    case Algo::naive: {
      PrOptions opt;
      opt.policy = cfg.policy;
      opt.timeout_ms = cfg.limits.timeout_ms;
      return ::dfamin::b200::naive_pr(d, opt);
    }
    case Algo::naive_cas: return ::dfamin::b200::naive_pr_cas(d, cfg.limits.timeout_ms);
    case Algo::sort: return ::dfamin::b200::sort_pr(d, cfg.limits.timeout_ms);
    case Algo::transpr: {
      PrOptions opt;
      opt.policy = cfg.policy;
      opt.timeout_ms = cfg.limits.timeout_ms;
      return ::dfamin::b200::trans_pr(d, opt, cfg.limits);
    }
    default:
      throw std::invalid_argument("the Moore oracle is a CPU reference, not a GPU algorithm");
  }
}

// ---- state-sharded sortPR: one process per GPU over NCCL, or (tests)
// one thread per rank over the in-process transport.  Collective: every rank calls.
class ShardedEngine {
 public:
  using NcclId = std::array<std::uint8_t, DFM_NCCL_ID_BYTES>;
  // rank 0 creates the id; the host distributes its bytes to the other ranks
  static NcclId nccl_unique_id() {
    NcclId id{};
    const int rc = dfm_nccl_get_unique_id(id.data());
    if (rc != DFM_OK) throw EngineError(rc, "ncclGetUniqueId failed");
    return id;
  }
  ShardedEngine(int device, int rank, int world, const NcclId& id) {
    const int rc = dfm_ctx_create_sharded(device, rank, world, id.data(), &ctx_);
    if (rc != DFM_OK) throw EngineError(rc, dfm_last_error(nullptr));
  }
  ShardedEngine(int device, int rank, int world, const std::string& local_group) {
    const int rc = dfm_ctx_create_sharded_local(device, rank, world, local_group.c_str(), &ctx_);
    if (rc != DFM_OK) throw EngineError(rc, dfm_last_error(nullptr));
  }
  ~ShardedEngine() { dfm_ctx_destroy(ctx_); }
  ShardedEngine(const ShardedEngine&) = delete;
  ShardedEngine& operator=(const ShardedEngine&) = delete;
  dfm_ctx* get() const { return ctx_; }
  void check(int rc) const {
    if (rc != DFM_OK) throw EngineError(rc, dfm_last_error(ctx_));
  }
  int rank() const {
    int r = 0;
    dfm_ctx_shard_info(ctx_, &r, nullptr, nullptr);
    return r;
  }
  int world() const {
    int w = 1;
    dfm_ctx_shard_info(ctx_, nullptr, &w, nullptr);
    return w;
  }
  // this rank's states [lo, hi)
  std::pair<std::uint64_t, std::uint64_t> bounds(std::uint64_t n) const {
    std::uint64_t lo = 0, hi = 0;
    dfm_shard_bounds(n, world(), rank(), &lo, &hi);
    return {lo, hi};
  }

 private:
  dfm_ctx* ctx_ = nullptr;
};

// sort_pr (min_sort.hpp:72) over state shards.  Every rank passes the same Dfa (the
// reference type); the engine reads only this rank's rows [lo, hi) (pointers into
// the row vectors, no copy on the host) and returns the whole canonical partition,
// block count and pass count — equal to the reference's — on every rank.
inline MinResult sort_pr(const Dfa& d, ShardedEngine& se, const SortOptions& opt = {}) {
  const auto [lo, hi] = se.bounds(d.num_states);
  std::vector<const std::uint32_t*> rows(d.alphabet_size);
  for (std::uint32_t a = 0; a < d.alphabet_size; ++a) rows[a] = d.delta[a].data() + lo;
  dfm_dfa local{};
  local.num_states = static_cast<std::uint32_t>(hi - lo);
  local.alphabet_size = d.alphabet_size;
  local.delta = rows.empty() ? nullptr : rows.data();
  local.accepting = d.accepting.data() + lo;
  local.initial = 0;
  detail::OutPartition block(d.num_states);
  block.ready();  // (the sharded entry has no out-ready hook)
  std::uint32_t nb = 0;
  dfm_stats st{};
  se.check(dfm_sort_pr_sharded(se.get(), d.num_states, &local, 1, block.data(), &nb,
                               opt.timeout_ms, &st));
  return detail::result(block.take(), nb, st);
}

}  // namespace dfamin::b200
