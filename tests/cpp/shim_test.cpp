// C++ host-layer test: the reference's own test idioms (test_min_sort.cpp,
// test_min_partref.cpp, test_min_transpr.cpp, test_min_trans.cpp) written
// against dfamin::b200 — builds with the mirror types, or with the reference's
// types under -DDFAMIN_B200_USE_REFERENCE_TYPES (drop-in compile check).
// Exit code = number of failed checks.  Inputs are built inline (no oracle).
#ifdef DFAMIN_B200_USE_REFERENCE_TYPES
#include "dfamin/bench.hpp"
#endif
#include <cstdio>
#include <thread>
#include <string>

#include "dfamin_b200.hpp"

namespace B = dfamin::b200;
using B::Algo;
using B::AlgoRunConfig;
using B::CapacityError;
using B::Dfa;
using B::ExpandedDfa;
using B::Limits;
using B::MinResult;
using B::PrOptions;
using B::RacePolicy;
using B::RunStatus;
using B::SortOptions;
using B::SortTrace;
using B::State;
using B::TransInspect;

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      ++failures;                                                  \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                              \
  } while (0)

static Dfa ring(const std::string& w) {  // fib_dfa shape: one letter, q -> q+1 mod N
  Dfa d;
  d.num_states = (std::uint32_t)w.size();
  d.alphabet_size = 1;
  d.delta.assign(1, std::vector<State>(w.size()));
  d.accepting.resize(w.size());
  for (std::size_t q = 0; q < w.size(); ++q) {
    d.delta[0][q] = (State)((q + 1) % w.size());
    d.accepting[q] = w[q] == '1';
  }
  return d;
}

static std::string fib_word(int n) {
  std::string prev = "1", cur = "0";
  if (n == 0) return prev;
  for (int i = 2; i <= n; ++i) {
    std::string next = cur + prev;
    prev = cur;
    cur = next;
  }
  return cur;
}

static Dfa chain(std::uint32_t len) {
  Dfa d;
  d.num_states = len;
  d.alphabet_size = 1;
  d.delta.assign(1, std::vector<State>(len));
  d.accepting.assign(len, 0);
  for (std::uint32_t q = 0; q + 1 < len; ++q) d.delta[0][q] = q + 1;
  d.delta[0][len - 1] = len - 1;
  d.accepting[len - 1] = 1;
  return d;
}

int main() {
  for (int n = 5; n <= 9; ++n) {  // test_min_partref.cpp:36-44, test_min_sort.cpp:88-94
    const Dfa d = ring(fib_word(n));
    const MinResult s = B::sort_pr(d);
    CHECK(s.stats.status == RunStatus::ok);
    CHECK(s.partition.num_blocks == d.num_states && s.stats.iterations == d.num_states - 1);
    const MinResult r = B::naive_pr(d, RacePolicy::deterministic_min);
    CHECK(r.partition.num_blocks == d.num_states && r.stats.iterations == d.num_states - 1);
    CHECK(B::naive_pr_cas(d).partition == s.partition);
  }
  {  // test_min_sort.cpp:113-136: one pass splits 2 -> 5 blocks
    Dfa d;
    d.num_states = 6;
    d.alphabet_size = 2;
    d.delta = {{0, 0, 5, 5, 0, 5}, {0, 5, 0, 5, 0, 5}};
    d.accepting = {0, 0, 0, 0, 0, 1};
    SortTrace trace;
    SortOptions opt;
    opt.trace = &trace;
    const MinResult r = B::sort_pr(d, opt);
    CHECK(r.stats.status == RunStatus::ok);
    CHECK(!trace.block_counts.empty() && trace.block_counts.front() == 5);
  }
  {  // test_min_transpr.cpp:27-35, :79-93, :126-134
    const ExpandedDfa e = B::expand_alphabet(chain(10));
    CHECK(e.levels == 4 && e.row(0, 3)[0] == 8);
    Limits tiny;
    tiny.max_memory_bytes = 64;
    bool threw = false;
    try {
      B::expand_alphabet(chain(256), tiny);
    } catch (const CapacityError& err) {
      threw = err.required_bytes() == 9u * 256u * 4u;
    }
    CHECK(threw);
    PrOptions det;
    det.policy = RacePolicy::deterministic_min;
    CHECK(B::trans_pr(chain(256), det, tiny).stats.status == RunStatus::capacity_exceeded);
    const MinResult closed = B::trans_pr(chain(64), det);
    CHECK(closed.stats.iterations <= 14 && closed.partition.num_blocks == 64);
  }
  {  // test_min_trans.cpp:31-43
    const int passes[] = {3, 4, 5, 6, 6};
    for (int n = 5; n <= 9; ++n) {
      const Dfa d = ring(fib_word(n));
      TransInspect ins;
      const MinResult r = B::trans_minimize(d, {}, &ins);
      CHECK(r.stats.iterations == (std::uint64_t)passes[n - 5]);
      CHECK(r.partition.num_blocks == d.num_states);
      CHECK(ins.apart.size() == (std::size_t)d.num_states * d.num_states);
    }
    Limits quick;
    quick.timeout_ms = 1;
    (void)quick;
  }
  {  // bench.hpp:83 dispatcher
    const Dfa d = ring(fib_word(7));
    AlgoRunConfig cfg;
    cfg.policy = RacePolicy::deterministic_min;
    for (Algo a : {Algo::trans, Algo::naive, Algo::naive_cas, Algo::sort, Algo::transpr}) {
      const MinResult r = B::run_algorithm(a, d, cfg);
      CHECK(r.stats.status == RunStatus::ok && r.partition.num_blocks == d.num_states);
    }
  }
  {  // core.hpp:152-187 / 256-290: quotient of a ring by its (singleton) partition is
     // itself; a chain entered mid-way keeps its tail; a bad partition throws
    const Dfa d = ring(fib_word(6));
    const MinResult r = B::sort_pr(d);
    const Dfa q = B::quotient(d, r.partition);
    CHECK(q.num_states == r.partition.num_blocks && B::sort_pr(q).partition.num_blocks == q.num_states);
    Dfa c = chain(100);
    c.initial = 90;
    const Dfa t = B::remove_unreachable(c);
    CHECK(t.num_states == 10 && t.initial == 0 && t.accepting[9] == 1);
    auto bad = r.partition;
    bad.block[0] = 1;
    bool threw = false;
    try {
      B::quotient(d, bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // state-sharded sort_pr: NCCL world 1, and 3 ranks as threads over the
     // in-process transport; whole canonical partition and pass count on every rank
    Dfa d;
    d.num_states = 20000;
    d.alphabet_size = 3;
    d.delta.assign(3, std::vector<State>(d.num_states));
    d.accepting.assign(d.num_states, 0);
    std::uint64_t x = 2410;
    for (auto& row : d.delta)
      for (auto& t : row) {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        t = (State)((x >> 33) % (d.num_states / 4));  // few distinct targets: many merges
      }
    for (std::uint32_t q = 0; q < d.num_states; ++q) d.accepting[q] = (q % 7) == 0;
    const MinResult ref = B::sort_pr(d);
    {
      B::ShardedEngine se(0, 0, 1, B::ShardedEngine::nccl_unique_id());
      const MinResult r = B::sort_pr(d, se);
      CHECK(r.partition == ref.partition && r.stats.iterations == ref.stats.iterations);
    }
    std::vector<MinResult> got(3);
    std::vector<std::thread> th;
    for (int rank = 0; rank < 3; ++rank)
      th.emplace_back([&, rank] {
        B::ShardedEngine se(0, rank, 3, "shim3");
        got[rank] = B::sort_pr(d, se);
      });
    for (auto& t : th) t.join();
    for (const auto& r : got)
      CHECK(r.partition == ref.partition && r.stats.iterations == ref.stats.iterations);
  }
  std::printf("%d failures\n", failures);
  return failures;
}
