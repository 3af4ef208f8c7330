// TEST INFRASTRUCTURE ONLY — a C-ABI wrapper around the UNMODIFIED reference
// `dfamin` headers (compiled from /root/reference/proj/include by
// oracle/Makefile into oracle/_ref/libdfamin_ref.so).  Used to pin the oracle
// restatement (tests/golden/make_golden.py) and as bench.py's cpu_baseline /
// `--impl reference` arm.  No reference source is copied: this file only
// converts flat C buffers to the reference's types and calls its public API
// (min_sort.hpp:72, min_partref.hpp:156/:170, min_transpr.hpp:59/:90,
// min_trans.hpp:81, core.hpp:220, generators.hpp:36-145).
#include <cstdint>
#include <chrono>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "dfamin/dfamin.hpp"

using namespace dfamin;

namespace {

struct RefStats {
  uint64_t iterations;
  uint64_t closure_steps;
  double elapsed_ms;
  uint64_t peak_memory_estimate;
  int32_t status;
  double call_ms;  // wall time of the whole reference call, incl. its final canonicalize
};

Dfa make(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc, uint32_t initial) {
  Dfa d;
  d.num_states = n;
  d.alphabet_size = k;
  d.delta.assign(k, std::vector<State>(n));
  for (uint32_t a = 0; a < k; ++a) std::memcpy(d.delta[a].data(), delta + (size_t)a * n, 4ull * n);
  d.accepting.assign(acc, acc + n);
  d.initial = initial;
  return d;
}

void out(const MinResult& r, uint32_t* block, uint32_t* nb, RefStats* st, double call_ms) {
  if (r.stats.status == RunStatus::ok && block != nullptr)
    std::memcpy(block, r.partition.block.data(), 4ull * r.partition.block.size());
  if (nb) *nb = r.partition.num_blocks;
  if (st) {
    st->iterations = r.stats.iterations;
    st->closure_steps = r.stats.closure_steps;
    st->elapsed_ms = r.stats.elapsed_ms;
    st->peak_memory_estimate = r.stats.peak_memory_estimate;
    st->status = static_cast<int32_t>(r.stats.status);
    st->call_ms = call_ms;
  }
}

template <class F>
MinResult timed_call(F&& f, double& ms) {
  const auto t0 = std::chrono::steady_clock::now();
  MinResult r = f();
  ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

substrate::RacePolicy policy_of(int p) {
  switch (p) {
    case 1: return substrate::RacePolicy::deterministic_min;
    case 2: return substrate::RacePolicy::deterministic_max;
    default: return substrate::RacePolicy::arbitrary_winner;
  }
}

void copy_dfa(const Dfa& d, uint32_t* delta, uint8_t* acc) {
  for (uint32_t a = 0; a < d.alphabet_size; ++a)
    std::memcpy(delta + (size_t)a * d.num_states, d.delta[a].data(), 4ull * d.num_states);
  std::memcpy(acc, d.accepting.data(), d.num_states);
}

}  // namespace

extern "C" {

void ref_set_threads(unsigned n) { substrate::set_worker_count(n); }
unsigned ref_worker_count() { return substrate::worker_count(); }

int ref_sort_pr(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc,
                int64_t timeout_ms, uint32_t* block, uint32_t* nb, RefStats* st,
                uint32_t* trace_counts, uint32_t trace_cap) {
  const Dfa d = make(n, k, delta, acc, 0);
  SortTrace trace;
  SortOptions opt;
  opt.timeout_ms = timeout_ms;
  if (trace_counts) opt.trace = &trace;
  { double ms_ = 0; const MinResult r_ = timed_call([&] { return sort_pr(d, opt); }, ms_); out(r_, block, nb, st, ms_); }
  if (trace_counts)
    for (size_t i = 0; i < trace.block_counts.size() && i < trace_cap; ++i)
      trace_counts[i] = trace.block_counts[i];
  return 0;
}

int ref_naive_pr(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc, int policy,
                 int fused_cas, int64_t timeout_ms, uint32_t* block, uint32_t* nb, RefStats* st) {
  const Dfa d = make(n, k, delta, acc, 0);
  if (fused_cas) {
    { double ms_ = 0; const MinResult r_ = timed_call([&] { return naive_pr_cas(d, timeout_ms); }, ms_); out(r_, block, nb, st, ms_); }
  } else {
    PrOptions opt;
    opt.policy = policy_of(policy);
    opt.timeout_ms = timeout_ms;
    { double ms_ = 0; const MinResult r_ = timed_call([&] { return naive_pr(d, opt); }, ms_); out(r_, block, nb, st, ms_); }
  }
  return 0;
}

int ref_trans_pr(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc, int policy,
                 int64_t timeout_ms, uint64_t max_memory, uint32_t* block, uint32_t* nb,
                 RefStats* st) {
  const Dfa d = make(n, k, delta, acc, 0);
  PrOptions opt;
  opt.policy = policy_of(policy);
  opt.timeout_ms = timeout_ms;
  Limits lim;
  lim.max_memory_bytes = max_memory;
  lim.timeout_ms = timeout_ms;
  { double ms_ = 0; const MinResult r_ = timed_call([&] { return trans_pr(d, opt, lim); }, ms_); out(r_, block, nb, st, ms_); }
  return 0;
}

int ref_expand_alphabet(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc,
                        uint64_t max_memory, uint32_t* rows, uint32_t* levels, uint64_t* required) {
  const Dfa d = make(n, k, delta, acc, 0);
  Limits lim;
  lim.max_memory_bytes = max_memory;
  try {
    const ExpandedDfa e = expand_alphabet(d, lim);
    *levels = e.levels;
    *required = expand_required_bytes(n, k);
    for (size_t r = 0; r < e.delta.size(); ++r)
      std::memcpy(rows + r * n, e.delta[r].data(), 4ull * n);
    return 0;
  } catch (const CapacityError& err) {
    *required = err.required_bytes();
    return -2;
  }
}

int ref_trans_minimize(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc,
                       int64_t timeout_ms, uint64_t max_memory, uint32_t* block, uint32_t* nb,
                       RefStats* st, uint8_t* apart, uint64_t* popcounts, uint32_t pop_cap) {
  const Dfa d = make(n, k, delta, acc, 0);
  Limits lim;
  lim.max_memory_bytes = max_memory;
  lim.timeout_ms = timeout_ms;
  TransInspect ins;
  { double ms_ = 0; const MinResult r_ = timed_call([&] { return trans_minimize(d, lim, &ins); }, ms_); out(r_, block, nb, st, ms_); }
  if (apart && !ins.apart.empty()) std::memcpy(apart, ins.apart.data(), ins.apart.size());
  if (popcounts)
    for (size_t i = 0; i < ins.apart_popcounts.size() && i < pop_cap; ++i)
      popcounts[i] = ins.apart_popcounts[i];
  return 0;
}

uint32_t ref_moore(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc,
                   uint32_t* block, uint64_t* rounds) {
  const Dfa d = make(n, k, delta, acc, 0);
  RunStats st;
  const Partition p = moore_oracle(d, &st);
  std::memcpy(block, p.block.data(), 4ull * n);
  if (rounds) *rounds = st.iterations;
  return p.num_blocks;
}

uint32_t ref_canonicalize(const uint32_t* raw, uint32_t n, uint32_t* outp) {
  const Partition p = canonicalize(std::vector<uint32_t>(raw, raw + n));
  std::memcpy(outp, p.block.data(), 4ull * n);
  return p.num_blocks;
}

// ---- sortPR one pass at a time (bench.py --impl reference: a bounded sample of
// the workload per step).  The session holds the reference loop's state
// (block, order, num_blocks; min_sort.hpp:80-91) and each call executes ONE
// iteration of the loop body (min_sort.hpp:100-118) with the reference's own
// functions: make_signature, substrate::par_sort with signature_key_less,
// substrate::adjacent_diff with signature_key_neq, substrate::inclusive_scan and
// the par_for scatter.  The fixpoint pass also runs the final canonicalize
// (min_sort.hpp:123) and re-initialises the session, so a whole number of
// cycles of calls times exactly that many sort_pr runs (minus RunStats
// bookkeeping).  The Dfa is generated in place by the reference generator.
struct RefSortSession {
  Dfa d;
  std::vector<std::uint32_t> block, order;
  std::uint32_t num_blocks = 1;
  std::uint64_t pass = 0;
  void init() {  // min_sort.hpp:80-91
    const std::uint32_t n = d.num_states;
    bool has_acc = false, has_rej = false;
    for (State q = 0; q < n; ++q) (d.accepting[q] != 0 ? has_acc : has_rej) = true;
    block.assign(n, 0);
    num_blocks = 1;
    if (has_acc && has_rej) {
      num_blocks = 2;
      for (State q = 0; q < n; ++q) block[q] = d.accepting[q] != 0 ? 0 : 1;
    }
    order.resize(n);
    std::iota(order.begin(), order.end(), 0u);
    pass = 0;
  }
};

void* ref_sort_session_random(uint32_t n, uint32_t k, uint64_t seed, double p) {
  auto* s = new RefSortSession;
  s->d = random_dfa(n, k, seed, p);
  s->init();
  return s;
}

// one pass; returns 1 when it was the fixpoint pass (canonicalize ran, session reset)
int ref_sort_session_pass(void* h, double* elapsed_ms, uint32_t* fresh_out) {
  auto* s = static_cast<RefSortSession*>(h);
  const Dfa& d = s->d;
  const std::uint32_t n = d.num_states, k = d.alphabet_size;
  const auto t0 = std::chrono::steady_clock::now();
  if (s->pass == 0) s->init();
  const std::vector<std::uint32_t> sig = make_signature(d, s->block);
  auto& block = s->block;
  auto& order = s->order;
  substrate::par_sort(order, [&](std::uint32_t a, std::uint32_t b) {
    return signature_key_less(a, b, block, sig, k);
  });
  const std::vector<std::uint32_t> marks =
      substrate::adjacent_diff(order, [&](std::uint32_t a, std::uint32_t b) {
        return signature_key_neq(a, b, block, sig, k);
      });
  const std::vector<std::uint32_t> labels = substrate::inclusive_scan(marks);
  substrate::par_for(n, [&](std::size_t i) { block[order[i]] = labels[i]; });
  const std::uint32_t fresh = labels[n - 1] + 1;
  ++s->pass;
  int done = 0;
  if (fresh == s->num_blocks) {
    const Partition canon = canonicalize(block);
    (void)canon;
    s->pass = 0;  // the next call starts a new run (init inside the timed call)
    done = 1;
  } else {
    s->num_blocks = fresh;
  }
  *elapsed_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (fresh_out) *fresh_out = fresh;
  return done;
}

// the next pass call starts a new sort_pr run (pass 1)
void ref_sort_session_reset(void* h) { static_cast<RefSortSession*>(h)->pass = 0; }
uint32_t ref_sort_session_states(void* h) { return static_cast<RefSortSession*>(h)->d.num_states; }
void ref_sort_session_free(void* h) { delete static_cast<RefSortSession*>(h); }

// whole sort_pr on a session's DFA (the reference's own entry point, RunStats timing)
int ref_sort_session_full(void* h, uint32_t* nb, RefStats* st) {
  auto* s = static_cast<RefSortSession*>(h);
  { double ms_ = 0; const MinResult r_ = timed_call([&] { return sort_pr(s->d, SortOptions{}); }, ms_); out(r_, nullptr, nb, st, ms_); }
  return 0;
}

// ---- ingestion (ingest.hpp:130-284): the whole parse -> determinize -> complete
// pipeline of the reference on one text, errors captured (tests/test_ingest.py)
struct RefIngest {
  Lts lts;
  PartialDfa p;
  Dfa d;
  int status = 0;  // 0 ok, 1 ParseError, 2 SubsetBudgetExceeded
  uint64_t line = 0;
  std::string what;
};

void* ref_ingest(const char* text, uint64_t len, uint64_t max_subsets) {
  auto* r = new RefIngest;
  try {
    r->lts = parse_lts(std::string_view(text, len));
    r->p = determinize(r->lts, max_subsets);
    r->d = complete(r->p);
  } catch (const ParseError& e) {
    r->status = 1;
    r->line = e.line();
    r->what = e.what();
  } catch (const SubsetBudgetExceeded& e) {
    r->status = 2;
    r->line = e.budget();
    r->what = e.what();
  }
  return r;
}
int ref_ingest_status(void* h, uint64_t* line, char* msg, uint32_t cap) {
  auto* r = static_cast<RefIngest*>(h);
  if (line) *line = r->line;
  if (msg && cap) {
    std::strncpy(msg, r->what.c_str(), cap - 1);
    msg[cap - 1] = 0;
  }
  return r->status;
}
void ref_ingest_lts(void* h, uint32_t* n, uint32_t* init, uint32_t* nl, uint64_t* m) {
  auto* r = static_cast<RefIngest*>(h);
  *n = r->lts.num_states;
  *init = r->lts.initial;
  *nl = (uint32_t)r->lts.labels.size();
  *m = r->lts.transitions.size();
}
void ref_ingest_lts_arrays(void* h, uint32_t* src, uint32_t* lab, uint32_t* dst) {
  auto* r = static_cast<RefIngest*>(h);
  for (size_t j = 0; j < r->lts.transitions.size(); ++j) {
    src[j] = r->lts.transitions[j].src;
    lab[j] = r->lts.transitions[j].label;
    dst[j] = r->lts.transitions[j].dst;
  }
}
const char* ref_ingest_label(void* h, uint32_t i) {
  return static_cast<RefIngest*>(h)->lts.labels[i].c_str();
}
void ref_ingest_pdfa(void* h, uint32_t* n, uint32_t* k, uint32_t* delta) {
  auto* r = static_cast<RefIngest*>(h);
  *n = r->p.num_states;
  *k = r->p.alphabet_size;
  if (delta)
    for (uint32_t a = 0; a < r->p.alphabet_size; ++a)
      std::memcpy(delta + (size_t)a * r->p.num_states, r->p.delta[a].data(),
                  4ull * r->p.num_states);
}
void ref_ingest_dfa(void* h, uint32_t* n, uint32_t* delta, uint8_t* acc) {
  auto* r = static_cast<RefIngest*>(h);
  *n = r->d.num_states;
  if (delta) copy_dfa(r->d, delta, acc);
}
void ref_ingest_free(void* h) { delete static_cast<RefIngest*>(h); }

// generators: n/k are known to the caller (fib_len etc. computed by the oracle)
void ref_random_dfa(uint32_t n, uint32_t k, uint64_t seed, double p, uint32_t* delta,
                    uint8_t* acc) {
  copy_dfa(random_dfa(n, k, seed, p), delta, acc);
}
void ref_fib_dfa(uint32_t idx, uint32_t* delta, uint8_t* acc) { copy_dfa(fib_dfa(idx), delta, acc); }
void ref_bit_splitter(uint32_t bits, uint32_t* delta, uint8_t* acc) {
  copy_dfa(bit_splitter(bits), delta, acc);
}
void ref_chain_dfa(uint32_t len, uint32_t* delta, uint8_t* acc) {
  copy_dfa(chain_dfa(len), delta, acc);
}

// quotient (core.hpp:256): 0 ok, 1 invalid_argument (message copied to err)
int ref_quotient(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc,
                 uint32_t initial, const uint32_t* block, uint32_t num_blocks, uint32_t* delta_out,
                 uint8_t* acc_out, uint32_t* initial_out, char* err, uint32_t err_cap) {
  Dfa d = make(n, k, delta, acc, initial);
  Partition p;
  p.block.assign(block, block + n);
  p.num_blocks = num_blocks;
  try {
    Dfa q = quotient(d, p);
    copy_dfa(q, delta_out, acc_out);
    *initial_out = q.initial;
    return 0;
  } catch (const std::invalid_argument& e) {
    if (err && err_cap) {
      std::strncpy(err, e.what(), err_cap - 1);
      err[err_cap - 1] = 0;
    }
    return 1;
  }
}

// remove_unreachable (core.hpp:152): returns the kept state count
uint32_t ref_remove_unreachable(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc,
                                uint32_t initial, uint32_t* delta_out, uint8_t* acc_out,
                                uint32_t* initial_out) {
  Dfa q = remove_unreachable(make(n, k, delta, acc, initial));
  copy_dfa(q, delta_out, acc_out);
  *initial_out = q.initial;
  return q.num_states;
}

}  // extern "C"
