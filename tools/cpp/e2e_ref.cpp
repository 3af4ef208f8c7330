// End to end through the C++ drop-in on the REFERENCE's own types: a dfamin::Dfa
// (std::vector rows in pageable memory, core.hpp:24-33) built by the reference's
// generator (or the builder-defined VLTS generator of SURVEY §8(d) for the C2
// shape, restated below on the reference's SplitMix64), minimized by dfamin::b200::sort_pr (include/dfamin_b200.hpp with
// DFAMIN_B200_USE_REFERENCE_TYPES), wall clock around the call — upload from the
// pageable rows, every pass, the canonical partition back in the MinResult.
// Built by the repo Makefile only where /root/reference exists (this container);
// the binary travels to the GPU box (rpath $ORIGIN).  bench.py reports it as
// e2e.cpp_reference_types.
//   e2e_ref random <n> <k> <seed> <reps> | vlts <m> <n> <k> <reps>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dfamin/dfamin.hpp"
#define DFAMIN_B200_USE_REFERENCE_TYPES
#include "dfamin_b200.hpp"

// SURVEY §8(d) C2 generator ("inflated VLTS-shaped quotient"), draw order as stated
// there, on the reference's SplitMix64 (generators.hpp:16-33); same DFA as
// paper_2410_22764_b200/generators.py::vlts_dfa
dfamin::Dfa vlts(uint32_t m, uint32_t n, uint32_t k, uint64_t base_seed = 7,
                 uint64_t inflate_seed = 9, double p = 0.4, uint32_t window = 16) {
  std::vector<std::vector<uint32_t>> bd(k, std::vector<uint32_t>(m, m - 1));
  std::vector<uint8_t> ba(m, 1);
  ba[m - 1] = 0;
  dfamin::SplitMix64 rng(base_seed);
  for (uint32_t q = 0; q + 1 < m; ++q) {
    uint32_t deg = 1;
    while (deg < k && rng.unit() > p) ++deg;
    for (uint32_t i = 0; i < deg; ++i) {
      const double u1 = rng.unit(), u2 = rng.unit();
      const uint32_t a = (uint32_t)((double)k * u1 * u2);
      const uint32_t t = rng.unit() < 0.8 ? (uint32_t)((q + 1 + rng.below(window)) % (m - 1))
                                          : (uint32_t)rng.below(m - 1);
      bd[a][q] = t;
    }
  }
  const uint64_t copies = n / m;
  dfamin::Dfa d;
  d.num_states = n;
  d.alphabet_size = k;
  d.initial = 0;
  d.delta.assign(k, std::vector<dfamin::State>(n));
  d.accepting.resize(n);
  dfamin::SplitMix64 inf(inflate_seed);
  for (uint32_t q = 0; q < n; ++q) {
    for (uint32_t a = 0; a < k; ++a)
      d.delta[a][q] = bd[a][q % m] + m * (uint32_t)(inf.next() % copies);
    d.accepting[q] = ba[q % m];
  }
  return d;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string kind = argv[1];
  dfamin::Dfa d;
  int reps = 3;
  std::string what;
  if (kind == "random" && argc >= 6) {
    const uint32_t n = (uint32_t)std::strtoul(argv[2], nullptr, 10);
    const uint32_t k = (uint32_t)std::strtoul(argv[3], nullptr, 10);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    reps = std::atoi(argv[5]);
    d = dfamin::random_dfa(n, k, seed, 0.5);  // generators.hpp:130-145
    what = "random_dfa(" + std::to_string(n) + ", " + std::to_string(k) + ", " +
           std::to_string(seed) + ")";
  } else if (kind == "vlts" && argc >= 6) {
    const uint32_t m = (uint32_t)std::strtoul(argv[2], nullptr, 10);
    const uint32_t n = (uint32_t)std::strtoul(argv[3], nullptr, 10);
    const uint32_t k = (uint32_t)std::strtoul(argv[4], nullptr, 10);
    reps = std::atoi(argv[5]);
    if (m < 2 || n % m != 0) return 3;
    d = vlts(m, n, k);
    what = "vlts(" + std::to_string(m) + ", " + std::to_string(n) + ", " + std::to_string(k) + ")";
  } else {
    return 2;
  }
  // FNV-1a over the rows then the acceptance bytes: ties the input to the Python
  // generators (tests/test_e2e_ref_tool.py)
  uint64_t h = 0xcbf29ce484222325ull;
  auto mix = [&](const void* p, size_t len) {
    const auto* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < len; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  };
  for (const auto& row : d.delta) mix(row.data(), row.size() * 4);
  mix(d.accepting.data(), d.accepting.size());
  if (reps < 0) {  // digest only (no GPU)
    std::printf("{\"input\": \"%s\", \"digest\": \"%016llx\"}\n", what.c_str(),
                (unsigned long long)h);
    return 0;
  }
  namespace B = dfamin::b200;
  dfamin::MinResult r = B::sort_pr(d);  // warm the context
  double best = 1e30, sum = 0;
  for (int i = 0; i < reps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    r = B::sort_pr(d);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    best = std::min(best, ms);
    sum += ms;
  }
  // partition digest: sum of block[i] * (2654435761 * i + 1) mod 2^64 (numpy-checkable)
  uint64_t ph = 0;
  for (size_t i = 0; i < r.partition.block.size(); ++i)
    ph += (uint64_t)r.partition.block[i] * (2654435761ull * i + 1ull);
  std::printf("{\"input\": \"%s\", \"digest\": \"%016llx\", \"n\": %u, \"k\": %u, \"passes\": %llu, \"blocks\": %u, "
              "\"ms_min\": %.3f, \"ms_mean\": %.3f, \"reps\": %d, \"status\": %d, \"partition_digest\": \"%016llx\"}\n",
              what.c_str(), (unsigned long long)h, d.num_states, d.alphabet_size,
              (unsigned long long)r.stats.iterations, r.partition.num_blocks, best, sum / reps, reps,
              (int)r.stats.status, (unsigned long long)ph);
  return r.stats.status == dfamin::RunStatus::ok ? 0 : 1;
}
