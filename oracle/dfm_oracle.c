/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the DFA-minimization hot path.
 * See dfm_oracle.h for the contract.  Each function names the reference
 * file:line (under /root/reference/proj/include/dfamin/) whose behaviour it
 * restates.  Sequential, single-threaded, written for clarity not speed.
 */
#include "dfm_oracle.h"

#include <stdlib.h>
#include <string.h>

#define NO_LEADER 0xFFFFFFFFu

/* ------------------------------------------------------------------ */
/* SplitMix64 — generators.hpp:16-33                                    */
/* ------------------------------------------------------------------ */
uint64_t orc_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t sm_below(uint64_t* s, uint64_t bound) { return orc_splitmix_next(s) % bound; }
static double sm_unit(uint64_t* s) {
  return (double)(orc_splitmix_next(s) >> 11) * (1.0 / 9007199254740992.0); /* 0x1.0p-53 */
}

/* random_dfa — generators.hpp:130-145: rows letter by letter, then acceptance */
void orc_random_dfa(uint32_t n, uint32_t k, uint64_t seed, double p, uint32_t* delta,
                    uint8_t* acc) {
  uint64_t s = seed;
  for (uint32_t a = 0; a < k; ++a)
    for (uint32_t q = 0; q < n; ++q) delta[(size_t)a * n + q] = (uint32_t)sm_below(&s, n);
  for (uint32_t q = 0; q < n; ++q) acc[q] = sm_unit(&s) < p ? 1 : 0;
}

/* fib_word / fib_dfa — generators.hpp:36-68.  |w_idx| = Fib(idx+1). */
uint32_t orc_fib_len(uint32_t idx) {
  uint64_t a = 1, b = 1; /* |w_0|, |w_1| */
  if (idx < 2) return 1;
  for (uint32_t i = 2; i <= idx; ++i) {
    uint64_t c = a + b;
    a = b;
    b = c;
  }
  return (uint32_t)b;
}

int orc_fib_dfa(uint32_t idx, uint32_t* delta, uint8_t* acc) {
  if (idx < 2 || idx > 45) return -1;
  const uint32_t len = orc_fib_len(idx);
  /* w_{i} = w_{i-1} ++ w_{i-2}: the word grows in place inside acc, since
   * every word starts with its predecessor; prev holds w_{i-2}. */
  uint8_t* prev = (uint8_t*)malloc(len);
  uint32_t prev_len = 1, cur_len = 1;
  prev[0] = 1; /* w_0 = "1" */
  acc[0] = 0;  /* w_1 = "0" */
  for (uint32_t i = 2; i <= idx; ++i) {
    memcpy(acc + cur_len, prev, prev_len);
    memcpy(prev, acc, cur_len);
    const uint32_t grown = cur_len + prev_len;
    prev_len = cur_len;
    cur_len = grown;
  }
  free(prev);
  for (uint32_t q = 0; q < len; ++q) delta[q] = (q + 1) % len;
  return 0;
}

/* bit_splitter — generators.hpp:76-107 (doubling construction) */
int orc_bit_splitter(uint32_t bits, uint32_t* delta, uint8_t* acc) {
  if (bits < 1 || bits > 26) return -1;
  const uint32_t N = 1u << bits;
  const uint32_t K = bits - 1;
  /* build level by level inside the final buffers: row a has stride N */
  uint32_t cur_n = 2, cur_k = 0;
  for (uint32_t level = 1; level < bits; ++level) {
    const uint32_t half = cur_n, full = half * 2;
    for (uint32_t a = 0; a < cur_k; ++a) {
      uint32_t* row = delta + (size_t)a * N;
      for (uint32_t q = 0; q < half; ++q) row[half + q] = half + row[q];
    }
    uint32_t* fresh = delta + (size_t)cur_k * N;
    const uint32_t suffix_top = half >> 1;
    for (uint32_t q = 0; q < full; ++q)
      fresh[q] = (q & suffix_top) != 0 ? ((q ^ half) & half) : q;
    cur_n = full;
    cur_k += 1;
  }
  (void)K;
  for (uint32_t q = 0; q < N; ++q) acc[q] = q >= N / 2 ? 1 : 0;
  return 0;
}

/* chain_dfa — generators.hpp:111-125 */
int orc_chain_dfa(uint32_t len, uint32_t* delta, uint8_t* acc) {
  if (len < 2 || len > 0x7FFFFFFFu) return -1;
  for (uint32_t q = 0; q + 1 < len; ++q) {
    delta[q] = q + 1;
    acc[q] = 0;
  }
  delta[len - 1] = len - 1;
  acc[len - 1] = 1;
  return 0;
}

/* comb(L,t) — builder-defined, SURVEY.md 8(d) C3.  n = L(t+1)+1, k = 2. */
uint32_t orc_comb_states(uint32_t L, uint32_t t) { return L * (t + 1) + 1; }
int orc_comb_dfa(uint32_t L, uint32_t t, uint32_t* delta, uint8_t* acc) {
  if (L < 1 || t < 1) return -1;
  const uint32_t n = orc_comb_states(L, t), sink = n - 1;
  uint32_t* da = delta;
  uint32_t* db = delta + n;
  for (uint32_t i = 0; i < L; ++i) {
    da[i] = (i + 1 < L) ? i + 1 : i;
    db[i] = L + i * t;
    acc[i] = (i + 1 == L) ? 1 : 0;
    for (uint32_t j = 0; j < t; ++j) {
      const uint32_t s = L + i * t + j;
      da[s] = sink;
      db[s] = (j + 1 < t) ? s + 1 : sink;
      acc[s] = (j + 1 == t) ? 1 : 0;
    }
  }
  da[sink] = sink;
  db[sink] = sink;
  acc[sink] = 0;
  return 0;
}

/* VLTS-shaped inflated quotient — builder-defined, SURVEY.md 8(d) C2.
 * base: vlts_base(m,k,base_seed,p,window); inflate(base,n,inflate_seed). */
int orc_vlts_dfa(uint32_t m, uint32_t n, uint32_t k, uint64_t base_seed, uint64_t inflate_seed,
                 double p, uint32_t window, uint32_t* delta, uint8_t* acc) {
  if (m < 2 || k < 1 || n % m != 0) return -1;
  uint32_t* bd = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m * k);
  uint8_t* ba = (uint8_t*)malloc(m);
  for (size_t i = 0; i < (size_t)m * k; ++i) bd[i] = m - 1;
  for (uint32_t q = 0; q < m; ++q) ba[q] = 1;
  ba[m - 1] = 0;
  uint64_t s = base_seed;
  for (uint32_t q = 0; q + 1 < m; ++q) {
    uint32_t deg = 1;
    while (deg < k && sm_unit(&s) > p) ++deg;
    for (uint32_t e = 0; e < deg; ++e) {
      const double u1 = sm_unit(&s);
      const double u2 = sm_unit(&s);
      const uint32_t a = (uint32_t)((double)k * u1 * u2);
      uint32_t t;
      if (sm_unit(&s) < 0.8)
        t = (uint32_t)((q + 1 + sm_below(&s, window)) % (m - 1));
      else
        t = (uint32_t)sm_below(&s, m - 1);
      bd[(size_t)a * m + q] = t;
    }
  }
  uint64_t s2 = inflate_seed;
  const uint32_t copies = n / m;
  for (uint32_t q = 0; q < n; ++q) {
    for (uint32_t a = 0; a < k; ++a)
      delta[(size_t)a * n + q] = bd[(size_t)a * m + q % m] + m * (uint32_t)sm_below(&s2, copies);
    acc[q] = ba[q % m];
  }
  free(bd);
  free(ba);
  return 0;
}

static int cmp64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* ------------------------------------------------------------------ */
/* canonicalize — core.hpp:123-136 (first-occurrence relabel)          */
/* ------------------------------------------------------------------ */
uint32_t orc_canonicalize(const uint32_t* raw, uint32_t n, uint32_t* out) {
  /* raw labels may be arbitrary u32: map through a sorted (label, first) table */
  if (n == 0) return 0;
  uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint64_t* pairs = (uint64_t*)malloc(sizeof(uint64_t) * n);
  for (uint32_t q = 0; q < n; ++q) pairs[q] = ((uint64_t)raw[q] << 32) | q;
  qsort(pairs, n, sizeof(uint64_t), cmp64);
  /* first occurrence of each label = min index within its run */
  uint32_t* first = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t q = (uint32_t)pairs[i];
    if (i == 0 || (pairs[i] >> 32) != (pairs[i - 1] >> 32)) first[q] = q; /* run head = min q */
    else first[q] = first[(uint32_t)pairs[i - 1]];
  }
  /* rank of the first-occurrence index among all first occurrences */
  uint32_t count = 0;
  for (uint32_t q = 0; q < n; ++q) idx[q] = (first[q] == q) ? count++ : 0;
  for (uint32_t q = 0; q < n; ++q) out[q] = idx[first[q]];
  free(idx);
  free(pairs);
  free(first);
  return count;
}

/* Group states by a row-major key table (w words per state): out[q] = dense
 * group id in sorted-key order.  Returns the group count. */
static const uint32_t* g_keys;
static uint32_t g_w;
static int cmp_key(const void* a, const void* b) {
  const uint32_t qa = *(const uint32_t*)a, qb = *(const uint32_t*)b;
  const uint32_t* ka = g_keys + (size_t)qa * g_w;
  const uint32_t* kb = g_keys + (size_t)qb * g_w;
  for (uint32_t i = 0; i < g_w; ++i) {
    if (ka[i] != kb[i]) return ka[i] < kb[i] ? -1 : 1;
  }
  return qa < qb ? -1 : (qa > qb ? 1 : 0);
}
static uint32_t group_by_keys(const uint32_t* keys, uint32_t w, uint32_t n, uint32_t* out) {
  if (n == 0) return 0;
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint32_t q = 0; q < n; ++q) order[q] = q;
  g_keys = keys;
  g_w = w;
  qsort(order, n, sizeof(uint32_t), cmp_key);
  uint32_t label = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (i > 0 && memcmp(keys + (size_t)order[i] * w, keys + (size_t)order[i - 1] * w,
                        sizeof(uint32_t) * w) != 0)
      ++label;
    out[order[i]] = label;
  }
  free(order);
  return label + 1;
}

/* ------------------------------------------------------------------ */
/* moore_oracle — core.hpp:220-250                                      */
/* ------------------------------------------------------------------ */
uint32_t orc_moore(const orc_dfa* d, uint32_t* out, uint64_t* rounds) {
  const uint32_t n = d->n, k = d->k;
  uint32_t* block = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* keys = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n * (k + 1) + 1));
  for (uint32_t q = 0; q < n; ++q) block[q] = d->acc[q] ? 0 : 1;
  uint32_t num_blocks = orc_canonicalize(block, n, out);
  uint64_t r = 0;
  for (;;) {
    ++r;
    for (uint32_t q = 0; q < n; ++q) {
      uint32_t* key = keys + (size_t)q * (k + 1);
      key[0] = block[q];
      for (uint32_t a = 0; a < k; ++a) key[a + 1] = block[d->delta[(size_t)a * n + q]];
    }
    const uint32_t count = group_by_keys(keys, k + 1, n, block);
    if (count == num_blocks) break;
    num_blocks = count;
  }
  if (rounds) *rounds = r;
  const uint32_t c = orc_canonicalize(block, n, out);
  free(block);
  free(keys);
  return c;
}

/* ------------------------------------------------------------------ */
/* sort_pr — min_sort.hpp:72-126                                        */
/* ------------------------------------------------------------------ */
int orc_sort_pr(const orc_dfa* d, uint32_t* block_out, uint32_t* num_blocks_out, orc_stats* st,
                orc_pass_cb cb, void* user) {
  const uint32_t n = d->n, k = d->k;
  int has_acc = 0, has_rej = 0;
  for (uint32_t q = 0; q < n; ++q) {
    if (d->acc[q]) has_acc = 1;
    else has_rej = 1;
  }
  uint32_t* block = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  uint32_t num_blocks = 1;
  if (has_acc && has_rej) {
    num_blocks = 2;
    for (uint32_t q = 0; q < n; ++q) block[q] = d->acc[q] ? 0 : 1;
  }
  /* key = (block[q], block[delta[0][q]], ..., block[delta[k-1][q]]) (min_sort.hpp:49-59);
   * new label = rank of the key class in sorted order (min_sort.hpp:101-109) */
  uint32_t* keys = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n * (k + 1) + 1));
  uint64_t iterations = 0;
  for (;;) {
    for (uint32_t q = 0; q < n; ++q) {
      uint32_t* key = keys + (size_t)q * (k + 1);
      key[0] = block[q];
      for (uint32_t a = 0; a < k; ++a) key[a + 1] = block[d->delta[(size_t)a * n + q]];
    }
    const uint32_t fresh = group_by_keys(keys, k + 1, n, block);
    ++iterations;
    if (cb) cb(user, iterations, block, n, fresh);
    if (fresh == num_blocks) break;
    num_blocks = fresh;
  }
  *num_blocks_out = orc_canonicalize(block, n, block_out);
  if (st) {
    st->iterations = iterations;
    st->closure_steps = 0;
    st->peak_memory_estimate = (uint64_t)n * (16 + 4 * (uint64_t)k);
    st->status = 0;
  }
  free(block);
  free(keys);
  return 0;
}

/* ------------------------------------------------------------------ */
/* leader_election_pr — min_partref.hpp:42-151 (sequential schedule)   */
/* rows: `letters` rows of n entries each, flat                         */
/* ------------------------------------------------------------------ */
static void elect(uint32_t* cell, uint32_t value, int policy) {
  /* substrate.hpp:99-120 */
  switch (policy) {
    case ORC_POLICY_ARBITRARY: *cell = value; return; /* sequential: last writer wins */
    case ORC_POLICY_MIN:
      if (value < *cell) *cell = value;
      return;
    case ORC_POLICY_MAX:
      if (*cell == NO_LEADER || value > *cell) *cell = value;
      return;
  }
}

static int leader_election(uint32_t n, const uint32_t* rows, size_t letters, const uint8_t* acc,
                           int policy, int fused_cas, uint32_t* block_out,
                           uint32_t* num_blocks_out, orc_stats* st, orc_pass_cb cb, void* user) {
  uint32_t leader_acc = NO_LEADER, leader_rej = NO_LEADER;
  for (uint32_t q = 0; q < n; ++q) {
    if (acc[q]) {
      if (leader_acc == NO_LEADER) leader_acc = q;
    } else if (leader_rej == NO_LEADER) {
      leader_rej = q;
    }
  }
  if (leader_acc == NO_LEADER) leader_acc = leader_rej;
  if (leader_rej == NO_LEADER) leader_rej = leader_acc;
  uint32_t* block = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* frozen = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* cells = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (uint32_t q = 0; q < n; ++q) {
    block[q] = acc[q] ? leader_acc : leader_rej;
    cells[q] = NO_LEADER;
  }
  uint64_t iterations = 0;
  int stable = 0;
  while (!stable) {
    stable = 1;
    memcpy(frozen, block, sizeof(uint32_t) * n);
    if (!fused_cas) {
      for (uint32_t q = 0; q < n; ++q) { /* phase A, min_partref.hpp:90-99 */
        const uint32_t leader = frozen[q];
        for (size_t a = 0; a < letters; ++a) {
          const uint32_t* row = rows + a * n;
          if (frozen[row[q]] != frozen[row[leader]]) {
            elect(&cells[leader], q, policy);
            break;
          }
        }
      }
      for (uint32_t q = 0; q < n; ++q) { /* phase B, :102-112 */
        const uint32_t leader = frozen[q];
        for (size_t a = 0; a < letters; ++a) {
          const uint32_t* row = rows + a * n;
          if (frozen[row[q]] != frozen[row[leader]]) {
            block[q] = cells[leader];
            stable = 0;
            break;
          }
        }
      }
    } else {
      for (uint32_t q = 0; q < n; ++q) { /* fused CAS, :116-132; first writer wins */
        const uint32_t leader = frozen[q];
        for (size_t a = 0; a < letters; ++a) {
          const uint32_t* row = rows + a * n;
          if (frozen[row[q]] != frozen[row[leader]]) {
            if (cells[leader] == NO_LEADER) cells[leader] = q;
            block[q] = cells[leader];
            stable = 0;
            break;
          }
        }
      }
    }
    ++iterations;
    for (uint32_t q = 0; q < n; ++q) cells[q] = NO_LEADER; /* :136-138 */
    if (cb) {
      uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
      const uint32_t c = orc_canonicalize(block, n, tmp);
      cb(user, iterations, block, n, c);
      free(tmp);
    }
  }
  *num_blocks_out = orc_canonicalize(block, n, block_out);
  if (st) {
    st->iterations = iterations;
    st->closure_steps = 0;
    st->peak_memory_estimate = (uint64_t)n * 12;
    st->status = 0;
  }
  free(block);
  free(frozen);
  free(cells);
  return 0;
}

int orc_naive_pr(const orc_dfa* d, int policy, int fused_cas, uint32_t* block_out,
                 uint32_t* num_blocks, orc_stats* st, orc_pass_cb cb, void* user) {
  /* naive_pr min_partref.hpp:156-166 / naive_pr_cas :170-176 */
  return leader_election(d->n, d->delta, d->k, d->acc, policy, fused_cas, block_out, num_blocks,
                         st, cb, user);
}

/* ------------------------------------------------------------------ */
/* transPR — min_transpr.hpp:21-122                                     */
/* ------------------------------------------------------------------ */
uint32_t orc_power_levels(uint32_t n) {
  uint32_t w = 0;
  while (n) {
    ++w;
    n >>= 1;
  }
  return w; /* std::bit_width */
}
uint64_t orc_expand_required_bytes(uint32_t n, uint32_t k) {
  return (uint64_t)orc_power_levels(n) * k * n * sizeof(uint32_t);
}

int orc_expand_alphabet(const orc_dfa* d, uint64_t max_memory_bytes, uint32_t* rows_out,
                        uint32_t* levels, uint64_t* required) {
  const uint32_t n = d->n, k = d->k;
  const uint64_t req = orc_expand_required_bytes(n, k);
  if (required) *required = req;
  if (req > max_memory_bytes) return -2; /* CapacityError, min_transpr.hpp:63-67 */
  const uint32_t L = orc_power_levels(n);
  if (levels) *levels = L;
  memcpy(rows_out, d->delta, sizeof(uint32_t) * (size_t)n * k);
  for (uint32_t lvl = 1; lvl < L; ++lvl) {
    for (uint32_t a = 0; a < k; ++a) {
      const uint32_t* prev = rows_out + ((size_t)(lvl - 1) * k + a) * n;
      uint32_t* cur = rows_out + ((size_t)lvl * k + a) * n;
      for (uint32_t q = 0; q < n; ++q) cur[q] = prev[prev[q]];
    }
  }
  return 0;
}

int orc_trans_pr(const orc_dfa* d, int policy, uint64_t max_memory_bytes, uint32_t* block_out,
                 uint32_t* num_blocks, orc_stats* st) {
  uint64_t req = 0;
  uint32_t L = 0;
  const uint64_t total = orc_expand_required_bytes(d->n, d->k);
  if (total > max_memory_bytes) {
    if (st) {
      st->iterations = 0;
      st->closure_steps = 0;
      st->peak_memory_estimate = total;
      st->status = 2;
    }
    *num_blocks = 0;
    return 0;
  }
  uint32_t* rows = (uint32_t*)malloc(total ? total : 4);
  orc_expand_alphabet(d, max_memory_bytes, rows, &L, &req);
  leader_election(d->n, rows, (size_t)L * d->k, d->acc, policy, 0, block_out, num_blocks, st,
                  NULL, NULL);
  if (st) {
    st->closure_steps = L - 1;
    st->peak_memory_estimate += total;
  }
  free(rows);
  return 0;
}

/* ------------------------------------------------------------------ */
/* trans_minimize (Cho–Huynh pair-graph closure) — min_trans.hpp:81-212 */
/* ------------------------------------------------------------------ */
static int popc64(uint64_t x) { return __builtin_popcountll(x); }

int orc_trans_minimize(const orc_dfa* d, uint64_t max_memory_bytes, uint32_t* block_out,
                       uint32_t* num_blocks, orc_stats* st, uint8_t* apart_out,
                       uint64_t* popcounts, uint32_t popcounts_cap) {
  const uint64_t n = d->n;
  /* trans_required_bytes, min_trans.hpp:24-27: ceil(n^4/8) as u128 */
  const unsigned __int128 bits = (unsigned __int128)n * n * n * n;
  const unsigned __int128 required = (bits + 7) / 8;
  if (required > max_memory_bytes) {
    if (st) {
      st->iterations = 0;
      st->closure_steps = 0;
      st->peak_memory_estimate =
          required > (unsigned __int128)UINT64_MAX ? UINT64_MAX : (uint64_t)required;
      st->status = 2;
    }
    *num_blocks = 0;
    return 0;
  }
  const size_t pairs = (size_t)(n * n);
  const size_t W = (pairs + 63) / 64;
  uint64_t* reach = (uint64_t*)calloc(pairs * W + 1, 8);
  uint64_t* next = (uint64_t*)calloc(pairs * W + 1, 8);
  uint64_t* apart = (uint64_t*)calloc(W + 1, 8);
  uint64_t* apart_next = (uint64_t*)calloc(W + 1, 8);
  for (size_t s = 0; s < pairs; ++s) { /* init :111-119 */
    const size_t q = s / n, r = s % n;
    for (uint32_t a = 0; a < d->k; ++a) {
      const size_t t = (size_t)d->delta[(size_t)a * n + q] * n + d->delta[(size_t)a * n + r];
      reach[s * W + (t >> 6)] |= 1ull << (t & 63);
    }
    if (d->acc[q] != d->acc[r]) apart[s >> 6] |= 1ull << (s & 63); /* :120-126 */
  }
  uint64_t iterations = 0;
  int changed = 1;
  while (changed) {
    memcpy(next, reach, pairs * W * 8); /* squaring :142-158 */
    for (size_t s = 0; s < pairs; ++s) {
      const uint64_t* src = reach + s * W;
      uint64_t* dst = next + s * W;
      for (size_t w = 0; w < W; ++w) {
        uint64_t b = src[w];
        while (b) {
          const size_t t = (w << 6) + (size_t)__builtin_ctzll(b);
          b &= b - 1;
          const uint64_t* via = reach + t * W;
          for (size_t i = 0; i < W; ++i) dst[i] |= via[i];
        }
      }
    }
    for (size_t w = 0; w < W; ++w) { /* propagation :164-179 */
      uint64_t b = apart[w];
      for (size_t j = 0; j < 64 && (w << 6) + j < pairs; ++j) {
        if ((b >> j) & 1) continue;
        const size_t s = (w << 6) + j;
        const uint64_t* row = next + s * W;
        for (size_t i = 0; i < W; ++i) {
          if (row[i] & apart[i]) {
            b |= 1ull << j;
            break;
          }
        }
      }
      apart_next[w] = b;
    }
    ++iterations;
    changed = memcmp(apart_next, apart, W * 8) != 0;
    uint64_t* t1 = apart;
    apart = apart_next;
    apart_next = t1;
    uint64_t* t2 = reach;
    reach = next;
    next = t2;
    if (popcounts && iterations <= popcounts_cap) {
      uint64_t c = 0;
      for (size_t w = 0; w < W; ++w) c += (uint64_t)popc64(apart[w]);
      popcounts[iterations - 1] = c;
    }
  }
  uint32_t* label = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (size_t q = 0; q < n; ++q) { /* labels :189-197 */
    for (size_t q0 = 0; q0 <= q; ++q0) {
      const size_t i = q0 * n + q;
      if (!((apart[i >> 6] >> (i & 63)) & 1)) {
        label[q] = (uint32_t)q0;
        break;
      }
    }
  }
  if (apart_out)
    for (size_t i = 0; i < pairs; ++i) apart_out[i] = (apart[i >> 6] >> (i & 63)) & 1;
  *num_blocks = orc_canonicalize(label, (uint32_t)n, block_out);
  if (st) {
    st->iterations = iterations;
    st->closure_steps = 0;
    st->peak_memory_estimate = 2 * (uint64_t)pairs * W * 8 + 2 * (uint64_t)W * 8;
    st->status = 0;
  }
  free(reach);
  free(next);
  free(apart);
  free(apart_next);
  free(label);
  return 0;
}

/* ------------------------------------------------------------------ quotient
 * core.hpp:256-290: check the partition is canonical (:259-262), then the first
 * state of each block defines its row (:270-277); every later state must agree
 * on acceptance (:279-281) and on each letter's target block (:282-286). */
int orc_quotient(const orc_dfa* d, const uint32_t* block, uint32_t num_blocks, uint32_t* delta_out,
                 uint8_t* acc_out, uint32_t* initial_out, uint32_t* bad_block,
                 uint32_t* bad_letter) {
  const uint32_t n = d->n, k = d->k;
  uint32_t* canon = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  const uint32_t nb = orc_canonicalize(block, n, canon);
  int bad = nb != num_blocks;
  for (uint32_t q = 0; q < n && !bad; ++q) bad = canon[q] != block[q];
  free(canon);
  if (bad) return 1;
  uint8_t* defined = (uint8_t*)calloc(num_blocks ? num_blocks : 1, 1);
  for (uint32_t b = 0; b < num_blocks; ++b) acc_out[b] = 0;
  for (size_t i = 0; i < (size_t)k * num_blocks; ++i) delta_out[i] = 0;
  int rc = 0;
  for (uint32_t q = 0; q < n && rc == 0; ++q) {
    const uint32_t b = block[q];
    if (!defined[b]) {
      defined[b] = 1;
      acc_out[b] = d->acc[q];
      for (uint32_t a = 0; a < k; ++a)
        delta_out[(size_t)a * num_blocks + b] = block[d->delta[(size_t)a * n + q]];
      continue;
    }
    if (acc_out[b] != d->acc[q]) {
      rc = 2;
      *bad_block = b;
      break;
    }
    for (uint32_t a = 0; a < k; ++a)
      if (delta_out[(size_t)a * num_blocks + b] != block[d->delta[(size_t)a * n + q]]) {
        rc = 3;
        *bad_block = b;
        *bad_letter = a;
        break;
      }
  }
  free(defined);
  if (rc == 0) *initial_out = n ? block[d->initial] : 0;
  return rc;
}

/* ------------------------------------------------------------------ remove_unreachable
 * core.hpp:152-187: breadth-first search from the initial state (:153-166), dense
 * renumbering in ascending original order (:167-171), induced rows (:172-186). */
uint32_t orc_remove_unreachable(const orc_dfa* d, uint32_t* delta_out, uint8_t* acc_out,
                                uint32_t* initial_out) {
  const uint32_t n = d->n, k = d->k;
  if (n == 0) return 0;
  uint8_t* seen = (uint8_t*)calloc(n, 1);
  uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * n);
  size_t tail = 0;
  queue[tail++] = d->initial;
  seen[d->initial] = 1;
  for (size_t head = 0; head < tail; ++head) {
    const uint32_t q = queue[head];
    for (uint32_t a = 0; a < k; ++a) {
      const uint32_t t = d->delta[(size_t)a * n + q];
      if (!seen[t]) {
        seen[t] = 1;
        queue[tail++] = t;
      }
    }
  }
  uint32_t* renumber = queue; /* reuse */
  uint32_t kept = 0;
  for (uint32_t q = 0; q < n; ++q) renumber[q] = seen[q] ? kept++ : 0;
  for (uint32_t q = 0; q < n; ++q) {
    if (!seen[q]) continue;
    const uint32_t nq = renumber[q];
    acc_out[nq] = d->acc[q];
    for (uint32_t a = 0; a < k; ++a)
      delta_out[(size_t)a * kept + nq] = renumber[d->delta[(size_t)a * n + q]];
  }
  *initial_out = renumber[d->initial];
  free(seen);
  free(queue);
  return kept;
}
