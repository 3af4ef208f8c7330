// sortPR, hash-grouping engine (the default).
//
// Same partition sequence, pass count and fixpoint as the reference
// (min_sort.hpp:72-126) and as the radix engine (sort_pr.cu): only the way
// states with equal keys are grouped differs.  Per pass, over the ACTIVE
// states (block size >= 2), kept in ascending-q order so every delta row and
// own-id read is coalesced:
//
//   K1 insert  : key = (block[q], id[delta_a(q)] ...) — packed exactly when it
//                fits 63 bits, else a 64-bit hash with the full signature row
//                kept for verification; one atomic slot update per state in an
//                open-addressing table (direct-indexed when the key space is
//                small; CTA shared-memory aggregation when it is tiny).  The
//                slot collects the group size, its minimum member and whether
//                it holds the old block's leader (minimum state).
//   K2 resolve : look-back scan over the active states: the minimum member of
//                every group decides the group's id — the old block id if the
//                group holds the old leader, else a fresh id B + rank; equal-
//                hash members are verified against the minimum member's row.
//   K3 apply   : writes the new ids in place (skipped if a hash collision was
//                found: the pass is then redone under a new seed — exact).
//
// Random accesses per active state: the k successor-id gathers (the floor of
// the algorithm) + one slot RMW + one slot read (+ one row for verified
// members).  Ids are gathered from packed 1/4/8/16-bit mirrors while
// B <= 2/16/256/65536, so early passes gather from L2.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include <cooperative_groups.h>

#include "prims.cuh"

namespace cg = cooperative_groups;

namespace dfm {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr int kSmallTable = 4096;  // direct tables up to this size aggregate in smem

// first seed of every run; DFM_SORTPR_WEAK_HASH=<bits> (tests) truncates the hashed
// keys of passes under this seed so that distinct signatures collide and the
// void-and-retry path runs
constexpr uint64_t kSeed0 = 0x5EED0001ull;
__device__ unsigned long long g_weak_mask = ~0ull;
__device__ __forceinline__ unsigned long long weak(unsigned long long h, uint64_t seed) {
  return seed == kSeed0 ? (h & g_weak_mask) : h;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Slot {
  unsigned long long key;  // 0 = empty; after resolve: the group's new id
  uint32_t rep;            // ~(minimum active position) — atomicMax
  uint32_t info;           // member count | (holds old leader) << 31
};
static_assert(sizeof(Slot) == 16, "slot is 16 bytes");

struct InsertParams {
  const uint32_t* __restrict__ delta;
  uint64_t n;
  uint32_t k;
  const uint32_t* __restrict__ block;
  const void* __restrict__ ids;  // gather source: mirror (u8/u16) or block
  const uint32_t* __restrict__ act;
  const uint8_t* __restrict__ lead;
  uint64_t m;
  int w;
  uint64_t seed;
  uint64_t cap;  // hash-table capacity (unused for direct tables)
  Slot* slots;
  uint32_t* __restrict__ slot_of;
  uint32_t* __restrict__ sig;
  uint32_t row;  // signature row stride (words)
  unsigned long long* keys;  // precomputed exact keys (swept passes), else unused
  // rank-compacted direct table: slot = rank of the key among the keys present
  // (bitmap + per-word exclusive popcount); no same-slot warp aggregation
  const uint32_t* present;  // {bitmap word, exclusive popcount} pairs
  const uint32_t* cand;  // filtered passes: the states left for the table (m = their count)
  uint64_t i0;           // first index (pipelined first pass: one chunk of states)
  // relabel-in-place passes: the slot (key or key rank) + id_off becomes the new id
  uint32_t* ids_out;
  uint32_t id_off;
};

// L2 eviction policies: the delta stream is read once per pass (evict first) so
// that the gathered id array — the u8/u16 mirror in early passes — stays resident
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 16-byte compare-and-swap (sm_90+): old = *p; if old == cmp then *p = val
__device__ __forceinline__ void cas128(void* p, unsigned long long cmp_lo, unsigned long long cmp_hi,
                                       unsigned long long val_lo, unsigned long long val_hi,
                                       unsigned long long& old_lo, unsigned long long& old_hi) {
  asm volatile(
      "{\n\t.reg .b128 d, c, v;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(old_lo), "=l"(old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(val_lo), "l"(val_hi), "l"(p)
      : "memory");
}

// (non-volatile asm: read-only data, so the compiler may batch these loads)
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* a, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}

// id gather from the mirror of width kIdBits: 1 (bitmap, B <= 2), 4 (nibbles,
// B <= 16), 8, 16, or 32 (the block array itself).  Narrow mirrors keep the
// gathered array L2-resident (12.5 / 50 MB at n = 1e8).
template <int kIdBits>
__device__ __forceinline__ uint32_t load_id(const void* ids, uint32_t t, uint64_t pol) {
  uint32_t v;
  if (kIdBits == 1) {
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;"
        : "=r"(v)
        : "l"(static_cast<const uint32_t*>(ids) + (t >> 5)), "l"(pol));
    return (v >> (t & 31)) & 1u;
  }
  if (kIdBits == 4) {
    asm("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;"
        : "=r"(v)
        : "l"(static_cast<const uint8_t*>(ids) + (t >> 1)), "l"(pol));
    return (v >> ((t & 1) * 4)) & 0xFu;
  }
  if (kIdBits == 8)
    asm("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;"
        : "=r"(v)
        : "l"(static_cast<const uint8_t*>(ids) + t), "l"(pol));
  else if (kIdBits == 16)
    asm("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;"
        : "=r"(v)
        : "l"(static_cast<const uint16_t*>(ids) + t), "l"(pol));
  else
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;"
        : "=r"(v)
        : "l"(static_cast<const uint32_t*>(ids) + t), "l"(pol));
  return v;
}

// kK > 0: compile-time alphabet size, so all delta loads, then all id gathers,
// are in flight together; kK == 0: runtime k
template <int kIdBits, bool kHashed, int kK>
__device__ __forceinline__ unsigned long long make_key(const InsertParams& p, uint64_t i, uint32_t q,
                                                       uint32_t b, uint64_t pol_stream,
                                                       uint64_t pol_ids) {
  const uint32_t k = kK > 0 ? (uint32_t)kK : p.k;
  if (kK > 0) {
    uint32_t t[kK > 0 ? kK : 1], s[kK > 0 ? kK : 1];
#pragma unroll
    for (int a = 0; a < kK; ++a) t[a] = ld_stream(p.delta + (uint64_t)a * p.n + q, pol_stream);
#pragma unroll
    for (int a = 0; a < kK; ++a) s[a] = load_id<kIdBits>(p.ids, t[a], pol_ids);
    if (!kHashed) {
      unsigned long long key = b;
#pragma unroll
      for (int a = 0; a < kK; ++a) key = (key << p.w) | s[a];
      return key;
    }
    uint32_t* row = p.sig + i * (uint64_t)p.row;
    row[0] = b;
    unsigned long long h = mix64(p.seed * kGolden + b);
#pragma unroll
    for (int a = 0; a < kK; ++a) {
      row[a + 1] = s[a];
      h = mix64(h + kGolden + s[a]);
    }
    return weak(h, p.seed);
  }
  if (!kHashed) {
    unsigned long long key = b;
    for (uint32_t a = 0; a < k; ++a)
      key = (key << p.w) |
            load_id<kIdBits>(p.ids, ld_stream(p.delta + (uint64_t)a * p.n + q, pol_stream),
                              pol_ids);
    return key;
  }
  uint32_t* row = p.sig + i * (uint64_t)p.row;
  row[0] = b;
  unsigned long long h = mix64(p.seed * kGolden + b);
  for (uint32_t a = 0; a < k; ++a) {
    const uint32_t s =
        load_id<kIdBits>(p.ids, ld_stream(p.delta + (uint64_t)a * p.n + q, pol_stream), pol_ids);
    row[a + 1] = s;
    h = mix64(h + kGolden + s);
  }
  return weak(h, p.seed);
}

// Hashed keys for a runtime (large) alphabet, one call per warp for 32 consecutive
// active positions i0 + lane: each lane hashes its own signature, and the rows are
// written 8 words at a time through a per-warp shared buffer so that every store
// fills whole 32-byte sectors (row stride a multiple of 8 words) instead of 32
// lanes touching 32 rows per store.
template <int kIdBits>
__device__ __forceinline__ unsigned long long make_key_rows_warp(
    const InsertParams& p, uint64_t i0, bool valid, uint32_t q, uint32_t b, uint64_t pol_stream,
    uint64_t pol_ids, uint32_t* s_buf /* [32][9] */) {
  // the row's k + 1 fields (own id, successor ids) are packed kPer to a word: every id
  // of this pass is below 2^kIdBits (the mirror width), so a row is (k+1) / kPer words —
  // 4 instead of 101 at k = 100 with 1-bit ids (the host sizes the rows to match:
  // packed_row_words); the hash runs over the fields, whatever the packing
  constexpr uint32_t kPer = 32 / kIdBits;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t fields = p.k + 1, words = (fields + kPer - 1) / kPer;
  const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
  unsigned long long h = mix64(p.seed * kGolden + b);
  uint32_t* my = s_buf + lane * 9;
  for (uint32_t w0 = 0; w0 < words; w0 += 8) {
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c) my[c] = 0u;
    const uint32_t f_end = min(fields, (w0 + 8) * kPer);
    for (uint32_t f0 = w0 * kPer; f0 < f_end; f0 += 8) {
      uint32_t t[8], v[8];
#pragma unroll
      for (uint32_t c = 0; c < 8; ++c) {
        const uint32_t f = f0 + c;
        t[c] = (valid && f >= 1 && f < f_end)
                   ? ld_stream(p.delta + (uint64_t)(f - 1) * p.n + q, pol_stream)
                   : 0u;
      }
#pragma unroll
      for (uint32_t c = 0; c < 8; ++c) {
        const uint32_t f = f0 + c;
        v[c] = f == 0 ? b : (valid && f < f_end) ? load_id<kIdBits>(p.ids, t[c], pol_ids) : 0u;
        if (f >= 1 && f < f_end) h = mix64(h + kGolden + v[c]);
        if (f < f_end) my[f / kPer - w0] |= v[c] << ((f % kPer) * kIdBits);
      }
    }
    __syncwarp();
    // lane L writes word L % 8 of row (4 r + L / 8): one full sector per 8 lanes
#pragma unroll
    for (uint32_t r = 0; r < 8; ++r) {
      const uint32_t row_lane = 4 * r + (lane >> 3), c = lane & 7;
      if (((vmask >> row_lane) & 1u) && w0 + c < words)
        p.sig[(i0 + row_lane) * (uint64_t)p.row + w0 + c] = s_buf[row_lane * 9 + c];
    }
    __syncwarp();
  }
  return weak(h, p.seed);
}

// K1, hash or large direct table; warp-level aggregation of equal slots
constexpr uint32_t kUnique = 0xFFFFFFFFu;  // slot_of mark: key seen once (filtered)

// runtime-k hashed inserts are gather-latency bound: at 79 registers only 3 CTAs (24
// warps) fit an SM; capped for DFM_INS_MINB CTAs per SM.  Measured on C2 sortPR
// vlts(1000, 1e7, 100) (profiles/r04/r04r-s): 3 CTAs 23.6 ms, 4: 22.4, 5: 22.0,
// 6: 20.9, 7: 23.3, 8: 23.4; vlts(1000, 1e7, 10): 4: 5.47, 6: 5.29, 8: 5.82
#ifndef DFM_INS_MINB
#define DFM_INS_MINB 6
#endif
template <int kIdBits, bool kHashed, bool kDirect, int kK, bool kFromKeys = false,
          bool kFilter = false>
__global__ void __launch_bounds__(256, (kHashed && kK == 0 && !kFromKeys && !kFilter) ? DFM_INS_MINB : 1)
    insert_kernel(InsertParams p) {
  // large runtime alphabets with hashed keys: warp-cooperative coalesced row writes
  constexpr bool kRowsWarp = kHashed && kK == 0 && !kFromKeys && !kFilter;
  __shared__ uint32_t s_rows[kRowsWarp ? 8 * 32 * 9 : 1];
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_ids = policy_evict_last();
  // each warp takes 64 consecutive active states per step (two per lane) so two
  // independent gather chains are in flight per thread
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 2;
  const uint64_t warp_first =
      ((uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) * 2;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t base = warp_first; base < p.m; base += stride) {
    uint64_t s[2] = {0, 0};
    uint32_t lead[2] = {0, 0};
    unsigned long long key[2] = {0, 0};
    bool valid[2];
    bool merge[2] = {!kHashed, !kHashed};  // slot needs the aggregated rep/info update
    uint64_t idx[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t j = base + u * 32 + lane;
      // filtered passes iterate the candidate list (keys the filter saw repeated)
      valid[u] = j < p.m;
      idx[u] = kFilter ? (valid[u] ? p.cand[j] : 0) : j;
      const uint64_t i = idx[u];
      if (kRowsWarp) {  // whole warp: coalesced signature rows (see make_key_rows_warp)
        const uint32_t q = valid[u] ? (p.act ? p.act[i] : (uint32_t)i) : 0u;
        const uint32_t b = valid[u] ? p.block[q] : 0u;
        if (valid[u]) lead[u] = p.lead[q];
        key[u] = make_key_rows_warp<kIdBits>(p, base + u * 32, valid[u], q, b, pol_stream,
                                             pol_ids, s_rows + (threadIdx.x >> 5) * (32 * 9));
      } else if (valid[u]) {
        const uint32_t q = p.act ? p.act[i] : (uint32_t)i;
        lead[u] = p.lead[q];
        key[u] = kFromKeys ? p.keys[i]
                           : make_key<kIdBits, kHashed, kK>(p, i, q, p.block[q], pol_stream,
                                                             pol_ids);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t i = idx[u];
      if (valid[u]) {
        if (kDirect) {
          if (p.present) {
            const uint32_t w = (uint32_t)(key[u] >> 5);
            // {bitmap word, exclusive popcount} pairs: one 8-byte gather per key
            const uint2 pw = *reinterpret_cast<const uint2*>(p.present + 2ull * w);
            s[u] = pw.y + __popc(pw.x & ((1u << (key[u] & 31)) - 1u));
          } else {
            s[u] = key[u];
          }
        } else {
          // stored key: never 0 (0 marks an empty slot); start slot = mulhi(hash, capacity)
          const unsigned long long stored = kHashed ? (key[u] | 1ull) : key[u] + 1ull;
          const unsigned long long h = kHashed ? key[u] : mix64(key[u] ^ p.seed);
          uint64_t t = __umul64hi(h, p.cap);
          if (kHashed) {
            // hashed keys are nearly all distinct: claim/update the whole 16-byte slot
            // {key, rep, info} with one blind 128-bit CAS (one random RMW per state)
            const unsigned long long mine =
                (unsigned long long)(~(uint32_t)i) |
                ((unsigned long long)(1u | (lead[u] ? 0x80000000u : 0u)) << 32);
            // a state finding its key already present joins the warp-aggregated
            // atomic update below (a CAS merge loop serialises large groups)
            while (true) {
              unsigned long long old_lo, old_hi;
              cas128(&p.slots[t], 0ull, 0ull, stored, mine, old_lo, old_hi);
              if (old_lo == 0ull && old_hi == 0ull) break;
              if (old_lo == stored) {
                merge[u] = true;
                break;
              }
              if (++t == p.cap) t = 0;  // another key owns this slot: probe on
            }
          } else {
            while (true) {
              const unsigned long long cur = atomicCAS(&p.slots[t].key, 0ull, stored);
              if (cur == 0ull || cur == stored) break;
              if (++t == p.cap) t = 0;
            }
          }
          s[u] = t;
        }
        // (relabel-in-place rank passes read no slot index back)
        if (!(kDirect && p.present && p.ids_out)) p.slot_of[i] = (uint32_t)s[u];
      }
      if (kDirect && p.present) {  // many distinct keys: consecutive states rarely share one
        if (valid[u]) {
          atomicMax(&p.slots[s[u]].rep, ~(uint32_t)i);
          if (p.ids_out)  // relabel in place: the rank is the id; no group size or leader bit
            p.ids_out[p.act ? p.act[i] : (uint32_t)i] = (uint32_t)s[u] + p.id_off;
          else
            atomicAdd(&p.slots[s[u]].info, 1u | (lead[u] ? 0x80000000u : 0u));
        }
        continue;
      }
      const uint32_t vmask = __ballot_sync(0xffffffffu, valid[u] && merge[u]);
      if (valid[u] && merge[u]) {
        // lanes with the same slot: the lowest lane updates for all, with the group's
        // minimum state (candidate lists are not in ascending order)
        const uint32_t peers = __match_any_sync(vmask, (unsigned long long)s[u]);
        const uint32_t leads = __ballot_sync(vmask, lead[u] != 0) & peers;
        const uint32_t imin = __reduce_min_sync(peers, (uint32_t)i);
        if (lane == (uint32_t)(__ffs(peers) - 1)) {
          atomicMax(&p.slots[s[u]].rep, ~imin);
          atomicAdd(&p.slots[s[u]].info, (uint32_t)__popc(peers) | (leads ? 0x80000000u : 0u));
        }
      }
    }
  }
}

// Target-range sweep for exact packed keys whose id mirror exceeds the L2 share
// a pass can keep resident (8/16-bit mirrors of 100/200 MB at n = 1e8): sweep s
// only gathers ids of targets in [lo, hi) — a <= 50 MB slice of the mirror that
// stays in L2 — and ORs them into the partial key (fields are disjoint bit
// ranges, so the sweeps commute).  delta is re-streamed per sweep (evict-first).
template <int kIdBits, int kK>
__global__ void __launch_bounds__(256) sweep_kernel(InsertParams p, uint32_t lo, uint32_t hi,
                                                    bool first) {
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_ids = policy_evict_last();
  const uint32_t k = kK > 0 ? (uint32_t)kK : p.k;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.m; i += stride) {
    const uint32_t q = p.act ? p.act[i] : (uint32_t)i;
    unsigned long long key = first ? (unsigned long long)p.block[q] << (k * p.w) : p.keys[i];
#pragma unroll
    for (int a = 0; a < (kK > 0 ? kK : 1); ++a) {
      for (uint32_t aa = (kK > 0 ? (uint32_t)a : 0u); aa < (kK > 0 ? (uint32_t)a + 1 : k); ++aa) {
        const uint32_t t = ld_stream(p.delta + (uint64_t)aa * p.n + q, pol_stream);
        if (t >= lo && t < hi)
          key |= (unsigned long long)load_id<kIdBits>(p.ids, t, pol_ids) << ((k - 1 - aa) * p.w);
      }
    }
    p.keys[i] = key;
  }
}

// K1 for tiny direct tables (pass 1: 2^(k+1) keys): CTA aggregation in smem
template <int kIdBits, int kK, bool kFromKeys = false>
__global__ void __launch_bounds__(256) insert_small_kernel(InsertParams p, uint32_t table) {
  extern __shared__ uint32_t s_small[];  // [table] rep, [table] info (dynamic: tiny tables
  uint32_t* s_rep = s_small;              //  leave room for many CTAs per SM)
  uint32_t* s_info = s_small + table;
  for (uint32_t t = threadIdx.x; t < table; t += blockDim.x) {
    s_rep[t] = 0;
    s_info[t] = 0;
  }
  __syncthreads();
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_ids = policy_evict_last();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t start = p.i0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t base = start - (threadIdx.x & 31); base < p.m; base += stride) {
    const uint64_t i = base + (threadIdx.x & 31);
    const bool valid = i < p.m;
    const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
    if (!valid) continue;
    const uint32_t q = p.act ? p.act[i] : (uint32_t)i;
    const uint32_t b = p.block[q];
    const uint32_t s = kFromKeys ? (uint32_t)p.keys[i]
                                 : (uint32_t)make_key<kIdBits, false, kK>(p, i, q, b, pol_stream,
                                                                          pol_ids);
    p.slot_of[i] = s;
    if (p.ids_out) p.ids_out[q] = s + p.id_off;
    // lanes are in ascending i: the lowest lane of each key group updates for all
    const uint32_t peers = __match_any_sync(vmask, s);
    const uint32_t leads = __ballot_sync(vmask, p.lead[q] != 0) & peers;
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) {
      atomicMax(&s_rep[s], ~(uint32_t)i);
      atomicAdd(&s_info[s], (uint32_t)__popc(peers) | (leads ? 0x80000000u : 0u));
    }
  }
  __syncthreads();
  for (uint32_t t = threadIdx.x; t < table; t += blockDim.x) {
    if (s_info[t] != 0) {
      atomicMax(&p.slots[t].rep, s_rep[t]);
      atomicAdd(&p.slots[t].info, s_info[t]);
    }
  }
}

// Uniqueness filter for hash-table passes (most keys distinct, e.g. the last
// refinement passes of random DFAs): 2^28 cells, a "seen" and a "seen twice" bit each (64 MB), an
// L2-resident footprint (tools/l2_bench.cu: ~190 G atomics/s vs ~21-25 G/s for
// a > L2 table).  Keys alone in their cell are singleton groups and skip the
// global table; only the rest (true duplicates + cell collisions) is inserted.
#ifndef DFM_FILTER_CELL_BITS  // (build-variant experiments)
#define DFM_FILTER_CELL_BITS 28
#endif
constexpr int kFilterCellBits = DFM_FILTER_CELL_BITS;
// "seen" and "seen twice" as two bitmaps of 2^28 bits: the returning atomics of every
// key hit the 32 MB "seen" half, the mark reads only the sparse "twice" half (0 = the
// 2-bit cells of round 1, for A/B builds): flag scans 935 -> 815 and 580 -> 457 us
#ifndef DFM_FILTER_SPLIT
#define DFM_FILTER_SPLIT 1
#endif
// cell c's "seen twice" bit
__device__ __forceinline__ bool filt_dup(const uint32_t* F, uint64_t c) {
  if (DFM_FILTER_SPLIT)
    return (F[(1ull << (kFilterCellBits - 5)) + (c >> 5)] >> (uint32_t)(c & 31)) & 1u;
  return (F[c >> 4] >> ((uint32_t)(c & 15) * 2 + 1)) & 1u;
}

__device__ __forceinline__ unsigned long long table_hash(unsigned long long key, bool hashed,
                                                         uint64_t seed) {
  return hashed ? key : mix64(key ^ seed);
}

// keys stream through L2 with evict_first so the 64 MB filter stays resident
__device__ __forceinline__ unsigned long long ld_key_stream(const unsigned long long* a,
                                                            uint64_t pol) {
  unsigned long long v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t atom_or_keep(uint32_t* a, uint32_t v, uint64_t pol) {
  uint32_t old;
  asm volatile("atom.global.or.L2::cache_hint.b32 %0, [%1], %2, %3;"
               : "=r"(old) : "l"(a), "r"(v), "l"(pol) : "memory");
  return old;
}
// (no result needed: a fire-and-forget reduction, no round trip)
__device__ __forceinline__ void red_or_keep(uint32_t* a, uint32_t v, uint64_t pol) {
  asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol)
               : "memory");
}

// level 0 uses hash bits [36, 64), level 1 bits [8, 36) of the same 64-bit table hash;
// level 1 only sees the candidates level 0 left (slot_of != kUnique)
__global__ void __launch_bounds__(256) filt_set_kernel(const unsigned long long* __restrict__ keys,
                                                       uint64_t m, bool hashed, uint64_t seed,
                                                       uint32_t* F, int level,
                                                       const uint32_t* __restrict__ cand) {
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  const int shift = level == 0 ? 64 - kFilterCellBits : 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    const uint64_t i = cand ? cand[j] : j;  // level 1: the candidates level 0 left
    const uint64_t c = (table_hash(ld_key_stream(keys + i, pol_stream), hashed, seed) >> shift) &
                       ((1ull << kFilterCellBits) - 1);
    if (DFM_FILTER_SPLIT) {
      const uint32_t bit = 1u << (uint32_t)(c & 31);
      const uint32_t old = atom_or_keep(&F[c >> 5], bit, pol_keep);
      if (old & bit) red_or_keep(&F[(1ull << (kFilterCellBits - 5)) + (c >> 5)], bit, pol_keep);
    } else {
      const uint32_t b = (uint32_t)(c & 15) * 2;
      const uint32_t old = atom_or_keep(&F[c >> 4], 1u << b, pol_keep);
      if (((old >> b) & 3u) == 1u) red_or_keep(&F[c >> 4], 2u << b, pol_keep);
    }
  }
}

// mark: keys alone in their cell leave (slot_of = kUnique), the others stay candidates
__global__ void __launch_bounds__(256) filt_mark_kernel(const unsigned long long* __restrict__ keys,
                                                        uint64_t m, bool hashed, uint64_t seed,
                                                        const uint32_t* __restrict__ F,
                                                        uint32_t* __restrict__ slot_of, int level,
                                                        const uint32_t* __restrict__ cand) {
  const uint64_t pol_stream = policy_evict_first();
  const int shift = level == 0 ? 64 - kFilterCellBits : 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    const uint64_t i = cand ? cand[j] : j;
    const uint64_t c = (table_hash(ld_key_stream(keys + i, pol_stream), hashed, seed) >> shift) &
                       ((1ull << kFilterCellBits) - 1);
    slot_of[i] = filt_dup(F, c) ? 0u : kUnique;
  }
}

// mark + compact in one look-back pass (prims::lookback_flags): a key alone in its
// cell leaves — as a singleton block right away under relabel-in-place (id B + i,
// its own leader; rip_hashed_cand_kernel then visits the table states only), else
// slot_of = kUnique — and the others stay candidates, in ascending state order
struct FiltPred {
  const unsigned long long* keys;
  const uint32_t* F;
  const uint32_t* cand;  // nullptr: the identity list 0..m-1
  uint64_t seed;
  bool hashed;
  int shift;
  __device__ bool operator()(uint64_t j) const {
    const uint64_t i = cand ? cand[j] : j;
    const uint64_t c = (table_hash(ld_key_stream(keys + i, policy_evict_first()), hashed, seed) >>
                        shift) & ((1ull << kFilterCellBits) - 1);
    return filt_dup(F, c);
  }
};
struct FiltOut {
  const uint32_t* cand;
  uint32_t* out;
  uint32_t* slot_of;  // plain passes
  uint32_t* ids;      // relabel-in-place passes (non-null): ids, lead, flag
  uint8_t* lead;
  uint8_t* flag;
  uint32_t B;
  __device__ void operator()(uint64_t j, uint32_t rank, uint32_t dup) const {
    const uint32_t i = cand ? cand[j] : (uint32_t)j;
    if (dup) {
      out[rank] = i;
      if (!ids) slot_of[i] = 0u;
    } else if (ids) {
      ids[i] = B + i;
      lead[i] = 1;
      flag[i] = 0;
    } else {
      slot_of[i] = kUnique;
    }
  }
};

// candidates in ascending state order (look-back scan over the previous list)
struct CandIn {
  const uint32_t* cand;  // nullptr: the identity list 0..m-1
  const uint32_t* slot_of;
  __device__ uint32_t operator()(uint64_t j) const {
    return slot_of[cand ? cand[j] : (uint32_t)j] != kUnique ? 1u : 0u;
  }
};
struct CandOut {
  const uint32_t* cand;
  uint32_t* out;
  __device__ void operator()(uint64_t j, uint32_t excl, uint32_t v) const {
    if (v) out[excl] = cand ? cand[j] : (uint32_t)j;
  }
};

// two signature rows differ?  Rows of large alphabets are padded to 8-word strides:
// 16-byte loads, 16 words of each row in flight per step (words past `words` are
// padding and masked)
__device__ __forceinline__ bool rows_differ(const uint32_t* __restrict__ sig, uint32_t row,
                                            uint32_t words, uint64_t i, uint64_t j) {
  const uint32_t* a = sig + i * (uint64_t)row;
  const uint32_t* b = sig + j * (uint64_t)row;
  if ((row & 7) == 0) {
    const uint4* a4 = reinterpret_cast<const uint4*>(a);
    const uint4* b4 = reinterpret_cast<const uint4*>(b);
    for (uint32_t x = 0; x < words; x += 16) {
      uint32_t diff = 0;
#pragma unroll
      for (uint32_t y = 0; y < 4; ++y) {
        const uint32_t w = x + 4 * y;
        if (w < words) {
          const uint4 u = a4[w / 4], v = b4[w / 4];
          diff |= (u.x ^ v.x) | (w + 1 < words ? u.y ^ v.y : 0u) |
                  (w + 2 < words ? u.z ^ v.z : 0u) | (w + 3 < words ? u.w ^ v.w : 0u);
        }
      }
      if (diff) return true;
    }
    return false;
  }
  uint32_t diff = 0;
  for (uint32_t x = 0; x < words; x += 4) {  // 4 independent words in flight
#pragma unroll
    for (uint32_t y = 0; y < 4; ++y)
      if (x + y < words) diff |= a[x + y] ^ b[x + y];
    if (diff) return true;
  }
  return false;
}

struct ResolveItem {
  uint32_t v;      // 1 = minimum member of a group that gets a fresh id
  uint32_t slot;
  uint32_t flags;  // bit0 rep, bit1 singleton, bit2 keeper
};

struct ResolveIn {
  const Slot* slots;
  const uint32_t* slot_of;
  const uint32_t* sig;  // nullptr: exact packed keys
  uint32_t words, row;
  unsigned long long* collision;
  const uint32_t* act;  // filtered passes: kUnique states are singleton groups
  const uint8_t* lead;
  __device__ ResolveItem operator()(uint64_t i) const {
    const uint32_t s = slot_of[i];
    if (s == kUnique) {
      const bool keeper = lead[act ? act[i] : (uint32_t)i] != 0;
      ResolveItem it;
      it.v = keeper ? 0u : 1u;
      it.slot = s;
      it.flags = 1u | 2u | (keeper ? 4u : 0u);
      return it;
    }
    const uint2 sl = *reinterpret_cast<const uint2*>(&slots[s].rep);
    const uint32_t rep_i = ~sl.x;
    const uint32_t cnt = sl.y & 0x7FFFFFFFu;
    const bool keeper = (sl.y >> 31) != 0;
    const bool is_rep = rep_i == (uint32_t)i;
    if (!is_rep && sig != nullptr) {  // equal hash: verify the full signature
      if (rows_differ(sig, row, words, i, rep_i)) atomicOr(collision, 1ull);
    }
    ResolveItem it;
    it.v = (is_rep && !keeper) ? 1u : 0u;
    it.slot = s;
    it.flags = (is_rep ? 1u : 0u) | (cnt == 1 ? 2u : 0u) | (keeper ? 4u : 0u);
    return it;
  }
};

// st[i]: bit0 take the id from the slot, bit1 stays active, bit2 new leader
struct ResolveOut {
  Slot* slots;
  const uint32_t* act;
  const uint32_t* block;
  uint32_t* res;
  uint8_t* st;
  uint32_t B;
  __device__ void operator()(uint64_t i, uint32_t excl, const ResolveItem& it) const {
    if (it.flags & 1u) {
      const uint32_t q = act ? act[i] : (uint32_t)i;
      const uint32_t gid = (it.flags & 4u) ? block[q] : B + excl;
      res[i] = gid;
      if (it.flags & 2u) {
        st[i] = (it.flags & 4u) ? 0u : 4u;
      } else {
        slots[it.slot].key = gid;  // publish for the other members
        st[i] = 2u | ((it.flags & 4u) ? 0u : 4u);
      }
    } else {
      st[i] = 3u;
    }
  }
};

// K2 without a global scan: fresh ids are handed out by one atomic per CTA step
// (any numbering of the new blocks yields the same partition; canonical labels
// come from the leader flags), so every state resolves independently
constexpr int kResolveItems = 4;

// *inactive is set when some group is a singleton (its state leaves the active list):
// passes without one reuse the active list instead of compacting it
__global__ void __launch_bounds__(256) resolve_kernel(uint64_t m, ResolveIn in, ResolveOut out,
                                                      unsigned long long* fresh,
                                                      unsigned long long* inactive) {
  constexpr int U = kResolveItems;
  __shared__ uint32_t s_cnt[8 * U];
  __shared__ uint32_t s_first;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  bool any_single = false;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * U; base < m; base += stride) {
    ResolveItem it[U];
    uint32_t want[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + u * blockDim.x + threadIdx.x;
      if (i < m) {
        it[u] = in(i);
        any_single |= (it[u].flags & 3u) == 3u;  // the rep of a one-member group
      } else {
        it[u].v = 0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      want[u] = __ballot_sync(0xffffffffu, it[u].v != 0);
      if (lane == 0) s_cnt[u * 8 + warp] = __popc(want[u]);
    }
    __syncthreads();
    // exclusive offsets of the (item slot, warp) groups; one atomic for the CTA step
    if (threadIdx.x == 0) {
      uint32_t total = 0;
      for (int g = 0; g < 8 * U; ++g) total += s_cnt[g];
      s_first = total ? (uint32_t)atomicAdd(fresh, (unsigned long long)total) : 0u;
    }
    __syncthreads();
    uint32_t off = s_first;
    for (int g = 0; g < (int)warp; ++g) off += s_cnt[g];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + u * blockDim.x + threadIdx.x;
      if (i < m) out(i, off + (uint32_t)__popc(want[u] & ((1u << lane) - 1u)), it[u]);
      // advance past this slot's remaining warps and the next slot's earlier warps
      for (int g = (int)warp; g < 8; ++g) off += s_cnt[u * 8 + g];
      if (u + 1 < U)
        for (int g = 0; g < (int)warp; ++g) off += s_cnt[(u + 1) * 8 + g];
    }
    __syncthreads();
  }
  if (__syncthreads_or(any_single) && threadIdx.x == 0) atomicOr(inactive, 1ull);
}

__global__ void __launch_bounds__(256) apply_kernel(uint64_t m, const uint32_t* __restrict__ act,
                                                    const uint32_t* __restrict__ res,
                                                    const uint8_t* __restrict__ st,
                                                    const uint32_t* __restrict__ slot_of,
                                                    const Slot* __restrict__ slots,
                                                    uint32_t* __restrict__ block,
                                                    uint8_t* __restrict__ flag,
                                                    uint8_t* __restrict__ lead,
                                                    const uint64_t* scalars) {
  if (scalars[2] != 0) return;  // collision: the pass is void
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint32_t s = st[i];
    const uint32_t q = act ? act[i] : (uint32_t)i;
    const uint32_t gid = (s & 1u) ? (uint32_t)slots[slot_of[i]].key : res[i];
    block[q] = gid;
    flag[q] = (s >> 1) & 1u;
    if (s & 4u) lead[q] = 1;
  }
}

// relabel-in-place passes (direct tables: the key, or its rank among the keys
// present, is the new id — any numbering gives the same partition): one thread per
// group marks its minimum member as the block leader (old leaders are the minimum
// of their group too) and counts groups; *single: a one-member group exists (only
// known where the slots keep group sizes; the rank-compacted passes do not, and
// their one-member groups simply stay on the active list)
__global__ void __launch_bounds__(256) rip_groups_kernel(const Slot* __restrict__ slots,
                                                         uint64_t ntab,
                                                         const uint32_t* __restrict__ act,
                                                         uint8_t* __restrict__ lead,
                                                         unsigned long long* groups,
                                                         unsigned long long* single) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t mine = 0;
  bool one = false;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntab; t += stride) {
    const uint2 sl = *reinterpret_cast<const uint2*>(&slots[t].rep);
    if (sl.x == 0) continue;  // no member (rep holds ~min member)
    const uint32_t i = ~sl.x;
    lead[act ? act[i] : i] = 1;
    ++mine;
    one |= (sl.y & 0x7FFFFFFFu) == 1u;  // (rank-compacted passes keep no sizes: never)
  }
  mine = __reduce_add_sync(0xffffffffu, mine);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(groups, (unsigned long long)mine);
  if (__any_sync(0xffffffffu, one) && (threadIdx.x & 31) == 0) atomicOr(single, 1ull);
}

// relabel-in-place for filtered (hash-table) passes over ALL states: a state the
// filter found unique is a singleton block (its own leader) with id B + i; a table
// state takes B + m + slot, members verified against the group's minimum (a hash
// collision voids the pass: the ids go to `ids` — swapped in for the block array
// only after the check — and every leader flag set here is right regardless)
__global__ void __launch_bounds__(256) rip_hashed_kernel(uint64_t m,
                                                         const uint32_t* __restrict__ slot_of,
                                                         const Slot* __restrict__ slots,
                                                         const uint32_t* __restrict__ sig,
                                                         uint32_t words, uint32_t row,
                                                         unsigned long long* collision,
                                                         uint32_t B, uint32_t* __restrict__ ids,
                                                         uint8_t* __restrict__ lead,
                                                         uint8_t* __restrict__ flag) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint32_t s = slot_of[i];
    if (s == kUnique) {
      ids[i] = B + (uint32_t)i;
      lead[i] = 1;
      flag[i] = 0;
      continue;
    }
    const uint2 sl = *reinterpret_cast<const uint2*>(&slots[s].rep);
    const uint32_t rep_i = ~sl.x;
    if (rep_i != (uint32_t)i && sig != nullptr && rows_differ(sig, row, words, i, rep_i))
      atomicOr(collision, 1ull);
    ids[i] = B + (uint32_t)m + s;
    flag[i] = (sl.y & 0x7FFFFFFFu) >= 2 ? 1 : 0;
  }
}

// the table states of a filtered relabel-in-place pass (FiltOut labelled the rest)
__global__ void __launch_bounds__(256) rip_hashed_cand_kernel(
    uint64_t nc, const uint32_t* __restrict__ cand, uint64_t m,
    const uint32_t* __restrict__ slot_of, const Slot* __restrict__ slots,
    const uint32_t* __restrict__ sig, uint32_t words, uint32_t row,
    unsigned long long* collision, uint32_t B, uint32_t* __restrict__ ids,
    uint8_t* __restrict__ flag) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nc; j += stride) {
    const uint32_t i = cand[j];
    const uint32_t s = slot_of[i];
    const uint2 sl = *reinterpret_cast<const uint2*>(&slots[s].rep);
    const uint32_t rep_i = ~sl.x;
    if (rep_i != i && sig != nullptr && rows_differ(sig, row, words, i, rep_i))
      atomicOr(collision, 1ull);
    ids[i] = B + (uint32_t)m + s;
    flag[i] = (sl.y & 0x7FFFFFFFu) >= 2 ? 1 : 0;
  }
}

// states of one-member groups leave the active list
__global__ void __launch_bounds__(256) rip_flag_kernel(uint64_t m, const uint32_t* __restrict__ act,
                                                       const uint32_t* __restrict__ slot_of,
                                                       const Slot* __restrict__ slots,
                                                       uint8_t* __restrict__ flag) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
    flag[act ? act[i] : (uint32_t)i] = (slots[slot_of[i]].info & 0x7FFFFFFFu) >= 2 ? 1 : 0;
}

struct PresentIn {
  const uint32_t* present;  // interleaved {bitmap word, prefix}
  __device__ uint32_t operator()(uint64_t w) const { return __popc(present[2 * w]); }
};
struct PresentOut {
  uint32_t* present;  // the prefix goes next to its bitmap word
  __device__ void operator()(uint64_t w, uint32_t excl, uint32_t) const { present[2 * w + 1] = excl; }
};

struct ActIn {
  const uint32_t* act;
  const uint8_t* flag;
  __device__ uint32_t operator()(uint64_t i) const { return flag[act ? act[i] : (uint32_t)i]; }
};
struct ActOut {
  const uint32_t* act;
  uint32_t* act_next;
  __device__ void operator()(uint64_t i, uint32_t excl, uint32_t v) const {
    if (v) act_next[excl] = act ? act[i] : (uint32_t)i;
  }
};

// split: both an accepting and a rejecting state exist (min_sort.hpp:80-88).  Also
// writes pass 1's 1-bit id mirror.  Four consecutive states per thread (vector
// accesses); the 8 lanes covering 32 states OR their nibbles into one mirror word.
__global__ void init_kernel(const uint8_t* __restrict__ acc, uint64_t n,
                            const uint32_t* __restrict__ first2, uint32_t* __restrict__ block,
                            uint8_t* __restrict__ lead, uint32_t* __restrict__ mirror1) {
  const uint32_t fa = first2[0], fr = first2[1];
  const bool split = fa != kNoLeader && fr != kNoLeader;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;  // a multiple of 128
  for (uint64_t q0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
       q0 - 4 * lane < n; q0 += stride) {
    uint32_t nib = 0;
    if (q0 + 4 <= n) {
      const uchar4 a4 = *reinterpret_cast<const uchar4*>(acc + q0);
      const uint32_t b0 = (split && a4.x == 0), b1 = (split && a4.y == 0),
                     b2 = (split && a4.z == 0), b3 = (split && a4.w == 0);
      *reinterpret_cast<uint4*>(block + q0) = make_uint4(b0, b1, b2, b3);
      uchar4 l4;
      l4.x = (q0 == fa || q0 == fr || (!split && q0 == 0)) ? 1 : 0;
      l4.y = (q0 + 1 == fa || q0 + 1 == fr) ? 1 : 0;
      l4.z = (q0 + 2 == fa || q0 + 2 == fr) ? 1 : 0;
      l4.w = (q0 + 3 == fa || q0 + 3 == fr) ? 1 : 0;
      *reinterpret_cast<uchar4*>(lead + q0) = l4;
      nib = b0 | b1 << 1 | b2 << 2 | b3 << 3;
    } else {
      for (uint64_t q = q0; q < n; ++q) {
        const uint32_t b = (split && acc[q] == 0) ? 1u : 0u;
        block[q] = b;
        // block leaders = minimum state of each initial block (min_partref.hpp:53-63 analogue)
        lead[q] = ((uint32_t)q == fa || (uint32_t)q == fr || (!split && q == 0)) ? 1 : 0;
        nib |= b << (q - q0);
      }
    }
    uint32_t word = nib << (4 * (lane & 7));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    word |= __shfl_xor_sync(0xffffffffu, word, 4);
    if ((lane & 7) == 0 && q0 < n) mirror1[q0 >> 5] = word;
  }
}

// first accepting / rejecting state among [lo, hi); a second launch over the rest
// of the states returns at once when the first (a prefix) found both
__global__ void first_states_kernel(const uint8_t* __restrict__ acc, uint64_t lo, uint64_t hi,
                                    uint32_t* out2) {
  if (lo > 0 && *reinterpret_cast<volatile uint32_t*>(&out2[0]) != kNoLeader &&
      *reinterpret_cast<volatile uint32_t*>(&out2[1]) != kNoLeader)
    return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t fa = kNoLeader, fr = kNoLeader;
  for (uint64_t q = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += stride) {
    if (acc[q]) fa = min(fa, (uint32_t)q);
    else fr = min(fr, (uint32_t)q);
  }
  fa = __reduce_min_sync(0xffffffffu, fa);
  fr = __reduce_min_sync(0xffffffffu, fr);
  if ((threadIdx.x & 31) == 0) {
    if (fa != kNoLeader) atomicMin(&out2[0], fa);
    if (fr != kNoLeader) atomicMin(&out2[1], fr);
  }
}

// packed id mirror: 32/kBits ids per 32-bit word (ids < 2^kBits by construction)
template <int kBits>
__global__ void mirror_kernel(const uint32_t* __restrict__ block, uint64_t n,
                              uint32_t* __restrict__ out) {
  constexpr int kPer = 32 / kBits;
  const uint64_t words = (n + kPer - 1) / kPer;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const uint64_t q = w * kPer + e;
      if (q < n) word |= block[q] << (e * kBits);
    }
    out[w] = word;
  }
}

// Packed mirror with FB-bit fields, 32/FB per word (FB = 5: six ids per word, 66.7
// MB at 1e8 states instead of the 8-bit mirror's 100 MB): the L2-resident source
// of the direct-gather keys below.
template <int FB>
__global__ void mirror_packed_kernel(const uint32_t* __restrict__ block, uint64_t n,
                                     uint32_t* __restrict__ out) {
  constexpr int kPer = 32 / FB;
  const uint64_t words = (n + kPer - 1) / kPer;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const uint64_t q = w * kPer + e;
      if (q < n) word |= block[q] << (e * FB);
    }
    out[w] = word;
  }
}

// Exact packed keys of the active states by direct gathers from the packed mirror
// (the blocked builder's output, without its layout): key = (block[q], id(δa(q))...)
// and the presence bit of the key in the rank-compacted direct table (interleaved
// {bitmap word, exclusive popcount} pairs).  Used for passes whose ids fit FB <= 8
// bits: the mirror is L2-resident, so the gathers run at the L2 request rate and the
// blocked layout is left to the 32-bit passes (built on the side stream meanwhile).
template <int FB, int kK>
__global__ void __launch_bounds__(256) direct_keys_kernel(
    const uint32_t* __restrict__ delta, uint64_t n, uint32_t kr, const uint32_t* __restrict__ mirror,
    const uint32_t* __restrict__ act, uint64_t m, const uint32_t* __restrict__ block, int w,
    unsigned long long* __restrict__ keys, uint32_t* present) {
  constexpr uint32_t kPer = 32 / FB;
  constexpr uint32_t kMask = (1u << FB) - 1u;
  const uint32_t k = kK > 0 ? (uint32_t)kK : kr;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_ids = policy_evict_last();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint32_t q = act ? act[i] : (uint32_t)i;
    unsigned long long key = block[q];
    uint32_t t[kK > 0 ? kK : 8];
    for (uint32_t a0 = 0; a0 < k; a0 += (kK > 0 ? kK : 8)) {
      const uint32_t na = kK > 0 ? (uint32_t)kK : min(8u, k - a0);
#pragma unroll
      for (uint32_t a = 0; a < (kK > 0 ? (uint32_t)kK : 8u); ++a)
        if (a < na) t[a] = ld_stream(delta + (uint64_t)(a0 + a) * n + q, pol_stream);
      uint32_t wd[kK > 0 ? kK : 8];
#pragma unroll
      for (uint32_t a = 0; a < (kK > 0 ? (uint32_t)kK : 8u); ++a)
        if (a < na) {
          asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;"
              : "=r"(wd[a]) : "l"(mirror + t[a] / kPer), "l"(pol_ids));
        }
#pragma unroll
      for (uint32_t a = 0; a < (kK > 0 ? (uint32_t)kK : 8u); ++a)
        if (a < na) key = (key << w) | ((wd[a] >> ((t[a] % kPer) * FB)) & kMask);
    }
    keys[i] = key;
    const uint32_t bit = 1u << (key & 31);
    uint32_t* word = present + 2 * (key >> 5);
    if (!(prims::ld_hint_u32(word) & bit)) atomicOr(word, bit);
  }
}

bool pass_timing() {
  const char* e = getenv("DFM_SORTPR_PASS_TIMING");
  return e != nullptr && e[0] == '1';
}

// opt-in (DFM_SORTPR_DIRECT=1): measured slower on random_dfa(1e8, 4) — 2.0 ms for the
// 4e8 gathers from the 66.7 MB 5-bit mirror while the layout streams beside it, vs
// 1.7 ms for the blocked pass (profiles/r02c)
bool pass_direct_enabled() {
  const char* e = getenv("DFM_SORTPR_DIRECT");
  return e != nullptr && e[0] == '1';
}

// canonical labels from maintained leaders (leader = minimum state of its block):
// label(block) = rank of its leader among all leaders (core.hpp:123-136)
struct LeadIn {
  const uint8_t* lead;
  __device__ uint32_t operator()(uint64_t q) const { return lead[q]; }
};
struct LeadOut {
  const uint32_t* block;
  uint32_t* canon_of_block;
  __device__ void operator()(uint64_t q, uint32_t excl, uint32_t v) const {
    if (v) canon_of_block[block[q]] = excl;
  }
};
__global__ void canon_gather_kernel(const uint32_t* __restrict__ block, uint64_t n,
                                    const uint32_t* __restrict__ canon_of_block,
                                    uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride)
    out[q] = canon_of_block[block[q]];
}
__global__ void iota_kernel(uint32_t* __restrict__ out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride)
    out[q] = (uint32_t)q;
}

constexpr uint64_t kBlockedMinTransitions = 1ull << 25;
constexpr uint64_t kPartMinStates = 1ull << 20;
constexpr uint64_t kFilterMinStates = 1ull << 22;
// below this the gathered id mirror stays in L2 and direct gathers win
constexpr uint64_t kBlockedMinMirror = 32ull << 20;

#include "sortpr_blocked.cuh"
#include "sortpr_group.cuh"
#include "sortpr_small.cuh"

unsigned grid_for(const Ctx& ctx, uint64_t items, int per_sm = 16) {
  return (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(items, 1), 256),
                                      (uint64_t)ctx.num_sms * per_sm);
}

int bit_width_u32(uint32_t x) { return x == 0 ? 0 : 32 - __builtin_clz(x); }

template <int kIdBits, int kK>
void launch_insert_k(Ctx& ctx, const InsertParams& p, bool hashed, bool direct, uint64_t table) {
  const unsigned grid = grid_for(ctx, p.m);
  constexpr uint64_t kSweepSlice = 48ull << 20;  // mirror bytes per sweep (L2-resident)
  const uint64_t mirror_bytes = p.n * (uint64_t)kIdBits / 8;
  if ((kIdBits == 8 || kIdBits == 16) && !hashed && !(direct && table <= kSmallTable) &&
      mirror_bytes > kSweepSlice && p.keys != nullptr) {
    const uint64_t sweeps = ceil_div(mirror_bytes, kSweepSlice);
    const uint64_t width = ceil_div(p.n, sweeps);
    for (uint64_t s = 0; s < sweeps; ++s) {
      const uint64_t lo = s * width, hi = std::min<uint64_t>(p.n, lo + width);
      sweep_kernel<kIdBits, kK><<<grid, 256, 0, ctx.stream>>>(p, (uint32_t)lo, (uint32_t)hi,
                                                              s == 0);
      DFM_LAUNCH_CHECK();
    }
    if (direct)
      insert_kernel<kIdBits, false, true, kK, true><<<grid, 256, 0, ctx.stream>>>(p);
    else
      insert_kernel<kIdBits, false, false, kK, true><<<grid, 256, 0, ctx.stream>>>(p);
    DFM_LAUNCH_CHECK();
    return;
  }
  if (direct && table <= kSmallTable)
    insert_small_kernel<kIdBits, kK><<<std::min<unsigned>(grid, ctx.num_sms * 8), 256,
                                       2 * table * sizeof(uint32_t), ctx.stream>>>(p, (uint32_t)table);
  else if (direct)
    insert_kernel<kIdBits, false, true, kK><<<grid, 256, 0, ctx.stream>>>(p);
  else if (hashed)
    insert_kernel<kIdBits, true, false, kK><<<grid, 256, 0, ctx.stream>>>(p);
  else
    insert_kernel<kIdBits, false, false, kK><<<grid, 256, 0, ctx.stream>>>(p);
  DFM_LAUNCH_CHECK();
}

template <int kIdBits>
void launch_insert(Ctx& ctx, const InsertParams& p, bool hashed, bool direct, uint64_t table) {
  switch (p.k) {  // compile-time alphabets for the common small k
    case 1: return launch_insert_k<kIdBits, 1>(ctx, p, hashed, direct, table);
    case 2: return launch_insert_k<kIdBits, 2>(ctx, p, hashed, direct, table);
    case 3: return launch_insert_k<kIdBits, 3>(ctx, p, hashed, direct, table);
    case 4: return launch_insert_k<kIdBits, 4>(ctx, p, hashed, direct, table);
    default: return launch_insert_k<kIdBits, 0>(ctx, p, hashed, direct, table);
  }
}

// K1 from precomputed keys (blocked builder): packed or hashed, direct or probed
template <int kK>
void launch_insert_keys(Ctx& ctx, const InsertParams& p, bool hashed, bool direct, uint64_t table,
                        bool filtered) {
  const unsigned grid = grid_for(ctx, p.m);
  if (filtered) {
    if (hashed) insert_kernel<32, true, false, kK, true, true><<<grid, 256, 0, ctx.stream>>>(p);
    else insert_kernel<32, false, false, kK, true, true><<<grid, 256, 0, ctx.stream>>>(p);
  } else if (direct && table <= kSmallTable)
    insert_small_kernel<32, kK, true><<<std::min<unsigned>(grid, ctx.num_sms * 8), 256,
                                        2 * table * sizeof(uint32_t), ctx.stream>>>(p, (uint32_t)table);
  else if (hashed)
    insert_kernel<32, true, false, kK, true><<<grid, 256, 0, ctx.stream>>>(p);
  else if (direct)
    insert_kernel<32, false, true, kK, true><<<grid, 256, 0, ctx.stream>>>(p);
  else
    insert_kernel<32, false, false, kK, true><<<grid, 256, 0, ctx.stream>>>(p);
  DFM_LAUNCH_CHECK();
}

// words of a signature row written by make_key_rows_warp (fields packed at the pass's
// mirror width; measured on C2 sortPR, vlts(1000, 1e7, 100): 29.2 -> 23.6 ms,
// profiles/r04/r04l.  Bit-exact packing at bits(B - 1) — 32 instead of 51 words at
// 10-bit ids — wrote less but cost more instructions per field: 31.4 ms, r04o)
uint32_t packed_row_words(uint64_t k, int id_bits) {
  const uint64_t per = 32 / (uint64_t)id_bits;
  return (uint32_t)((k + 1 + per - 1) / per);
}

bool layout_overlap_enabled() {  // DFM_SORTPR_LAYOUT_OVERLAP=0: build it at pass 2 (tests)
  const char* e = getenv("DFM_SORTPR_LAYOUT_OVERLAP");
  return e == nullptr || e[0] != '0';
}

bool tile24_enabled() {  // DFM_SORTPR_TILE24=0: 4-byte tiles for all 32-bit passes (tests)
  const char* e = getenv("DFM_SORTPR_TILE24");
  return e == nullptr || e[0] != '0';
}

bool rip_enabled() {  // DFM_SORTPR_RIP=0: resolve/apply on every pass (tests)
  const char* e = getenv("DFM_SORTPR_RIP");
  return e == nullptr || e[0] != '0';
}

bool small_enabled() {
  const char* e = getenv("DFM_SORTPR_SMALL");
  return e == nullptr || e[0] != '0';
}

unsigned small_grid(const Ctx& ctx, uint64_t n) {
  const int per_sm = per_device_memo((const void*)small_sortpr_kernel, ctx.device,
                                     [](const void*) {
    int v = 0;
    DFM_CUDA(cudaFuncSetAttribute(small_sortpr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSmallSmem));
    DFM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, small_sortpr_kernel,
                                                           kSmallThreads, kSmallSmem));
    return v;
  });
  // >= 256 states per CTA (fewer CTAs: cheaper grid barriers), all SMs once n > 37,888
  const uint64_t grid = std::min<uint64_t>((uint64_t)per_sm * ctx.num_sms, ceil_div(n, 256));
  return grid * kSmallThreads * kSmallPer >= n ? (unsigned)grid : 0u;
}

bool small_timing() {
  const char* e = getenv("DFM_SMALL_TIMING");
  return e != nullptr && e[0] == '1';
}

// Small automata: the whole minimization in one persistent kernel (sortpr_small.cuh):
// initial partition, every pass, canonical labels.  Returns 1 at the fixpoint
// (canonical labels in `canon`), 0 when the host loop must take over (keys wider
// than 62 bits; block / lead / B and the pass count are then in its format), -1 on
// deadline expiry.
constexpr uint64_t kSmallSeed = 0x5EED5A11ull;

int run_small(Ctx& ctx, const DevDfa& d, const Deadline& dl, unsigned grid, uint32_t* block,
              uint8_t* lead, uint8_t* flag, uint32_t* canon, uint32_t& B,
              uint64_t& iterations) {
  const uint32_t n = d.n;
  const uint64_t cap0 = small_cap(n);
  Slot* t0 = static_cast<Slot*>(ctx.slot("ss.tab0", cap0 * sizeof(Slot)));
  Slot* t1 = static_cast<Slot*>(ctx.slot("ss.tab1", cap0 * sizeof(Slot)));
  auto* ctr = ctx.slot_t<unsigned long long>("ss.ctr", 6);
  auto* st = ctx.slot_t<uint32_t>("ss.state", 4);
  uint32_t* cob = ctx.slot_t<uint32_t>("ss.cob", n);
  uint32_t* cta_cnt = ctx.slot_t<uint32_t>("ss.ctacnt", grid);
  uint32_t* cta_first = ctx.slot_t<uint32_t>("ss.ctafirst", 2ull * grid);
  uint32_t* h = reinterpret_cast<uint32_t*>(ctx.h_scalars + 24);
  h[1] = 0;
  const bool timing = small_timing();
  unsigned long long* tdbg =
      timing ? ctx.slot_t<unsigned long long>("ss.tdbg", 8 * 4096 + 1) : nullptr;
  // per pass and state: delta k*4, ids (k+1)*4, flag + lead 2, slot CAS/atomics 16,
  // slot read 8, id write 4
  const uint64_t pass_bytes = (uint64_t)n * (8ull * d.k + 34);
  const uint32_t per_cta = (uint32_t)ceil_div(ceil_div(n, grid), 32) * 32;
  uint32_t tab = 1024;
  while (tab < 2 * per_cta && tab < kSmallTab) tab <<= 1;
  uint32_t chunk = 64;
  bool first_launch = true;
  while (true) {
    if (dl.expired()) return -1;
    SmallArgs a{d.delta, n,          d.k,     block,    lead,  flag,   t0,
                t1,      ctr,        st,      chunk,    kSmallSeed,     per_cta,
                tab - 1, d.acc,      cta_first, first_launch, canon, cob, cta_cnt, tdbg};
    first_launch = false;
    chunk = std::min<uint32_t>(4096, chunk * 2);
    void* args[] = {&a};
    const uint32_t before = h[1];
    ProfScope prof(ctx, "small", 0);
    DFM_CUDA(cudaLaunchCooperativeKernel((const void*)small_sortpr_kernel, grid, kSmallThreads,
                                         args, kSmallSmem, ctx.stream));
    DFM_LAUNCH_CHECK();
    prof.stop();
    DFM_CUDA(cudaMemcpyAsync(h, st, 16, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    const uint32_t done = h[1] - before;
    prof.bytes = (uint64_t)done * pass_bytes;
    if (timing) {
      std::vector<unsigned long long> t(8 * done + 1);
      DFM_CUDA(cudaMemcpy(t.data(), tdbg, t.size() * 8, cudaMemcpyDeviceToHost));
      auto us = [&](uint32_t x, int a, int b) {
        return t[8 * x + b] > t[8 * x + a] ? (t[8 * x + b] - t[8 * x + a]) * 1e-3 : 0.0;
      };
      for (uint32_t x = 0; x < done; ++x)
        fprintf(stderr, "small pass %u: A %.2f us (keys %.2f flush %.2f)  B %.2f us\n",
                before + x + 1, us(x, 0, 1), us(x, 0, 4), us(x, 4, 5), us(x, 1, 2));
    }
    B = h[0];
    iterations = h[1];
    if (h[3] == 1) return 1;
    if (h[3] == 2) return 0;
  }
}

// partitioned grouping (sortpr_group.cuh) is opt-in until its radix passes beat the
// filter mark fused with its candidate compaction (DFM_SORTPR_FILT_FUSED=0: the
// separate mark kernel + scan, for A/B runs)
bool filt_fused() {
  const char* e = getenv("DFM_SORTPR_FILT_FUSED");
  return !(e && e[0] == '0');
}

// global table: DFM_SORTPR_PARTITION=1
bool partition_enabled() {
  const char* e = getenv("DFM_SORTPR_PARTITION");
  return e != nullptr && e[0] == '1';
}

bool blocked_disabled() {
  const char* e = getenv("DFM_SORTPR_BLOCKED");
  return e != nullptr && e[0] == '0';
}

// the blocked builder needs u16 range offsets / tile slots and 32-bit positions
bool layout_possible(uint64_t n, uint32_t k) {
  const uint64_t T = n * (uint64_t)k;
  return k > 0 && k <= 1024 && T < (1ull << 32) && ceil_div(n, kRs) <= kMaxRanges &&
         T >= kBlockedMinTransitions && !blocked_disabled();
}

// source window of the layout: W*k ~ kWinElems transitions, and the scatter kernel
// stages 6 bytes per window transition + 12 per range in shared memory
uint32_t layout_window(uint64_t n, uint32_t k) {
  const uint64_t R = ceil_div(n, kRs);
  uint32_t W = std::max<uint32_t>(32, (kWinElems / k) & ~31u);
  while (W > 32 && R * 12 + 4 + (uint64_t)W * k * 6 > (227u << 10))
    W = std::max<uint32_t>(32, (W / 2) & ~31u);
  return W;
}

// layout buffers and geometry; chunks of wc windows (0: one chunk)
void layout_init(Ctx& ctx, const DevDfa& d, Layout& L, uint32_t wc, uint64_t nt = 0) {
  L.n = d.n;
  L.nt = (uint32_t)(nt ? nt : d.n);
  L.k = d.k;
  L.T = L.n * L.k;
  L.R = (uint32_t)ceil_div(L.nt, kRs);
  L.W = layout_window(L.nt, L.k);
  L.E = L.W * L.k;
  L.nW = (uint32_t)ceil_div(L.n, L.W);
  L.Wc = wc == 0 ? L.nW : std::min(wc, L.nW);
  L.nC = (uint32_t)ceil_div(L.nW, L.Wc);
  const uint64_t cells = (uint64_t)L.R * L.nW;
  L.tgt = ctx.slot_t<uint16_t>("ly.tgt", L.T);
  L.lsf = ctx.slot_t<uint16_t>("ly.lsf", (uint64_t)L.nW * L.E);
  L.eidx = ctx.slot_t<uint32_t>("ly.eidx", (uint64_t)L.nW * L.E);
  L.off = ctx.slot_t<uint32_t>("ly.off", cells + 1);
  L.gb = ctx.slot_t<uint32_t>("ly.gb", (uint64_t)L.nC * L.R);
  L.pre = ctx.slot_t<uint16_t>("ly.pre", cells);
  L.wstart = ctx.slot_t<uint32_t>("ly.wstart", L.nW + 1);
  L.v = ctx.slot("ly.v", L.T * 4);
}

// chunk ch of the layout: its windows' range histograms, their bucket offsets
// (chunk-major order: the chunk's base is the transitions before it) and the
// scatter; needs only the chunk's rows of delta
void layout_chunk(Ctx& ctx, const DevDfa& d, Layout& L, uint32_t ch) {
  const uint32_t w0 = ch * L.Wc, w1 = std::min(L.nW, w0 + L.Wc), wc = w1 - w0;
  const uint64_t cells = (uint64_t)L.R * wc;
  uint32_t* cnt_w = ctx.slot_t<uint32_t>("ly.cntw", (uint64_t)L.R * L.nW);
  uint32_t* cnt_j = ctx.slot_t<uint32_t>("ly.cntj", (uint64_t)L.R * L.nW);
  const uint64_t ct = std::min<uint64_t>((uint64_t)w1 * L.W, L.n) * L.k - (uint64_t)w0 * L.E;
  // delta read twice + tgt/lsf/eidx writes + the count/offset matrices
  ProfScope ps(ctx, "layout", ct * (4ull + 4 + 2 + 2 + 4) + cells * (4ull * 4 + 2 * 2));
  const unsigned grid = (unsigned)std::min<uint64_t>(wc, (uint64_t)ctx.num_sms * 4);
  lay_count_kernel<<<grid, 512, L.R * 6 + 16, ctx.stream>>>(d.delta, L, cnt_w, w0, w1);
  DFM_LAUNCH_CHECK();
  lay_transpose_kernel<<<dim3((unsigned)ceil_div(L.R, 32), (unsigned)ceil_div(wc, 32)),
                         dim3(32, 8), 0, ctx.stream>>>(cnt_w + (uint64_t)w0 * L.R,
                                                       cnt_j + (uint64_t)w0 * L.R, wc, L.R);
  DFM_LAUNCH_CHECK();
  prims::lookback_scan(ctx, "sc.lyoff", cells, LayOffIn{cnt_j + (uint64_t)w0 * L.R},
                       LayOffOut{L.off, L.gb, L.R, wc, w0, ch, w0 * L.E, cells,
                                 ch + 1 == L.nC ? (uint64_t)L.nW * L.R : ~0ull},
                       nullptr);
  const size_t smem = (size_t)L.R * 12 + 4 + (size_t)L.E * 6;
  DFM_CUDA(cudaFuncSetAttribute(lay_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  lay_scatter_kernel<<<(unsigned)std::min<uint64_t>(wc, (uint64_t)ctx.num_sms * 2), 1024, smem,
                       ctx.stream>>>(d.delta, L, w0, w1);
  DFM_LAUNCH_CHECK();
}

// pipelined upload: validate one chunk of rows as it lands (the reference rejects
// out-of-range targets; a bad one is zeroed so no consumer gathers out of bounds,
// and the run fails after the first pass)
__global__ void sanitize_rows_kernel(uint32_t* __restrict__ delta, uint64_t n, uint32_t k,
                                     uint64_t q0, uint64_t q1, unsigned long long* bad) {
  const uint64_t len = q1 - q0, total = len * k;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  bool b = false;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const uint64_t a = i / len;
    uint32_t* x = delta + a * n + q0 + (i - a * len);
    if (*x >= n) {
      *x = 0;
      b = true;
    }
  }
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1ull);
}

void wait_chunk(Ctx& ctx, const DevDfa& d, uint32_t c) {
  if (d.gate) d.gate->wait_recorded(c);
  DFM_CUDA(cudaStreamWaitEvent(ctx.stream, d.ready[c], 0));
  const uint64_t q0 = c * d.chunk_states, q1 = std::min<uint64_t>(d.n, q0 + d.chunk_states);
  ProfScope p(ctx, "init", (q1 - q0) * d.k * 4ull);
  sanitize_rows_kernel<<<grid_for(ctx, (q1 - q0) * d.k), 256, 0, ctx.stream>>>(d.delta, d.n, d.k, q0,
                                                                             q1, d.bad);
  DFM_LAUNCH_CHECK();
}

uint32_t layout_chunk_windows() {  // DFM_LAYOUT_CHUNK_WINDOWS (tests): force chunking
  const char* e = getenv("DFM_LAYOUT_CHUNK_WINDOWS");
  return e ? (uint32_t)strtoul(e, nullptr, 10) : 0u;
}

void build_layout(Ctx& ctx, const DevDfa& d, Layout& L, uint64_t nt = 0) {
  layout_init(ctx, d, L, layout_chunk_windows(), nt);
  for (uint32_t ch = 0; ch < L.nC; ++ch) layout_chunk(ctx, d, L, ch);
}

template <int kIdBits>
void launch_layout_gather(Ctx& ctx, const Layout& L, const uint32_t* ids) {
  // ranges per CTA: the slice fills <= 192 KB, but keep >= 2 CTAs per SM busy
  const uint32_t cmax = std::max<uint32_t>(1, (uint32_t)((uint64_t)kSliceBytes * 8 / ((uint64_t)kRs * kIdBits)));
  const uint32_t c = std::max<uint32_t>(1, std::min<uint32_t>(cmax, L.R / (2 * ctx.num_sms)));
  const size_t smem = (size_t)c * kRs * kIdBits / 8 + 16;
  DFM_CUDA(cudaFuncSetAttribute(lay_gather_kernel<kIdBits>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  lay_gather_kernel<kIdBits><<<(unsigned)ceil_div(L.R, c), 1024, smem, ctx.stream>>>(L, ids, c);
  DFM_LAUNCH_CHECK();
}

template <int kIdBits, int kK>
void launch_layout_sig(Ctx& ctx, const SigParams& sp0, bool hashed, bool tile24) {
  using V = typename IdT<kIdBits>::type;
  SigParams sp = sp0;
  sp.tile_bytes = (uint32_t)(((size_t)sp.L.E * (tile24 ? 3 : sizeof(V)) + 15) & ~size_t(15));
  const size_t smem = sp.tile_bytes;
  auto go = [&](auto kern) {
    DFM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<sp.L.nW, 1024, smem, ctx.stream>>>(sp);
    DFM_LAUNCH_CHECK();
  };
  if (kIdBits == 32 && tile24) {
    if (hashed) go(lay_sig_kernel<kIdBits, kK, true, true>);
    else go(lay_sig_kernel<kIdBits, kK, false, true>);
  } else {
    if (hashed) go(lay_sig_kernel<kIdBits, kK, true>);
    else go(lay_sig_kernel<kIdBits, kK, false>);
  }
}

template <int kIdBits>
void layout_keys_bits(Ctx& ctx, const Layout& L, const uint32_t* ids, const SigParams& sp,
                      bool hashed, bool tile24) {
  launch_layout_gather<kIdBits>(ctx, L, ids);
  switch (L.k) {
    case 2: return launch_layout_sig<kIdBits, 2>(ctx, sp, hashed, tile24);
    case 4: return launch_layout_sig<kIdBits, 4>(ctx, sp, hashed, tile24);
    default: return launch_layout_sig<kIdBits, 0>(ctx, sp, hashed, tile24);
  }
}

// one pass of the blocked builder: keys[i] (+ signature rows) for the active states
void layout_keys(Ctx& ctx, Layout& L, int mirror_bits, const void* ids, const uint32_t* act,
                 uint64_t m, const uint32_t* block, int w, bool hashed, uint64_t seed,
                 unsigned long long* keys, uint32_t* sig, uint32_t row, uint32_t* vals,
                 const uint8_t* lead, uint32_t* present) {
  if (act) {
    ProfScope ps(ctx, "scan", m * 4 + L.nW * 4ull);
    lay_wstart_kernel<<<grid_for(ctx, m + 1), 256, 0, ctx.stream>>>(act, m, L.W, L.nW, L.wstart);
    DFM_LAUNCH_CHECK();
  }
  const uint64_t idb = (uint64_t)std::max(8, mirror_bits) / 8;
  SigParams sp{L,   act ? L.wstart : nullptr, act, block, w, seed, keys, hashed ? sig : nullptr,
               row, vals, lead, present};
  // per transition: tgt 2 + id write + lsf 2 + eidx 4 + id read; id slices once; per active
  // state: act 4 + own id 4 + key 8 (+ signature row)
  ProfScope ps(ctx, "sig", L.T * (8 + 2 * idb) + L.n * (uint64_t)mirror_bits / 8 +
                               m * (4ull + 4 + 8 + (vals ? 5 : 0) + (hashed ? 4ull * row : 0)));
  const uint32_t* ids32 = static_cast<const uint32_t*>(ids);
  const bool t24 = w <= 24 && tile24_enabled();  // 32-bit ids below 2^24: 3-byte tiles
  switch (mirror_bits) {
    case 1: return layout_keys_bits<1>(ctx, L, ids32, sp, hashed, t24);
    case 4: return layout_keys_bits<4>(ctx, L, ids32, sp, hashed, t24);
    case 8: return layout_keys_bits<8>(ctx, L, ids32, sp, hashed, t24);
    case 16: return layout_keys_bits<16>(ctx, L, ids32, sp, hashed, t24);
    default: return layout_keys_bits<32>(ctx, L, ids32, sp, hashed, t24);
  }
}
// partitioned grouping of one pass (sortpr_group.cuh); keys/vals from layout_keys
void group_partitioned(Ctx& ctx, uint64_t m, const uint32_t* act, unsigned long long* keys,
                       uint32_t* vals, const uint32_t* sig, uint32_t words, uint32_t row,
                       uint32_t B, uint32_t* block, uint8_t* flag, uint8_t* lead, uint64_t* sc) {
  auto* k2 = ctx.slot_t<uint64_t>("gp.k2", m);
  auto* v2 = ctx.slot_t<uint32_t>("gp.v2", m);
  auto* ok = ctx.slot_t<uint64_t>("gp.ok", m);
  auto* ov = ctx.slot_t<uint32_t>("gp.ov", m);
  auto* res = ctx.slot_t<unsigned long long>("gp.res", m);
  const uint32_t nb = 1u << kGroupBits;
  uint32_t* bstart = ctx.slot_t<uint32_t>("gp.bstart", nb + 1);
  uint64_t* Hs = reinterpret_cast<uint64_t*>(keys);
  uint32_t* Vs = vals;
  {
    ProfScope ps(ctx, "group", m * (8ull + 8));  // bucket bounds: one read of the sorted keys
    if (prims::radix_sort_pairs_bits(ctx, Hs, Vs, k2, v2, m, 0, kGroupBits, false)) {
      Hs = k2;
      Vs = v2;
    }
    grp_bounds_kernel<<<grid_for(ctx, m + 1), 256, 0, ctx.stream>>>(Hs, m, nb, bstart);
    DFM_LAUNCH_CHECK();
  }
  {
    // per item: key 8 + val 4 read, record 8 + 4 written (+ signature rows when hashed)
    ProfScope ps(ctx, "group", m * (24ull + (sig ? 8ull * words : 0)));
    GroupParams gp{Hs, Vs, bstart, nb, reinterpret_cast<unsigned long long*>(ok), ov,
                   reinterpret_cast<unsigned long long*>(sc + 1),
                   reinterpret_cast<unsigned long long*>(sc + 2), sig, words, row, B};
    const size_t smem = (size_t)kGroupTable * (sizeof(GSlot) + 4);
    per_device_memo((const void*)grp_group_kernel, ctx.device, [](const void*) {
      DFM_CUDA(cudaFuncSetAttribute(grp_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)((size_t)kGroupTable * (sizeof(GSlot) + 4))));
      return 1;
    });
    grp_group_kernel<<<nb, 512, smem, ctx.stream>>>(gp);
    DFM_LAUNCH_CHECK();
  }
  // back to i order: one radix pass by the top 8 bits of i, then an L2-local placement
  const int ib = std::max(1, 64 - __builtin_clzll(std::max<uint64_t>(m - 1, 1)));
  uint64_t* rk = ok;
  uint32_t* rv = ov;
  if (prims::radix_sort_pairs_bits(ctx, ok, ov, k2, v2, m, 32 + std::max(0, ib - 8), 8, false)) {
    rk = k2;
    rv = v2;
  }
  {
    ProfScope ps(ctx, "relabel", m * (12ull + 8));
    // resident CTAs only: the grid sweeps the i windows together, so the window being
    // placed stays in L2 and its sectors leave complete
    grp_place_kernel<<<(unsigned)std::min<uint64_t>(ceil_div(m, 256), ctx.num_sms * 8ull), 256, 0,
                       ctx.stream>>>(
        reinterpret_cast<const unsigned long long*>(rk), rv, m, res);
    DFM_LAUNCH_CHECK();
  }
  {
    ProfScope ps(ctx, "relabel", m * (8ull + 4 + 4 + 1 + 1));
    grp_apply_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(
        m, act, res, block, flag, lead, reinterpret_cast<const unsigned long long*>(sc + 2));
    DFM_LAUNCH_CHECK();
  }
}

}  // namespace

uint64_t sortpr_upload_chunk(uint64_t n, uint32_t k) {
  // the first pass consumes chunks only on its tiny direct table (2^(k+1) <= 4096 keys)
  if (k == 0 || k + 1 > 12 || n * k * 4 < (256ull << 20)) return 0;
  const uint32_t W = layout_window(n, k);
  const uint64_t wc = std::max<uint64_t>(1, ((64ull << 20) / (4ull * k)) / W);
  return wc * W;
}

// ---- the blocked builder over a shard's rows (csrc/shard_driver.cu): sources = the
// owned states, targets = all n_total states, ids from the all-gathered vector; keys
// and rows as the shard kernels make them (same packing, same hash chain)
struct ShardLayout {
  Layout L;
};
ShardLayout* shard_layout_build(Ctx& ctx, const DevDfa& loc, uint64_t n_total) {
  const uint64_t T = (uint64_t)loc.n * loc.k;
  if (!(loc.k > 0 && loc.k <= 1024 && T < (1ull << 32) && ceil_div(n_total, kRs) <= kMaxRanges &&
        T >= kBlockedMinTransitions && !blocked_disabled()))
    return nullptr;
  auto* s = new ShardLayout;
  build_layout(ctx, loc, s->L, n_total);
  return s;
}
void shard_layout_free(ShardLayout* s) { delete s; }
void shard_layout_keys(Ctx& ctx, ShardLayout* s, int id_bits, const uint32_t* full,
                       const uint32_t* own, uint64_t m, int w, bool hashed, uint64_t seed,
                       unsigned long long* keys, uint32_t* sig, uint32_t row) {
  layout_keys(ctx, s->L, id_bits, full, nullptr, m, own, w, hashed, seed, keys, sig, row,
              nullptr, nullptr, nullptr);
}

ShardLayout* radix_layout_build(Ctx& ctx, const DevDfa& d) { return shard_layout_build(ctx, d, d.n); }

// DFM_SORTPR_WEAK_HASH=<bits> (tests): the hashed keys of passes under the first seed
// (both engines' blocked builder) keep only that many bits
void sortpr_weak_hash_setup() {
  static unsigned long long mask_set = ~0ull;
  const char* e = getenv("DFM_SORTPR_WEAK_HASH");
  const unsigned long long mask =
      e ? ((1ull << std::min(63ul, strtoul(e, nullptr, 10))) - 1) : ~0ull;
  if (mask != mask_set) {
    DFM_CUDA(cudaMemcpyToSymbol(g_weak_mask, &mask, sizeof(mask)));
    mask_set = mask;
  }
}
void radix_layout_keys(Ctx& ctx, ShardLayout* s, int id_bits, const uint32_t* ids,
                       const uint32_t* act, uint64_t m, const uint32_t* block, int w, bool hashed,
                       uint64_t seed, unsigned long long* keys, uint32_t* sig, uint32_t row) {
  layout_keys(ctx, s->L, id_bits, ids, act, m, block, w, hashed, seed, keys, sig, row, nullptr,
              nullptr, nullptr);
}

AlgoOut run_sort_pr_hash(Ctx& ctx, const DevDfa& d, const Deadline& dl, const dfm_trace* trace) {
  AlgoOut out;
  const uint64_t n = d.n;
  const uint32_t k = d.k;
  out.peak_memory_estimate = n * (16 + 4ull * k);  // min_sort.hpp:121
  uint32_t* block = ctx.slot_t<uint32_t>("sh.block", n);
  uint8_t* flag = ctx.slot_t<uint8_t>("sh.flag", n);
  uint8_t* lead = ctx.slot_t<uint8_t>("sh.lead", n);
  // packed id mirror for the gathers (sized for the widest packed case, 16 bits)
  uint32_t* mirror = ctx.slot_t<uint32_t>("sh.mirror", ceil_div(n, 2) + 1);
  uint32_t* act_buf[2] = {ctx.slot_t<uint32_t>("sh.act0", n), ctx.slot_t<uint32_t>("sh.act1", n)};
  uint32_t* slot_of = ctx.slot_t<uint32_t>("sh.slotof", n);
  uint32_t* res = ctx.slot_t<uint32_t>("sh.res", n);
  uint8_t* st = ctx.slot_t<uint8_t>("sh.st", n);
  uint32_t* sig = nullptr;
  // signature rows packed back to back: a warp's consecutive rows cover whole sectors
  // (rows of large alphabets padded to whole 32-byte sectors: coalesced row writes)
  const uint32_t row = k + 1 > 8 ? ((k + 1 + 7) & ~7u) : k + 1;
  uint64_t* sc = ctx.d_scalars;  // [1] fresh [2] collision [3] next active [4] accepting
  uint32_t* first2 = reinterpret_cast<uint32_t*>(ctx.d_scalars + 16);
  const unsigned sgrid =
      (n <= kSmallMaxStates && !(trace && trace->on_pass) && small_enabled()) ? small_grid(ctx, n)
                                                                              : 0u;
  if (!sgrid) {  // (the single-kernel path initialises its own state)
    DFM_CUDA(cudaMemsetAsync(sc, 0, 40, ctx.stream));
    DFM_CUDA(cudaMemsetAsync(first2, 0xFF, 8, ctx.stream));
  }
  uint32_t B = 0;
  if (sgrid) {
    out.canon_dev = ctx.slot_t<uint32_t>("canon", n);
    const int r = run_small(ctx, d, dl, sgrid, block, lead, flag, out.canon_dev, B,
                            out.iterations);
    if (r < 0) {
      out.status = DFM_STATUS_TIMEOUT;
      return out;
    }
    if (r == 1) {
      out.num_blocks = B;
      out.canon_identity = B == n;
      out.status = DFM_STATUS_OK;
      return out;
    }
  } else {
    {
      ProfScope p(ctx, "init", n * 2);
      const uint64_t pre = std::min<uint64_t>(n, 1u << 20);
      first_states_kernel<<<grid_for(ctx, pre), 256, 0, ctx.stream>>>(d.acc, 0, pre, first2);
      DFM_LAUNCH_CHECK();
      if (pre < n)
        first_states_kernel<<<grid_for(ctx, n - pre), 256, 0, ctx.stream>>>(d.acc, pre, n, first2);
      DFM_LAUNCH_CHECK();
    }
    {
      ProfScope p(ctx, "init", n * 10);
      init_kernel<<<grid_for(ctx, ceil_div(n, 4)), 256, 0, ctx.stream>>>(d.acc, n, first2, block,
                                                                       lead, mirror);
      DFM_LAUNCH_CHECK();
    }
    DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 16, first2, 8, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    const uint32_t fa = (uint32_t)(ctx.h_scalars[16] & 0xFFFFFFFFu);
    const uint32_t fr = (uint32_t)(ctx.h_scalars[16] >> 32);
    B = (fa != kNoLeader && fr != kNoLeader) ? 2u : 1u;  // min_sort.hpp:80-88
  }
  int mirror_bits = 0;  // id width of the current gather source (32 = block itself)
  auto build_mirror = [&](uint32_t blocks) {
    const int bits = blocks <= 2 ? 1 : blocks <= 16 ? 4 : blocks <= 256 ? 8 : blocks <= 65536 ? 16 : 32;
    mirror_bits = bits;
    if (bits == 32) return;
    ProfScope p(ctx, "mirror", n * 4 + n * bits / 8);
    const unsigned g = grid_for(ctx, ceil_div(n, 32 / bits));
    if (bits == 1) mirror_kernel<1><<<g, 256, 0, ctx.stream>>>(block, n, mirror);
    else if (bits == 4) mirror_kernel<4><<<g, 256, 0, ctx.stream>>>(block, n, mirror);
    else if (bits == 8) mirror_kernel<8><<<g, 256, 0, ctx.stream>>>(block, n, mirror);
    else mirror_kernel<16><<<g, 256, 0, ctx.stream>>>(block, n, mirror);
    DFM_LAUNCH_CHECK();
  };
  if (sgrid) build_mirror(B);  // (else init_kernel wrote the 1-bit mirror of pass 1)
  else mirror_bits = 1;
  // B bounds the ids (key packing, mirror width, fresh ids start there); nb counts the
  // blocks.  They differ after a relabel-in-place pass, whose ids are direct-table
  // slots (the key, not all of which occur)
  uint32_t nb = B;
  const bool rip_on = rip_enabled();
  Layout lay;
  bool lay_built = false;
  bool force_global = false;
  const bool part_on = partition_enabled();
  const bool lay_ok = layout_possible(n, k);
  // Device-resident input whose later passes will want the blocked layout: build it
  // on the side stream while pass 1 (gather-rate bound) runs on the main one.
  bool lay_pending = false;
  cudaEvent_t lay_ready = nullptr;
  struct JoinSide {  // every exit joins the side stream into the main one
    Ctx& ctx;
    bool& pending;
    cudaEvent_t& ev;
    ~JoinSide() {
      if (pending) cudaStreamWaitEvent(ctx.stream, ev, 0);
    }
  } join_side{ctx, lay_pending, lay_ready};
  if (lay_ok && d.nready == 0 && n > kBlockedMinMirror && layout_overlap_enabled()) {
    cudaStream_t main = ctx.stream, side = ctx.copy();
    lay_ready = ctx.chunk_event_pool(1)[0];
    DFM_CUDA(cudaEventRecord(lay_ready, main));
    DFM_CUDA(cudaStreamWaitEvent(side, lay_ready, 0));
    ctx.stream = side;  // the build's kernels, scans and scratch follow ctx.stream
    try {
      build_layout(ctx, d, lay);
    } catch (...) {
      ctx.stream = main;
      throw;
    }
    ctx.stream = main;
    DFM_CUDA(cudaEventRecord(lay_ready, side));
    lay_built = true;
    lay_pending = true;
  }
  const uint32_t* act = nullptr;  // identity at pass 1
  int act_sel = 0;
  uint64_t m = n;
  uint64_t seed = kSeed0;
  sortpr_weak_hash_setup();
  std::vector<uint32_t> trace_buf;
  bool prog_pending = d.nready > 0;  // pipelined upload: rows still landing chunk by chunk

  while (true) {
    if (dl.expired()) {
      out.status = DFM_STATUS_TIMEOUT;
      return out;
    }
    const int w = std::max(1, bit_width_u32(B - 1));
    const uint64_t kbits = (uint64_t)(k + 1) * (uint64_t)w;
    const bool packed = kbits <= 63;
    // direct-indexed table (slot = key, no probing) when the key space is small
    const bool direct = packed && kbits <= 30 && (1ull << kbits) <= std::max<uint64_t>(2 * m, 4096);
    // hash tables: load <= 0.4 (a warp waits for its longest probe chain)
    const uint64_t table = direct ? (1ull << kbits) : std::max<uint64_t>(1024, m * 5 / 2);
    DFM_CUDA(cudaMemsetAsync(sc + 1, 0, 24, ctx.stream));
    DFM_CUDA(cudaMemsetAsync(sc + 8, 0, 8, ctx.stream));
    uint32_t* act_next = act_buf[act_sel ^ 1];
    bool rip = false;        // this pass relabels in place (no resolve / apply)
    uint64_t rip_bound = 0;  // its id bound: the direct table's size
    const Slot* rip_slots = nullptr;
    bool hrip = false;        // filtered pass relabelled in place (ids into res, swapped in)
    bool hrip_pre = false;    // ... with its singletons labelled by the filter itself
    uint64_t hrip_table = 0;  // states that reached its table
    bool act_scanned = false;  // the partitioned path compacts inside the pass
    if (m > 0) {
      if (!packed && sig == nullptr) sig = ctx.slot_t<uint32_t>("sh.sig", n * (uint64_t)row);
      const void* ids = mirror_bits == 32 ? (const void*)block : (const void*)mirror;
      unsigned long long* keys = nullptr;
      uint32_t* present = nullptr;  // rank-compacted direct table (blocked passes)
      if (packed && (mirror_bits == 8 || mirror_bits == 16))
        keys = ctx.slot_t<unsigned long long>("sh.keys", m);
      // blocked signature builder whenever most states are active (it streams all n*k
      // transitions); sparse late passes gather directly
      const bool blocked = lay_ok && m >= n / 4 && n * (uint64_t)mirror_bits / 8 > kBlockedMinMirror;
      if (prog_pending && (blocked || act != nullptr || mirror_bits != 1 || !packed || !direct ||
                           table > kSmallTable)) {
        for (uint32_t c = 0; c < d.nready; ++c) wait_chunk(ctx, d, c);  // not chunkable
        prog_pending = false;
      }
      // partitioned grouping for the large passes (not the tiny direct tables)
      const bool part = blocked && part_on && !force_global && !(direct && table <= kSmallTable) &&
                        m >= kPartMinStates && m < (1ull << 31);
      force_global = false;
      // narrow exact passes (ids <= 8 bits): keys by direct gathers from an L2-resident
      // packed mirror; the blocked layout keeps building on the side stream for the
      // 32-bit passes
      const bool dgather = blocked && !part && packed && direct && table > kSmallTable && w <= 8 &&
                           pass_direct_enabled();
      if (dgather) {
        keys = ctx.slot_t<unsigned long long>("sh.keys", m);
        const uint64_t words = ceil_div(table, 32);
        present = ctx.slot_t<uint32_t>("sh.present", 2 * words);
        DFM_CUDA(cudaMemsetAsync(present, 0, 2 * words * 4, ctx.stream));
        const int FB = w <= 1 ? 1 : w <= 2 ? 2 : w <= 4 ? 4 : w;  // 5, 6, 7 pack 6/5/4 per word
        const uint64_t per = 32 / FB;
        uint32_t* pm = ctx.slot_t<uint32_t>("sh.pmirror", ceil_div(n, per));
        {
          ProfScope p(ctx, "mirror", n * 4 + ceil_div(n, per) * 4);
          const unsigned g = grid_for(ctx, ceil_div(n, per));
          switch (FB) {
            case 1: mirror_packed_kernel<1><<<g, 256, 0, ctx.stream>>>(block, n, pm); break;
            case 2: mirror_packed_kernel<2><<<g, 256, 0, ctx.stream>>>(block, n, pm); break;
            case 4: mirror_packed_kernel<4><<<g, 256, 0, ctx.stream>>>(block, n, pm); break;
            case 5: mirror_packed_kernel<5><<<g, 256, 0, ctx.stream>>>(block, n, pm); break;
            case 6: mirror_packed_kernel<6><<<g, 256, 0, ctx.stream>>>(block, n, pm); break;
            case 7: mirror_packed_kernel<7><<<g, 256, 0, ctx.stream>>>(block, n, pm); break;
            default: mirror_packed_kernel<8><<<g, 256, 0, ctx.stream>>>(block, n, pm); break;
          }
          DFM_LAUNCH_CHECK();
        }
        // delta 4k + k gathers (4 B requests) + own id 4 + act 4 + key 8 per active state
        ProfScope p(ctx, "sig", m * (8ull * k + 4 + (act ? 4 : 0) + 8));
        const unsigned g = grid_for(ctx, m);
#define DFM_DK(FBV)                                                                        \
  if (k == 2)                                                                              \
    direct_keys_kernel<FBV, 2><<<g, 256, 0, ctx.stream>>>(d.delta, n, k, pm, act, m, block, w, \
                                                          keys, present);                  \
  else if (k == 4)                                                                         \
    direct_keys_kernel<FBV, 4><<<g, 256, 0, ctx.stream>>>(d.delta, n, k, pm, act, m, block, w, \
                                                          keys, present);                  \
  else                                                                                     \
    direct_keys_kernel<FBV, 0><<<g, 256, 0, ctx.stream>>>(d.delta, n, k, pm, act, m, block, w, \
                                                          keys, present);
        switch (FB) {
          case 1: DFM_DK(1) break;
          case 2: DFM_DK(2) break;
          case 4: DFM_DK(4) break;
          case 5: DFM_DK(5) break;
          case 6: DFM_DK(6) break;
          case 7: DFM_DK(7) break;
          default: DFM_DK(8) break;
        }
#undef DFM_DK
        DFM_LAUNCH_CHECK();
      } else if (blocked) {
        if (lay_pending) {  // built on the side stream during pass 1
          DFM_CUDA(cudaStreamWaitEvent(ctx.stream, lay_ready, 0));
          lay_pending = false;
        }
        if (!lay_built) {
          build_layout(ctx, d, lay);
          lay_built = true;
        }
        keys = ctx.slot_t<unsigned long long>("sh.keys", m);
        uint32_t* vals = part ? ctx.slot_t<uint32_t>("gp.v", m) : nullptr;
        if (!part && direct && table > kSmallTable) {
          const uint64_t words = ceil_div(table, 32);
          // interleaved {bitmap word, exclusive popcount}: the rank is one 8-byte read
          present = ctx.slot_t<uint32_t>("sh.present", 2 * words);
          DFM_CUDA(cudaMemsetAsync(present, 0, 2 * words * 4, ctx.stream));
        }
        layout_keys(ctx, lay, mirror_bits, ids, act, m, block, w, !packed, seed, keys, sig, row,
                    vals, lead, present);
        if (part) {
          group_partitioned(ctx, m, act, keys, vals, packed ? nullptr : sig, k + 1, row, B, block,
                            flag, lead, sc);
          ProfScope p(ctx, "scan", m * 9ull);
          prims::lookback_flags(ctx, "sc.act", m, ActIn{act, flag}, ActOut{act, act_next}, sc + 3);
          act_scanned = true;
        }
      }
      if (!part) {
      // uniqueness filter in front of large hash tables (keys are precomputed)
      const bool filtered = blocked && !direct && m >= kFilterMinStates;
      uint64_t cap = table;
      const uint32_t* cand = nullptr;  // filtered: the states that reach the table
      uint64_t ncand = 0;
      if (present) {
        // dense slots for the keys present: exclusive popcount over the bitmap words
        const uint64_t words = ceil_div(table, 32);
        ProfScope p(ctx, "insert", words * 8);
        prims::lookback_scan(ctx, "sc.present", words, PresentIn{present},
                             PresentOut{present}, sc + 9);
        DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 9, sc + 9, 8, cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
        cap = std::max<uint64_t>(1, ctx.h_scalars[9]);
      }
      if (filtered) {
        uint32_t* F = ctx.slot_t<uint32_t>("sh.filter", 1ull << (kFilterCellBits - 4));
        uint32_t* cbuf[2] = {ctx.slot_t<uint32_t>("sh.cand0", m), ctx.slot_t<uint32_t>("sh.cand1", m)};
        uint64_t dups = m;
        // a second level on independent hash bits re-tests only the first level's
        // candidates: ~31 % -> ~4 % of the keys reach the table at 1e8 distinct keys
        // relabel-in-place over all states (decided before the filter: the table's
        // capacity is at most max(1024, 5m/2)): the filter labels its singletons
        hrip_pre = rip_on && act == nullptr &&
                   (uint64_t)B + m + std::max<uint64_t>(1024, m * 5 / 2) < (1ull << 32);
        for (int level = 0; level < 2 && dups >= kFilterMinStates; ++level) {
          ProfScope p(ctx, "insert", (1ull << (kFilterCellBits - 2)) + dups * (8ull + 8 + 4));
          DFM_CUDA(cudaMemsetAsync(sc + 6, 0, 8, ctx.stream));
          const uint32_t* cin = level == 0 ? nullptr : cand;
          DFM_CUDA(cudaMemsetAsync(F, 0, 1ull << (kFilterCellBits - 2), ctx.stream));
          filt_set_kernel<<<grid_for(ctx, dups), 256, 0, ctx.stream>>>(keys, dups, !packed, seed,
                                                                       F, level, cin);
          DFM_LAUNCH_CHECK();
          if (filt_fused()) {
            prims::lookback_flags(
                ctx, "sc.cand", dups,
                FiltPred{keys, F, cin, seed, !packed, level == 0 ? 64 - kFilterCellBits : 8},
                FiltOut{cin, cbuf[level], slot_of, hrip_pre ? res : nullptr, lead, flag, B},
                sc + 6);
          } else {
            filt_mark_kernel<<<grid_for(ctx, dups), 256, 0, ctx.stream>>>(
                keys, dups, !packed, seed, F, slot_of, level, cin);
            DFM_LAUNCH_CHECK();
            prims::lookback_flags(ctx, "sc.cand", dups, CandIn{cin, slot_of},
                                 CandOut{cin, cbuf[level]}, sc + 6);
          }
          DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 6, sc + 6, 8, cudaMemcpyDeviceToHost,
                                   ctx.stream));
          ctx.sync();
          dups = ctx.h_scalars[6];
          cand = cbuf[level];
        }
        ncand = dups;
        // load <= 0.4: a warp waits for its longest probe chain of DRAM-latency CASes
        cap = std::max<uint64_t>(1024, dups * 5 / 2);
      }
      // signature rows of this pass: the warp-cooperative writer of the direct hashed
      // insert (runtime k: launch_insert compiles k = 1..4) packs the fields at the
      // mirror width
      const bool row_pack = !blocked && !packed && k > 4;
      const uint32_t pw = row_pack ? packed_row_words(k, mirror_bits) : k + 1;
      const uint32_t prow = row_pack ? (pw > 8 ? (pw + 7) & ~7u : pw) : row;
      Slot* slots = static_cast<Slot*>(ctx.slot("sh.table", cap * sizeof(Slot)));
      DFM_CUDA(cudaMemsetAsync(slots, 0, cap * sizeof(Slot), ctx.stream));
      InsertParams ip{d.delta, n, k, block, ids, act, lead, filtered ? ncand : m, w, seed, cap,
                      slots, slot_of, packed ? nullptr : sig, prow, keys, present,
                      filtered ? cand : nullptr};
      // direct tables whose slot can become the id at once: the tiny smem-aggregated
      // ones (the ids are gathered from a mirror or were gathered by the layout) and
      // the rank-compacted ones (slot = rank of the key: dense ids)
      // States off the active list keep their ids (< B): the new ids then start at B.
      rip = rip_on && packed && direct && !filtered &&
            (present != nullptr || (table <= kSmallTable && (blocked || mirror_bits < 32))) &&
            (act == nullptr || (uint64_t)B + cap < (1ull << 32));
      const uint32_t rip_off = act ? B : 0u;
      rip_bound = rip_off + cap;
      ip.ids_out = rip ? block : nullptr;
      ip.id_off = rip_off;
      hrip = rip_on && filtered && act == nullptr && (uint64_t)B + m + cap < (1ull << 32);
      hrip_pre = hrip_pre && filtered && filt_fused();  // (implies hrip)
      hrip_table = ncand;
      if (blocked) {
        ProfScope p(ctx, "insert", m * (8ull + 4 + 1 + 4 + 16 + 4));
        switch (k) {
          case 2: launch_insert_keys<2>(ctx, ip, !packed, direct, table, filtered); break;
          case 4: launch_insert_keys<4>(ctx, ip, !packed, direct, table, filtered); break;
          default: launch_insert_keys<0>(ctx, ip, !packed, direct, table, filtered); break;
        }
      } else if (prog_pending) {
        // first pass over the pipelined upload: each chunk's keys (tiny direct table)
        // and its share of the layout as soon as its rows land
        const bool lay_early = lay_ok && n > kBlockedMinMirror && !lay_built;
        if (lay_early) {
          layout_init(ctx, d, lay, (uint32_t)(d.chunk_states / layout_window(n, k)));
          lay_built = true;
        }
        for (uint32_t c = 0; c < d.nready; ++c) {
          wait_chunk(ctx, d, c);
          InsertParams ipc = ip;
          ipc.i0 = c * d.chunk_states;
          ipc.m = std::min<uint64_t>(n, ipc.i0 + d.chunk_states);
          {
            ProfScope p(ctx, "sig", (ipc.m - ipc.i0) * (4ull * k + k / 8 + 4 + 1 + 16 + 4));
            launch_insert<1>(ctx, ipc, false, true, table);
          }
          if (lay_early) layout_chunk(ctx, d, lay, c);
        }
        prog_pending = false;
      } else {
        // delta 4k + gathered ids (mirror width) k + own id 4 + lead 1 + active id 4 +
        // slot RMW 16 + slot_of 4 (+ signature row 4*row when hashed) per active state
        ProfScope p(ctx, "sig",
                    m * (4ull * k + (uint64_t)std::max(1, mirror_bits / 8) * k + 4 + 1 +
                         (act ? 4 : 0) + 16 + 4 + (packed ? 0 : 4ull * prow)));
        switch (mirror_bits) {
          case 1: launch_insert<1>(ctx, ip, !packed, direct, table); break;
          case 4: launch_insert<4>(ctx, ip, !packed, direct, table); break;
          case 8: launch_insert<8>(ctx, ip, !packed, direct, table); break;
          case 16: launch_insert<16>(ctx, ip, !packed, direct, table); break;
          default: launch_insert<32>(ctx, ip, !packed, direct, table); break;
        }
      }
      if (hrip) {
        {
          // slot_of 4 + id 4 + flag 1 (+ lead 1 for unique states) + slot 8 for table states
          ProfScope p(ctx, "scan", (hrip_pre ? 0 : m * 10ull) + ncand * 8ull);
          if (hrip_pre) {
            rip_hashed_cand_kernel<<<grid_for(ctx, ncand), 256, 0, ctx.stream>>>(
                ncand, cand, m, slot_of, slots, packed ? nullptr : sig, pw, prow,
                reinterpret_cast<unsigned long long*>(sc + 2), B, res, flag);
          } else {
            rip_hashed_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(
                m, slot_of, slots, packed ? nullptr : sig, pw, prow,
                reinterpret_cast<unsigned long long*>(sc + 2), B, res, lead, flag);
          }
          DFM_LAUNCH_CHECK();
        }
        ProfScope p(ctx, "scan", cap * 8ull);
        rip_groups_kernel<<<grid_for(ctx, cap), 256, 0, ctx.stream>>>(
            slots, cap, nullptr, lead, reinterpret_cast<unsigned long long*>(sc + 1),
            reinterpret_cast<unsigned long long*>(sc + 8));
        DFM_LAUNCH_CHECK();
        rip_bound = (uint64_t)B + m + cap;
      } else if (rip) {
        ProfScope p(ctx, "scan", cap * 8ull);
        rip_groups_kernel<<<grid_for(ctx, cap), 256, 0, ctx.stream>>>(
            slots, cap, act, lead, reinterpret_cast<unsigned long long*>(sc + 1),
            reinterpret_cast<unsigned long long*>(sc + 8));
        DFM_LAUNCH_CHECK();
      } else {
      {
        ProfScope p(ctx, "scan", m * (4ull + 16 + 4 + 4 + 1));  // slot_of, slot, own id, res, st
        resolve_kernel<<<grid_for(ctx, ceil_div(m, kResolveItems)), 256, 0, ctx.stream>>>(
            m,
            ResolveIn{slots, slot_of, packed ? nullptr : sig, pw, prow,
                      reinterpret_cast<unsigned long long*>(sc + 2), act, lead},
            ResolveOut{slots, act, block, res, st, B}, reinterpret_cast<unsigned long long*>(sc + 1),
            reinterpret_cast<unsigned long long*>(sc + 8));
        DFM_LAUNCH_CHECK();
      }
      {
        ProfScope p(ctx, "relabel", m * (1ull + 4 + 4 + 4 + 1 + 1));
        apply_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(m, act, res, st, slot_of, slots,
                                                               block, flag, lead, sc);
        DFM_LAUNCH_CHECK();
      }
      }
      rip_slots = slots;
      }
    }
    DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 1, sc + 1, 64, cudaMemcpyDeviceToHost, ctx.stream));
    if (pass_timing()) {  // DFM_SORTPR_PASS_TIMING=1: host timestamps at each pass end
      ctx.sync();
      const bool lay_done = lay_ready == nullptr || cudaEventQuery(lay_ready) == cudaSuccess;
      fprintf(stderr, "pass %llu done at %.3f ms (m=%llu, layout %s)\n",
              (unsigned long long)out.iterations + 1, dl.elapsed(), (unsigned long long)m,
              lay_done ? "ready" : "pending");
    }
    if (d.nready) DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 40, d.bad, 8, cudaMemcpyDeviceToHost,
                                           ctx.stream));
    ctx.sync();
    if (d.nready && ctx.h_scalars[40]) throw Error(DFM_ERR_INVALID, "transition target out of range");
    if (ctx.h_scalars[2] & kFlagOverflow) {  // partitioned grouping overflowed a bucket:
      force_global = true;                    // redo the pass with the global table
      continue;
    }
    if (ctx.h_scalars[2] != 0) {  // hash collision: redo the pass under a new seed
      seed = seed * kGolden + 0x632BE59BD9B4E019ull;
      continue;
    }
    // regular pass: [1] = fresh ids; relabel-in-place pass: [1] = groups of the active
    // states (the others are singleton blocks)
    const uint32_t nb_next =
        rip    ? (uint32_t)(n - m + ctx.h_scalars[1])
        : hrip ? (uint32_t)(m - hrip_table + ctx.h_scalars[1])  // unique states + groups
               : nb + (uint32_t)ctx.h_scalars[1];
    const uint64_t fresh = nb_next - nb;
    ++out.iterations;
    const uint32_t B_next = (rip || hrip) ? (uint32_t)rip_bound : B + (uint32_t)fresh;
    if (hrip) {
      std::swap(block, res);  // verified: the new ids become the block array
      if (m > hrip_table) ctx.h_scalars[8] = 1;  // unique states leave the active list
    }
    if (trace && trace->on_pass) {
      trace_buf.resize(n);
      DFM_CUDA(cudaMemcpyAsync(trace_buf.data(), block, n * 4, cudaMemcpyDeviceToHost, ctx.stream));
      ctx.sync();
      trace->on_pass(trace->user, out.iterations, trace_buf.data(), (uint32_t)n, nb_next);
    }
    if (fresh == 0) {  // fixpoint, min_sort.hpp:111-117 (a relabelled pass renamed the ids)
      B = B_next;
      break;
    }
    B = B_next;
    nb = nb_next;
    if (rip && m > 0 && ctx.h_scalars[8] != 0) {  // one-member groups: flags for the compaction
      ProfScope p(ctx, "relabel", m * 9ull);
      rip_flag_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(m, act, slot_of, rip_slots, flag);
      DFM_LAUNCH_CHECK();
    }
    if (nb == n && !(trace && trace->on_pass)) {
      // every block a singleton: the next pass splits nothing and is the fixpoint
      // pass the reference counts; no active state is left to run it on
      ++out.iterations;
      ++out.skipped_passes;
      break;
    }
    if (!act_scanned && m > 0 && ctx.h_scalars[8] != 0) {
      // some states became singletons: compact the active list (ascending q)
      ProfScope p(ctx, "scan", m * 9ull);
      prims::lookback_flags(ctx, "sc.act", m, ActIn{act, flag}, ActOut{act, act_next}, sc + 3);
      DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 3, sc + 3, 8, cudaMemcpyDeviceToHost, ctx.stream));
      ctx.sync();
      act_scanned = true;
    }
    if (act_scanned) {
      m = ctx.h_scalars[3];
      act = act_next;
      act_sel ^= 1;
    }
    build_mirror(B);  // id mirror for the next pass's gathers
  }
  out.canon_dev = ctx.slot_t<uint32_t>("canon", n);
  if (nb == n) {  // every block a singleton: first-occurrence labels are the identity
    ProfScope p(ctx, "canon", n * 4);
    iota_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(out.canon_dev, n);
    DFM_LAUNCH_CHECK();
    out.num_blocks = nb;
    out.canon_identity = true;
  } else {
    uint32_t* cob = ctx.slot_t<uint32_t>("sh.cob", std::max<uint64_t>(n, B));
    ProfScope p(ctx, "canon", n * 13ull);
    prims::lookback_flags(ctx, "sc.canon", n, LeadIn{lead}, LeadOut{block, cob}, sc + 5);
    canon_gather_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(block, n, cob, out.canon_dev);
    DFM_LAUNCH_CHECK();
    out.num_blocks = nb;  // one leader per block
  }
  out.status = DFM_STATUS_OK;
  return out;
}

}  // namespace dfm
