// Device primitives of the state-sharded sortPR.
// One process per GPU; the collectives (all-gather of block ids, the key
// exchange, count all-gathers) are issued by the host driver
// (paper_2410_22764_b200/sharded.py) through torch.distributed/NCCL.  Here:
//   shard_signature : per owned state, the full signature row (block[q], block[δa(q)])
//                     read from the all-gathered block vector, its 64-bit hash and
//                     the destination rank that groups that key
//   shard_group     : exact grouping of the (key, signature) pairs a rank received:
//                     dense local group ids; equal-hash members are verified
//                     against the group's first member (collision flag otherwise)
//   sort_pairs      : the onesweep radix sort (routing by destination rank)
//   random slice    : bit-exact random_dfa rows for an owned state range
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "prims.cuh"

namespace dfm {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
// DFM_SHARD_WEAK_HASH=<bits> (tests): hashed keys of passes under the first seed are
// truncated so that distinct signatures collide and the void-and-retry path runs
constexpr uint64_t kShardSeed0 = 0x5EED0001ull;
__device__ unsigned long long g_shard_weak_mask = ~0ull;
__device__ __forceinline__ unsigned long long shard_weak(unsigned long long h, uint64_t seed) {
  return seed == kShardSeed0 ? (h & g_shard_weak_mask) : h;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ids of the all-gathered block vector at kBits per state (1/2/4/8/16/32, packed
// 32/kBits per word, little-endian: 8/16 bits are plain byte / short arrays)
template <int kBits>
__device__ __forceinline__ uint32_t full_id(const uint32_t* __restrict__ full, uint64_t t) {
  if constexpr (kBits == 32) {
    return full[t];
  } else {
    constexpr uint32_t per = 32 / kBits;
    return (full[t / per] >> ((uint32_t)(t % per) * kBits)) & ((1u << kBits) - 1u);
  }
}

// Exact packed keys while (k+1) * bits(B-1) <= 63 (the early passes): no signature
// rows to route or verify; ids are read from the all-gathered block vector at its
// narrow width (1/2/4/8/16/32 bits: the early passes' vectors stay L2-resident)
template <int kBits>
__global__ void __launch_bounds__(256) shard_packed_kernel(
    const uint32_t* __restrict__ delta, uint64_t n_local, uint32_t k, const uint32_t* __restrict__ full,
    uint64_t lo, uint32_t w, uint32_t ranks, unsigned long long* __restrict__ keys,
    uint32_t* __restrict__ dest) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_local; i += stride) {
    unsigned long long key = full_id<kBits>(full, lo + i);
    for (uint32_t a = 0; a < k; ++a)
      key = (key << w) | full_id<kBits>(full, delta[(uint64_t)a * n_local + i]);
    keys[i] = key + 1ull;  // never 0: 0 marks an empty table slot
    dest[i] = (uint32_t)__umul64hi(mix64(key ^ 0xD1B54A32D192ED03ull), ranks);
  }
}

template <int kBits>
__global__ void __launch_bounds__(256) shard_sig_kernel_w(
    const uint32_t* __restrict__ delta, uint64_t n_local, uint32_t k,
    const uint32_t* __restrict__ full, uint64_t lo, uint64_t seed, uint32_t ranks,
    unsigned long long* __restrict__ keys, uint32_t* __restrict__ sig,
    uint32_t* __restrict__ dest) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_local; i += stride) {
    const uint32_t b = full_id<kBits>(full, lo + i);
    uint32_t* row = sig + i * (uint64_t)(k + 1);
    row[0] = b;
    unsigned long long h = mix64(seed * kGolden + b);
    for (uint32_t a = 0; a < k; ++a) {
      const uint32_t s = full_id<kBits>(full, delta[(uint64_t)a * n_local + i]);
      row[a + 1] = s;
      h = mix64(h + kGolden + s);
    }
    h = shard_weak(h, seed);
    keys[i] = h | 1ull;
    dest[i] = (uint32_t)__umul64hi(mix64(h ^ 0xD1B54A32D192ED03ull), ranks);
  }
}

__global__ void __launch_bounds__(256) shard_sig_kernel(
    const uint32_t* __restrict__ delta, uint64_t n_local, uint32_t k,
    const uint32_t* __restrict__ block_full, uint64_t lo, uint64_t seed, uint32_t ranks,
    unsigned long long* __restrict__ keys, uint32_t* __restrict__ sig,
    uint32_t* __restrict__ dest) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_local; i += stride) {
    const uint32_t b = block_full[lo + i];
    uint32_t* row = sig + i * (uint64_t)(k + 1);
    row[0] = b;
    unsigned long long h = mix64(seed * kGolden + b);
    for (uint32_t a = 0; a < k; ++a) {
      const uint32_t s = block_full[delta[(uint64_t)a * n_local + i]];
      row[a + 1] = s;
      h = mix64(h + kGolden + s);
    }
    keys[i] = h | 1ull;  // never 0: 0 marks an empty table slot
    dest[i] = (uint32_t)__umul64hi(mix64(h ^ 0xD1B54A32D192ED03ull), ranks);
  }
}

struct GSlot {
  unsigned long long key;
  uint32_t rep;  // ~(first member) via atomicMax
  uint32_t gid;
};

// Grouping of the received keys (64-bit signature hashes, never 0) — the hash
// engine's recipe (sortpr_hash.cu): a two-level uniqueness filter ("seen" and "seen
// twice" bitmaps of 2^28 cells, 64 MB, L2-resident) lets keys alone in their cell skip the table;
// the rest goes through an open-addressing table at load <= 0.4; group ids come
// from one atomic per CTA step (no global scan).
constexpr uint32_t kUniq = 0xFFFFFFFFu;
constexpr int kCellBits = 28;
constexpr uint64_t kFilterMin = 1ull << 22;

__device__ __forceinline__ uint64_t cell_of(unsigned long long key, int level) {
  return (key >> (level == 0 ? 64 - kCellBits : 8)) & ((1ull << kCellBits) - 1);
}

// L2 policies as in the single-GPU engine's filter: keys stream with evict_first, the
// 64 MB filter is kept with evict_last, the second bit is a fire-and-forget reduction
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long ld_key(const unsigned long long* a, uint64_t pol) {
  unsigned long long v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}

// Fused mark + compaction (prims::lookback_flags, as the single-GPU engine's filter):
// a key alone in its cell is a group of its own and is labelled on the spot — the
// u-th singleton of the level takes base + u (u = position - candidates before it) —
// and the others leave as the next level's list, in ascending order.  The table then
// sees the last list only, and so do the label and member kernels.
struct GFiltPred {
  const unsigned long long* keys;
  const uint32_t* F;
  const uint32_t* cand;  // nullptr: all items
  int level;
  __device__ bool operator()(uint64_t j) const {
    const uint64_t i = cand ? cand[j] : j;
    const uint64_t c = cell_of(ld_key(keys + i, pol_first()), level);
    return (F[(1ull << (kCellBits - 5)) + (c >> 5)] >> (uint32_t)(c & 31)) & 1u;
  }
};
struct GFiltOut {
  const uint32_t* cand;
  uint32_t* out;
  uint32_t* label;
  uint32_t base;
  __device__ void operator()(uint64_t j, uint32_t rank, uint32_t dup) const {
    const uint32_t i = cand ? cand[j] : (uint32_t)j;
    if (dup) out[rank] = i;
    else label[i] = base + (uint32_t)j - rank;
  }
};

__global__ void __launch_bounds__(256) gfilt_set_list_kernel(
    const unsigned long long* __restrict__ keys, uint64_t count, uint32_t* F, int level,
    const uint32_t* __restrict__ cand) {
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
    const uint64_t i = cand ? cand[j] : j;
    // "seen" bitmap (first 2^28 bits) and "seen twice" bitmap (next 2^28 bits)
    const uint64_t c = cell_of(ld_key(keys + i, pf), level);
    const uint32_t bit = 1u << (uint32_t)(c & 31);
    uint32_t old;
    asm volatile("atom.global.or.L2::cache_hint.b32 %0, [%1], %2, %3;"
                 : "=r"(old) : "l"(&F[c >> 5]), "r"(bit), "l"(pl) : "memory");
    if (old & bit)
      asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(
                       &F[(1ull << (kCellBits - 5)) + (c >> 5)]),
                   "r"(bit), "l"(pl) : "memory");
  }
}

// Insert with CTA-level pre-aggregation: a tile's keys first meet in a shared-memory
// table, and each distinct key of the tile costs one global CAS + one atomicMax —
// early passes have a handful of keys over 1e8 items, and per-item atomics on the
// same few slots would serialise.  Keys that do not fit the tile table go straight
// to the global table.
constexpr int kTileItems = 2048;
constexpr int kTileTable = 2048;

__device__ __forceinline__ uint64_t global_insert(GSlot* slots, uint64_t cap,
                                                  unsigned long long key) {
  uint64_t t = __umul64hi(mix64(key), cap);
  while (true) {
    const unsigned long long cur = atomicCAS(&slots[t].key, 0ull, key);
    if (cur == 0ull || cur == key) return t;
    if (++t == cap) t = 0;
  }
}

__global__ void __launch_bounds__(256) group_insert_kernel(const unsigned long long* __restrict__ keys,
                                                           uint64_t count, GSlot* slots,
                                                           uint64_t cap, uint32_t* __restrict__ slot_of) {
  __shared__ unsigned long long s_key[kTileTable];
  __shared__ uint32_t s_min[kTileTable];
  __shared__ uint32_t s_gslot[kTileTable];
  constexpr int kPer = kTileItems / 256;
  for (uint64_t base = (uint64_t)blockIdx.x * kTileItems; base < count;
       base += (uint64_t)gridDim.x * kTileItems) {
    for (int t = threadIdx.x; t < kTileTable; t += blockDim.x) {
      s_key[t] = 0;
      s_min[t] = 0xFFFFFFFFu;
    }
    __syncthreads();
    int ent[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint64_t i = base + u * 256 + threadIdx.x;
      ent[u] = -2;  // -2: nothing to do, -1: global path, >= 0: tile entry
      if (i >= count || slot_of[i] == kUniq) continue;
      const unsigned long long key = keys[i];
      uint32_t t = (uint32_t)mix64(key) & (kTileTable - 1);
      ent[u] = -1;
      for (int probe = 0; probe < 16; ++probe) {
        const unsigned long long cur = atomicCAS(&s_key[t], 0ull, key);
        if (cur == 0ull || cur == key) {
          ent[u] = (int)t;
          atomicMin(&s_min[t], (uint32_t)i);
          break;
        }
        t = (t + 1) & (kTileTable - 1);
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kTileTable; t += blockDim.x)
      if (s_key[t] != 0ull) {
        const uint64_t g = global_insert(slots, cap, s_key[t]);
        atomicMax(&slots[g].rep, ~s_min[t]);
        s_gslot[t] = (uint32_t)g;
      }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint64_t i = base + u * 256 + threadIdx.x;
      if (ent[u] >= 0) {
        slot_of[i] = s_gslot[ent[u]];
      } else if (ent[u] == -1) {
        const uint64_t g = global_insert(slots, cap, keys[i]);
        atomicMax(&slots[g].rep, ~(uint32_t)i);
        slot_of[i] = (uint32_t)g;
      }
    }
    __syncthreads();
  }
}

// the filtered list's states: table insert, then label / members as below
__global__ void __launch_bounds__(256) group_insert_list_kernel(
    const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ list, uint64_t nl,
    GSlot* slots, uint64_t cap, uint32_t* __restrict__ slot_of) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nl; j += stride) {
    const uint32_t i = list[j];
    const uint64_t g = global_insert(slots, cap, keys[i]);
    atomicMax(&slots[g].rep, ~i);
    slot_of[i] = (uint32_t)g;
  }
}

// a member is the representative of its group if it is alone (filter) or the table's
// minimum; representatives take an id from one atomic per CTA step
__global__ void __launch_bounds__(256) group_label_kernel(uint64_t count, GSlot* slots,
                                                          const uint32_t* __restrict__ list,
                                                          const uint32_t* __restrict__ slot_of,
                                                          const uint32_t* __restrict__ sig,
                                                          uint32_t words, uint32_t* __restrict__ label,
                                                          unsigned long long* groups,
                                                          unsigned long long* collision) {
  __shared__ uint32_t s_cnt[8];
  __shared__ uint32_t s_first;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < count; base += stride) {
    const uint64_t j = base + threadIdx.x;
    const uint64_t i = j < count ? (list ? list[j] : j) : 0;
    bool rep = false;
    uint32_t s = kUniq;
    if (j < count) {
      s = slot_of[i];
      if (s == kUniq) {
        rep = true;
      } else {
        const uint32_t r = ~slots[s].rep;
        rep = r == (uint32_t)i;
        if (!rep && words > 0) {  // equal hash: verify the whole signature vs the representative
          const uint32_t* a = sig + i * (uint64_t)words;
          const uint32_t* b = sig + (uint64_t)r * words;
          for (uint32_t x = 0; x < words; ++x)
            if (a[x] != b[x]) {
              atomicOr(collision, 1ull);
              break;
            }
        }
      }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, rep);
    if (lane == 0) s_cnt[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int g = 0; g < 8; ++g) t += s_cnt[g];
      s_first = t ? (uint32_t)atomicAdd(groups, (unsigned long long)t) : 0u;
    }
    __syncthreads();
    uint32_t off = s_first;
    for (uint32_t g = 0; g < warp; ++g) off += s_cnt[g];
    if (rep) {
      const uint32_t gid = off + __popc(m & ((1u << lane) - 1u));
      label[i] = gid;
      if (s != kUniq) slots[s].gid = gid;
    }
    __syncthreads();
  }
}

__global__ void group_members_kernel(uint64_t count, const GSlot* __restrict__ slots,
                                     const uint32_t* __restrict__ list,
                                     const uint32_t* __restrict__ slot_of,
                                     uint32_t* __restrict__ label) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
    const uint32_t i = list ? list[j] : (uint32_t)j;
    const uint32_t s = slot_of[i];
    if (s == kUniq) continue;
    if (~slots[s].rep != (uint32_t)i) label[i] = slots[s].gid;
  }
}

__global__ void random_slice_kernel(uint32_t* __restrict__ delta, uint8_t* __restrict__ acc,
                                    uint64_t n_total, uint32_t k, uint64_t lo, uint64_t count,
                                    uint64_t seed, double p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    for (uint32_t a = 0; a <= k; ++a) {
      // draw j of SplitMix64(seed): row a, state q -> j = a*n + q; acceptance -> k*n + q
      uint64_t z = seed + ((uint64_t)a * n_total + lo + i + 1) * kGolden;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      if (a < k) delta[(uint64_t)a * count + i] = (uint32_t)(z % n_total);
      else acc[i] = ((double)(z >> 11) * 0x1.0p-53) < p ? 1 : 0;
    }
  }
}

// Direct grouping of exact packed keys from a small key space (2^bits keys): a
// presence bitmap (L2-resident) and the key's rank among the present keys as its
// dense group id — one atomic per warp-distinct key, no table, no probing.
// bitmap words interleaved with their exclusive popcounts: word w of the bitmap at
// [2w], its prefix at [2w+1] — a key's rank is one 8-byte read
__global__ void __launch_bounds__(256) direct_set_kernel(const unsigned long long* __restrict__ keys,
                                                         uint64_t count, uint32_t* bp) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint64_t key = keys[i] - 1;  // packed keys are stored + 1
    const uint32_t m = 1u << (key & 31);
    uint32_t* w = bp + 2 * (key >> 5);
    // test before set: most keys of a dense pass repeat
    if ((prims::ld_hint_u32(w) & m) == 0) atomicOr(w, m);
  }
}

// small key spaces (<= 2^16 keys: the early passes, a handful of keys over all
// items): each CTA ORs its keys into a shared bitmap, then one global OR per word
__global__ void __launch_bounds__(256) direct_set_small_kernel(
    const unsigned long long* __restrict__ keys, uint64_t count, uint32_t* bp, uint32_t words) {
  extern __shared__ uint32_t s_bits[];
  for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) s_bits[w] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint64_t key = keys[i] - 1;
    const uint32_t m = 1u << (key & 31);
    if ((s_bits[key >> 5] & m) == 0) atomicOr(&s_bits[key >> 5], m);
  }
  __syncthreads();
  for (uint32_t w = threadIdx.x; w < words; w += blockDim.x)
    if (s_bits[w]) atomicOr(&bp[2 * w], s_bits[w]);
}

struct DirPopIn {
  const uint32_t* bp;
  __device__ uint32_t operator()(uint64_t w) const { return __popc(bp[2 * w]); }
};
struct DirPopOut {
  uint32_t* bp;
  __device__ void operator()(uint64_t w, uint32_t excl, uint32_t) const { bp[2 * w + 1] = excl; }
};

__global__ void __launch_bounds__(256) direct_label_kernel(const unsigned long long* __restrict__ keys,
                                                           uint64_t count,
                                                           const uint32_t* __restrict__ bp,
                                                           uint32_t* __restrict__ label) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint64_t key = keys[i] - 1;
    const uint2 wp = *reinterpret_cast<const uint2*>(bp + 2 * (key >> 5));
    label[i] = wp.y + __popc(wp.x & ((1u << (key & 31)) - 1u));
  }
}

unsigned grid_for(const Ctx& ctx, uint64_t items) {
  return (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(items, 1), 256),
                                      (uint64_t)ctx.num_sms * 16);
}

}  // namespace
}  // namespace dfm


namespace dfm {
void shard_weak_hash_setup() {
  static unsigned long long set = ~0ull;
  const char* e = getenv("DFM_SHARD_WEAK_HASH");
  const unsigned long long mask =
      e ? ((1ull << std::min(63ul, strtoul(e, nullptr, 10))) - 1) : ~0ull;
  if (mask != set) {
    DFM_CUDA(cudaMemcpyToSymbol(g_shard_weak_mask, &mask, sizeof(mask)));
    set = mask;
  }
}

void shard_signature(Ctx& ctx, const void* delta_local, uint64_t n_local, uint32_t k,
                     const void* block_full, uint32_t id_bits, uint64_t lo, uint64_t seed,
                     uint32_t ranks, uint32_t pack_bits, void* keys_out, void* sig_out,
                     void* dest_out) {
  shard_weak_hash_setup();
  if (ranks == 0) throw Error(DFM_ERR_INVALID, "ranks must be >= 1");
  if (id_bits != 1 && id_bits != 2 && id_bits != 4 && id_bits != 8 && id_bits != 16 && id_bits != 32)
    throw Error(DFM_ERR_INVALID, "id_bits must be 1, 2, 4, 8, 16 or 32");
  if (pack_bits && (uint64_t)(k + 1) * pack_bits > 63)
    throw Error(DFM_ERR_INVALID, "packed key does not fit 63 bits");
  if (n_local == 0) return;
  const auto* d = static_cast<const uint32_t*>(delta_local);
  const auto* full = static_cast<const uint32_t*>(block_full);
  auto* keys = static_cast<unsigned long long*>(keys_out);
  auto* dest = static_cast<uint32_t*>(dest_out);
  auto* sig = static_cast<uint32_t*>(sig_out);
  const unsigned g = grid_for(ctx, n_local);
  // delta 4k + k+1 id gathers (4-byte requests) + key 8 + dest 4 (+ row when hashed)
  ProfScope p(ctx, "sig", n_local * (8ull * k + 4 + 8 + 4 + (pack_bits ? 0 : 4ull * (k + 1))));
#define DFM_SHARD_KEYS(B)                                                                    \
  if (pack_bits)                                                                             \
    shard_packed_kernel<B><<<g, 256, 0, ctx.stream>>>(d, n_local, k, full, lo, pack_bits, ranks, \
                                                      keys, dest);                           \
  else                                                                                       \
    shard_sig_kernel_w<B><<<g, 256, 0, ctx.stream>>>(d, n_local, k, full, lo, seed, ranks, keys, \
                                                     sig, dest);
  switch (id_bits) {
    case 1: DFM_SHARD_KEYS(1) break;
    case 2: DFM_SHARD_KEYS(2) break;
    case 4: DFM_SHARD_KEYS(4) break;
    case 8: DFM_SHARD_KEYS(8) break;
    case 16: DFM_SHARD_KEYS(16) break;
    default: DFM_SHARD_KEYS(32) break;
  }
#undef DFM_SHARD_KEYS
  DFM_LAUNCH_CHECK();
}

void shard_group_direct(Ctx& ctx, const void* keys, uint64_t count, uint32_t key_bits,
                        void* label_out, uint64_t* groups_out) {
  if (count >= (1ull << 32)) throw Error(DFM_ERR_INVALID, "too many items for one rank");
  if (key_bits > 32) throw Error(DFM_ERR_INVALID, "direct grouping needs <= 32 key bits");
  const uint64_t words = ceil_div(1ull << key_bits, 32);
  uint32_t* bp = ctx.slot_t<uint32_t>("shard.dbits", 2 * words);  // {bitmap, prefix} pairs
  uint64_t* total = ctx.d_scalars + 48;
  ProfScope p(ctx, "group", count * 16ull + words * 12);
  DFM_CUDA(cudaMemsetAsync(bp, 0, 2 * words * 4, ctx.stream));
  const auto* k = static_cast<const unsigned long long*>(keys);
  if (count && words <= 2048) {
    direct_set_small_kernel<<<grid_for(ctx, count), 256, words * 4, ctx.stream>>>(
        k, count, bp, (uint32_t)words);
    DFM_LAUNCH_CHECK();
  } else if (count) {
    direct_set_kernel<<<grid_for(ctx, count), 256, 0, ctx.stream>>>(k, count, bp);
    DFM_LAUNCH_CHECK();
  }
  prims::lookback_scan(ctx, "shard.dscan", words, DirPopIn{bp}, DirPopOut{bp}, total);
  if (count) {
    direct_label_kernel<<<grid_for(ctx, count), 256, 0, ctx.stream>>>(
        k, count, bp, static_cast<uint32_t*>(label_out));
    DFM_LAUNCH_CHECK();
  }
  DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 48, total, 8, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  if (groups_out) *groups_out = ctx.h_scalars[48];
}

void shard_group(Ctx& ctx, const void* keys, const void* sig, uint32_t words, uint64_t count,
                 void* label_out, uint64_t* groups_out, int* collision_out) {
    if (count >= (1ull << 32)) throw Error(DFM_ERR_INVALID, "too many items for one rank");
    uint64_t* sc = ctx.d_scalars + 48;  // [0] groups [1] collision [2] filter duplicates
    DFM_CUDA(cudaMemsetAsync(sc, 0, 24, ctx.stream));
    if (count > 0) {
      uint32_t* slot_of = ctx.slot_t<uint32_t>("shard.slotof", count);
      uint64_t dups = count;
      ProfScope p(ctx, "group", count * (8ull + 16 + 4 + 4 + 4 + 4ull * words));
      // the filter pays off for hashed keys (late, mostly-distinct passes); exact packed
      // keys belong to the early passes, where a few keys repeat over all items.  Above
      // one key per cell (2^28) nearly every key shares its cell: straight to the table
      if (count >= kFilterMin && count <= (1ull << kCellBits) && words > 0) {
        // filtered: singletons labelled by the fused mark, the table sees the last list
        uint32_t* F = ctx.slot_t<uint32_t>("shard.filter", 1ull << (kCellBits - 4));
        uint32_t* lbuf[2] = {ctx.slot_t<uint32_t>("shard.cand0", count),
                             ctx.slot_t<uint32_t>("shard.cand1", count)};
        uint32_t* label = static_cast<uint32_t*>(label_out);
        const uint32_t* list = nullptr;
        uint64_t nl = count, singles = 0;
        for (int level = 0; level < 2 && nl >= kFilterMin; ++level) {
          DFM_CUDA(cudaMemsetAsync(F, 0, 1ull << (kCellBits - 2), ctx.stream));
          gfilt_set_list_kernel<<<grid_for(ctx, nl), 256, 0, ctx.stream>>>(
              static_cast<const unsigned long long*>(keys), nl, F, level, list);
          DFM_LAUNCH_CHECK();
          prims::lookback_flags(
              ctx, "shard.fscan", nl,
              GFiltPred{static_cast<const unsigned long long*>(keys), F, list, level},
              GFiltOut{list, lbuf[level], label, (uint32_t)singles}, sc + 2);
          DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 50, sc + 2, 8, cudaMemcpyDeviceToHost,
                                   ctx.stream));
          ctx.sync();
          const uint64_t d = ctx.h_scalars[50];
          singles += nl - d;
          nl = d;
          list = lbuf[level];
        }
        const uint64_t cap = std::max<uint64_t>(1024, nl * 5 / 2);  // load <= 0.4
        auto* slots = static_cast<GSlot*>(ctx.slot("shard.table", cap * sizeof(GSlot)));
        DFM_CUDA(cudaMemsetAsync(slots, 0, cap * sizeof(GSlot), ctx.stream));
        // table groups are numbered after the singletons
        ctx.h_scalars[51] = singles;
        DFM_CUDA(cudaMemcpyAsync(sc, ctx.h_scalars + 51, 8, cudaMemcpyHostToDevice, ctx.stream));
        if (nl) {
          group_insert_list_kernel<<<grid_for(ctx, nl), 256, 0, ctx.stream>>>(
              static_cast<const unsigned long long*>(keys), list, nl, slots, cap, slot_of);
          DFM_LAUNCH_CHECK();
          group_label_kernel<<<grid_for(ctx, nl), 256, 0, ctx.stream>>>(
              nl, slots, list, slot_of, static_cast<const uint32_t*>(sig), words, label,
              reinterpret_cast<unsigned long long*>(sc),
              reinterpret_cast<unsigned long long*>(sc + 1));
          DFM_LAUNCH_CHECK();
          group_members_kernel<<<grid_for(ctx, nl), 256, 0, ctx.stream>>>(nl, slots, list,
                                                                            slot_of, label);
          DFM_LAUNCH_CHECK();
        }
      } else {
        DFM_CUDA(cudaMemsetAsync(slot_of, 0, count * 4, ctx.stream));
        const uint64_t cap = std::max<uint64_t>(1024, dups * 5 / 2);  // load <= 0.4
        auto* slots = static_cast<GSlot*>(ctx.slot("shard.table", cap * sizeof(GSlot)));
        DFM_CUDA(cudaMemsetAsync(slots, 0, cap * sizeof(GSlot), ctx.stream));
        group_insert_kernel<<<(unsigned)std::min<uint64_t>(ceil_div(count, kTileItems),
                                                           ctx.num_sms * 8ull),
                              256, 0, ctx.stream>>>(
            static_cast<const unsigned long long*>(keys), count, slots, cap, slot_of);
        DFM_LAUNCH_CHECK();
        group_label_kernel<<<grid_for(ctx, count), 256, 0, ctx.stream>>>(
            count, slots, nullptr, slot_of, static_cast<const uint32_t*>(sig), words,
            static_cast<uint32_t*>(label_out), reinterpret_cast<unsigned long long*>(sc),
            reinterpret_cast<unsigned long long*>(sc + 1));
        DFM_LAUNCH_CHECK();
        group_members_kernel<<<grid_for(ctx, count), 256, 0, ctx.stream>>>(
            count, slots, nullptr, slot_of, static_cast<uint32_t*>(label_out));
        DFM_LAUNCH_CHECK();
      }
    }
    DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 48, sc, 16, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    if (groups_out) *groups_out = ctx.h_scalars[48];
    if (collision_out) *collision_out = ctx.h_scalars[49] != 0;
  }
}  // namespace dfm

using namespace dfm;

namespace {
template <class F>
int guarded_shard(dfm_ctx* c, F&& f) {
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
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
  } catch (const std::exception& e) {
    ctx->last_error = e.what();
    return DFM_ERR_INVALID;
  }
}
}  // namespace

extern "C" {

int dfm_shard_signature(dfm_ctx* c, const void* delta_local, uint64_t n_local, uint32_t k,
                        const void* block_full, uint64_t lo, uint64_t seed, uint32_t ranks,
                        void* keys_out, void* sig_out, void* dest_out) {
  return guarded_shard(c, [&](Ctx& ctx) {
    if (ranks == 0) throw Error(DFM_ERR_INVALID, "ranks must be >= 1");
    if (n_local == 0) return;
    ProfScope p(ctx, "sig", n_local * (4ull * k + 4ull * k + 4 + 8 + 4ull * (k + 1) + 4));
    shard_sig_kernel<<<grid_for(ctx, n_local), 256, 0, ctx.stream>>>(
        static_cast<const uint32_t*>(delta_local), n_local, k,
        static_cast<const uint32_t*>(block_full), lo, seed, ranks,
        static_cast<unsigned long long*>(keys_out), static_cast<uint32_t*>(sig_out),
        static_cast<uint32_t*>(dest_out));
    DFM_LAUNCH_CHECK();
  });
}

int dfm_shard_signature_ex(dfm_ctx* c, const void* delta_local, uint64_t n_local, uint32_t k,
                           const void* block_full, uint32_t id_bytes, uint64_t lo, uint64_t seed,
                           uint32_t ranks, uint32_t pack_bits, void* keys_out, void* sig_out,
                           void* dest_out) {
  return guarded_shard(c, [&](Ctx& ctx) {
    if (id_bytes != 1 && id_bytes != 2 && id_bytes != 4)
      throw Error(DFM_ERR_INVALID, "id_bytes must be 1, 2 or 4");
    shard_signature(ctx, delta_local, n_local, k, block_full, 8 * id_bytes, lo, seed, ranks,
                    pack_bits, keys_out, sig_out, dest_out);
  });
}

int dfm_shard_group(dfm_ctx* c, const void* keys, const void* sig, uint32_t words, uint64_t count,
                    void* label_out, uint64_t* groups_out, int* collision_out) {
  return guarded_shard(c, [&](Ctx& ctx) {
    shard_group(ctx, keys, sig, words, count, label_out, groups_out, collision_out);
  });
}

int dfm_sort_pairs(dfm_ctx* c, void* keys, void* values, uint64_t count, uint32_t bits) {
  return guarded_shard(c, [&](Ctx& ctx) {
    if (count == 0) return;
    auto* k2 = ctx.slot_t<uint64_t>("sp2.keys", count);
    auto* v2 = ctx.slot_t<uint32_t>("sp2.vals", count);
    const bool alt = prims::radix_sort_pairs(ctx, static_cast<uint64_t*>(keys),
                                             static_cast<uint32_t*>(values), k2, v2, count,
                                             (int)std::max(1u, bits), false);
    if (alt) {
      DFM_CUDA(cudaMemcpyAsync(keys, k2, count * 8, cudaMemcpyDeviceToDevice, ctx.stream));
      DFM_CUDA(cudaMemcpyAsync(values, v2, count * 4, cudaMemcpyDeviceToDevice, ctx.stream));
    }
    ctx.sync();
  });
}

int dfm_canonicalize_dev(dfm_ctx* c, const void* raw_dev, uint64_t n, void* out_dev,
                         uint32_t* num_blocks_out) {
  return guarded_shard(c, [&](Ctx& ctx) {
    const uint32_t nb = canonicalize_dev(ctx, static_cast<const uint32_t*>(raw_dev), n,
                                         static_cast<uint32_t*>(out_dev));
    if (num_blocks_out) *num_blocks_out = nb;
  });
}

int dfm_random_dfa_slice_dev(dfm_ctx* c, uint64_t n_total, uint32_t k, uint64_t seed,
                             double accept_prob, uint64_t lo, uint64_t count, void* delta_out,
                             void* accepting_out) {
  return guarded_shard(c, [&](Ctx& ctx) {
    if (n_total < 1 || n_total > 0xFFFFFFFFull || lo + count > n_total)
      throw Error(DFM_ERR_INVALID, "bad random_dfa slice");
    if (count == 0) return;
    random_slice_kernel<<<grid_for(ctx, count), 256, 0, ctx.stream>>>(
        static_cast<uint32_t*>(delta_out), static_cast<uint8_t*>(accepting_out), n_total, k, lo,
        count, seed, accept_prob);
    DFM_LAUNCH_CHECK();
    ctx.sync();
  });
}

}  // extern "C"
