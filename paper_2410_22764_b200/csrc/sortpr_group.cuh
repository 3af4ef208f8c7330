// Partitioned exact grouping for sortPR's large passes (included by
// sortpr_hash.cu inside its anonymous namespace).
//
// The global open-addressing table of the hash engine costs one random HBM
// atomic per active state (measured ~21-25 G/s on B200 once the table exceeds
// L2, tools/l2_bench.cu) plus one random slot read to resolve.  Here the keys
// are grouped with streaming passes and shared memory only:
//   1. P emits H = a BIJECTIVE mix of the exact packed key (mix64 is invertible,
//      so equal H <=> equal key) or the 64-bit signature hash (hashed passes,
//      verified against signature rows), with v = i | lead << 31;
//   2. two onesweep radix passes partition (H, v) by the low 16 bits of H:
//      65,536 buckets of ~m/65,536 items;
//   3. one CTA per bucket groups it in a shared-memory table: group size,
//      minimum member (the new leader) and whether it holds the old leader
//      (keeps the old id); fresh ids come from one atomic per bucket;
//   4. one radix pass by the top 8 bits of i brings the (i, id, flags) records
//      back into L2-sized i windows, and a scatter places them (L2-resident);
//   5. apply in i order.
// A bucket whose distinct keys overflow the table, or that is too large for one
// CTA, voids the pass; it is then redone with the global-table path.
#pragma once

constexpr int kGroupBits = 16;
constexpr uint32_t kGroupTable = 4096;      // shared-memory slots per bucket
constexpr uint32_t kGroupHeavy = 1u << 20;  // larger buckets: global-table path
constexpr uint32_t kKeep = 0xFFFFFFFFu;     // group keeps its old block id
constexpr uint64_t kFlagCollision = 1, kFlagOverflow = 2;

// start of every bucket in the sorted H (bstart[nb] = m)
__global__ void grp_bounds_kernel(const uint64_t* __restrict__ H, uint64_t m, uint32_t nb,
                                  uint32_t* __restrict__ bstart) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= m; p += stride) {
    const int64_t b = p < m ? (int64_t)(H[p] & (nb - 1)) : (int64_t)nb;
    const int64_t bp = p > 0 ? (int64_t)(H[p - 1] & (nb - 1)) : -1;
    for (int64_t x = bp + 1; x <= b; ++x) bstart[x] = (uint32_t)p;
  }
}

struct GSlot {
  unsigned long long key;  // (H >> kGroupBits) | 1 << 63; 0 = empty
  uint32_t rep;            // minimum member i
  uint32_t info;           // member count | holds the old leader << 31
};

struct GroupParams {
  const uint64_t* H;
  const uint32_t* V;
  const uint32_t* bstart;
  uint32_t nb;
  unsigned long long* out_key;  // i << 32 | new id (kKeep: unchanged)
  uint32_t* out_val;            // bit0 stays active, bit1 new leader
  unsigned long long* fresh;    // fresh-id counter
  unsigned long long* flags;    // kFlagCollision | kFlagOverflow
  const uint32_t* sig;          // hashed passes: signature rows, else nullptr
  uint32_t words, row;
  uint32_t B;
};

__device__ __forceinline__ int grp_find(const GSlot* t, uint32_t tsize, unsigned long long stored) {
  uint32_t s = (uint32_t)stored & (tsize - 1);
  for (uint32_t probe = 0; probe < tsize; ++probe) {
    if (t[s].key == stored) return (int)s;
    s = (s + 1) & (tsize - 1);
  }
  return -1;
}

__global__ void __launch_bounds__(512) grp_group_kernel(GroupParams p) {
  extern __shared__ uint4 s_raw[];
  GSlot* s_t = reinterpret_cast<GSlot*>(s_raw);
  uint32_t* s_gid = reinterpret_cast<uint32_t*>(s_t + kGroupTable);
  __shared__ uint32_t s_warp[512 / 32 + 1];
  __shared__ uint32_t s_base;
  for (uint32_t b = blockIdx.x; b < p.nb; b += gridDim.x) {
    const uint32_t start = p.bstart[b], end = p.bstart[b + 1];
    const uint32_t cnt = end - start;
    if (cnt == 0) continue;
    if (cnt > kGroupHeavy) {
      if (threadIdx.x == 0) atomicOr(p.flags, kFlagOverflow);
      continue;
    }
    uint32_t tsize = 64;
    while (tsize < kGroupTable && tsize < cnt + cnt / 4) tsize <<= 1;
    for (uint32_t s = threadIdx.x; s < tsize; s += blockDim.x) {
      s_t[s].key = 0;
      s_t[s].rep = 0xFFFFFFFFu;
      s_t[s].info = 0;
    }
    __syncthreads();
    bool overflow = false;
    for (uint32_t q = start + threadIdx.x; q < end; q += blockDim.x) {
      const uint64_t h = p.H[q];
      const uint32_t v = p.V[q];
      const unsigned long long stored = (h >> kGroupBits) | (1ull << 63);
      uint32_t s = (uint32_t)stored & (tsize - 1);
      bool placed = false;
      for (uint32_t probe = 0; probe < tsize; ++probe) {
        const unsigned long long cur = atomicCAS(&s_t[s].key, 0ull, stored);
        if (cur == 0ull || cur == stored) {
          placed = true;
          break;
        }
        s = (s + 1) & (tsize - 1);
      }
      if (!placed) {
        overflow = true;
        continue;
      }
      atomicMin(&s_t[s].rep, v & 0x7FFFFFFFu);
      atomicAdd(&s_t[s].info, 1u | (v & 0x80000000u));
    }
    if (__syncthreads_or(overflow)) {
      if (threadIdx.x == 0) atomicOr(p.flags, kFlagOverflow);
      continue;
    }
    // fresh ids for the groups without the old leader: one global atomic per bucket
    uint32_t mine = 0;
    for (uint32_t s = threadIdx.x; s < tsize; s += blockDim.x)
      mine += (s_t[s].key != 0 && (s_t[s].info >> 31) == 0) ? 1u : 0u;
    uint32_t total;
    uint32_t run = prims::block_exclusive_sum<512>(mine, s_warp, &total);
    if (threadIdx.x == 0) s_base = total ? (uint32_t)atomicAdd(p.fresh, (unsigned long long)total) : 0u;
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < tsize; s += blockDim.x)
      if (s_t[s].key != 0 && (s_t[s].info >> 31) == 0) s_gid[s] = p.B + s_base + run++;
    __syncthreads();
    bool collision = false;
    for (uint32_t q = start + threadIdx.x; q < end; q += blockDim.x) {
      const uint64_t h = p.H[q];
      const uint32_t i = p.V[q] & 0x7FFFFFFFu;
      const int s = grp_find(s_t, tsize, (h >> kGroupBits) | (1ull << 63));
      const uint32_t rep = s_t[s].rep, info = s_t[s].info;
      const bool keeper = (info >> 31) != 0, is_rep = rep == i;
      if (p.sig != nullptr && !is_rep) {  // equal hash: verify the whole signature
        const uint32_t* ra = p.sig + (uint64_t)i * p.row;
        const uint32_t* rb = p.sig + (uint64_t)rep * p.row;
        for (uint32_t x = 0; x < p.words; ++x)
          if (ra[x] != rb[x]) {
            collision = true;
            break;
          }
      }
      p.out_key[q] = ((unsigned long long)i << 32) | (keeper ? kKeep : s_gid[s]);
      p.out_val[q] = ((info & 0x7FFFFFFFu) >= 2 ? 1u : 0u) | ((is_rep && !keeper) ? 2u : 0u);
    }
    if (__syncthreads_or(collision) && threadIdx.x == 0) atomicOr(p.flags, kFlagCollision);
  }
}

// records sorted into L2-sized i windows -> res[i] = id | flags << 32
__global__ void __launch_bounds__(256) grp_place_kernel(const unsigned long long* __restrict__ key,
                                                        const uint32_t* __restrict__ val, uint64_t m,
                                                        unsigned long long* __restrict__ res) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += stride) {
    const unsigned long long k = key[q];
    res[k >> 32] = (k & 0xFFFFFFFFull) | ((unsigned long long)val[q] << 32);
  }
}

__global__ void __launch_bounds__(256) grp_apply_kernel(uint64_t m, const uint32_t* __restrict__ act,
                                                        const unsigned long long* __restrict__ res,
                                                        uint32_t* __restrict__ block,
                                                        uint8_t* __restrict__ flag,
                                                        uint8_t* __restrict__ lead,
                                                        const unsigned long long* flags) {
  if (*flags != 0) return;  // collision / overflow: the pass is void
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const unsigned long long r = res[i];
    const uint32_t q = act ? act[i] : (uint32_t)i;
    const uint32_t gid = (uint32_t)r, fl = (uint32_t)(r >> 32);
    if (gid != kKeep) block[q] = gid;
    flag[q] = fl & 1u;
    if (fl & 2u) lead[q] = 1;
  }
}
