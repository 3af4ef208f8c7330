// sortPR — sort-based partition refinement (paper Alg. 4; reference
// min_sort.hpp:72-126), B200 edition.
//
// Per pass the reference sorts ALL n states by (block, signature), marks key
// changes, scans the marks into dense labels and scatters them back.  Here:
//
//  * Only ACTIVE states are processed: states whose block has >= 2 members.
//    A singleton block can never split, so its state keeps its label; the
//    partition sequence (and so the pass count) is exactly the reference's.
//  * Block ids are STABLE: when a block b splits, one sub-block keeps b and the
//    others get fresh ids B, B+1, ... (dense, so ids stay < n).
//  * The key (block[q], block[delta[a][q]] for a < k) is packed exactly into
//    64 bits when (k+1)*bits(B-1) <= 64; otherwise it is a 64-bit hash, and
//    every pair of equal-hash neighbours after the sort is verified on the
//    full signature.  A collision aborts the pass (no state is written) and
//    the pass is redone under a new hash seed: the result is always exact.
//  * Grouping = onesweep radix sort + decoupled-look-back scan of run heads.
//
// Kernels: K1 sig_kernel, K3 radix sort (prims.cu), K4 heads scan /
// keep_kernel / fresh scan / scatter_kernel, active-list compaction scan,
// K5 canonicalize (canon.cu).
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <vector>

#include "prims.cuh"

namespace dfm {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct SigParams {
  const uint32_t* __restrict__ delta;
  uint64_t n;
  uint32_t k;
  const uint32_t* __restrict__ block;
  const uint32_t* __restrict__ act;  // nullptr: identity (all states)
  uint64_t m;
  int w;  // packed field width
  uint64_t seed;
  uint64_t* __restrict__ keys;
  uint32_t* __restrict__ sig;  // (k+1) words per active item, hashed mode only
  const uint32_t* __restrict__ mirror;  // successor ids at kBits < 32 (32/kBits per word)
};

// successor id from the packed mirror (kBits < 32: L2-resident at 1/4/8/16 bits while
// B <= 2/16/256/65536 — 12.5 / 50 / 100 / 200 MB at 1e8 states) or the block array
template <int kBits>
__device__ __forceinline__ uint32_t succ_id(const SigParams& p, uint32_t t) {
  if constexpr (kBits == 32) {
    return p.block[t];
  } else {
    constexpr uint32_t per = 32 / kBits;
    return (p.mirror[t / per] >> ((t % per) * kBits)) & ((1u << kBits) - 1u);
  }
}

template <int kBits>
__global__ void __launch_bounds__(256) rmirror_kernel(const uint32_t* __restrict__ block, uint64_t n,
                                                      uint32_t* __restrict__ out) {
  constexpr int per = 32 / kBits;
  const uint64_t words = (n + per - 1) / per;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < per; ++e) {
      const uint64_t q = w * per + e;
      if (q < n) word |= block[q] << (e * kBits);
    }
    out[w] = word;
  }
}

__global__ void __launch_bounds__(256) riota_kernel(uint32_t* __restrict__ out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride)
    out[q] = (uint32_t)q;
}

// first seed of every run; DFM_SORTPR_WEAK_HASH=<bits> (tests) truncates the hashed
// keys under it so that distinct signatures collide and the void-and-retry path runs
constexpr uint64_t kRadixSeed0 = 0x5EED0001ull;
__device__ unsigned long long g_radix_weak_mask = ~0ull;

// K1: signature gather + key build, one thread per active state.  delta rows
// are read coalesced (active list is ascending in q); block[] is gathered.
template <bool kHashed, int kBits>
__global__ void __launch_bounds__(256) sig_kernel(SigParams p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.m; i += stride) {
    const uint32_t q = p.act ? p.act[i] : (uint32_t)i;
    const uint32_t b = p.block[q];
    if (!kHashed) {
      uint64_t key = b;
      for (uint32_t a = 0; a < p.k; ++a)
        key = (key << p.w) | succ_id<kBits>(p, p.delta[(uint64_t)a * p.n + q]);
      p.keys[i] = key;
    } else {
      uint32_t* row = p.sig + i * (uint64_t)(p.k + 1);
      row[0] = b;
      uint64_t h = mix64(p.seed * kGolden + b);
      for (uint32_t a = 0; a < p.k; ++a) {
        const uint32_t s = succ_id<kBits>(p, p.delta[(uint64_t)a * p.n + q]);
        row[a + 1] = s;
        h = mix64(h + kGolden + s);
      }
      p.keys[i] = p.seed == kRadixSeed0 ? (h & g_radix_weak_mask) : h;
    }
  }
}

// run heads over the sorted keys (+ exact verification of equal-hash neighbours)
struct HeadIn {
  const uint64_t* keys;
  const uint32_t* vals;
  const uint32_t* sig;  // nullptr in packed mode
  uint32_t words;
  unsigned long long* collision;
  __device__ uint32_t operator()(uint64_t j) const {
    if (j == 0) return 1u;
    if (keys[j] != keys[j - 1]) return 1u;
    if (sig != nullptr) {
      // (bit 31 of a value may carry the item's leader flag)
      const uint32_t* a = sig + (uint64_t)(vals[j] & 0x7FFFFFFFu) * words;
      const uint32_t* b = sig + (uint64_t)(vals[j - 1] & 0x7FFFFFFFu) * words;
      for (uint32_t i = 0; i < words; ++i) {
        if (a[i] != b[i]) {
          atomicOr(collision, 1ull);
          break;
        }
      }
    }
    return 0u;
  }
};
struct HeadOut {
  uint32_t* run_of;
  uint32_t* runstart;
  uint64_t m;
  __device__ void operator()(uint64_t j, uint32_t excl, uint32_t v) const {
    const uint32_t run = excl + v - 1;
    run_of[j] = run;
    if (v) runstart[run] = (uint32_t)j;
    if (j + 1 == m) runstart[run + 1] = (uint32_t)m;
  }
};

__device__ __forceinline__ unsigned long long keep_tag(uint32_t epoch, uint32_t j) {
  return ((unsigned long long)epoch << 32) | (0xFFFFFFFFu - j);
}

// one thread per run: the run with the smallest head position in each old
// block keeps the block's id (epoch-tagged atomicMax: no per-pass reset)
__global__ void __launch_bounds__(256) keep_kernel(const uint32_t* __restrict__ runstart,
                                                   const uint32_t* __restrict__ vals,
                                                   const uint32_t* __restrict__ act,
                                                   const uint32_t* __restrict__ block,
                                                   uint32_t* __restrict__ runblock,
                                                   unsigned long long* cells,
                                                   const uint64_t* scalars, uint32_t epoch) {
  if (scalars[2] != 0) return;  // collision: pass is void
  const uint64_t R = scalars[0];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride) {
    const uint32_t j = runstart[r];
    const uint32_t pos = vals[j];
    const uint32_t q = act ? act[pos] : pos;
    const uint32_t b = block[q];
    runblock[r] = b;
    atomicMax(&cells[b], keep_tag(epoch, j));
  }
}

struct FreshIn {
  const uint32_t* runblock;
  const uint32_t* runstart;
  const unsigned long long* cells;
  const uint64_t* scalars;
  uint32_t epoch;
  __device__ uint32_t operator()(uint64_t r) const {
    if (r >= scalars[0] || scalars[2] != 0) return 0u;
    return cells[runblock[r]] != keep_tag(epoch, runstart[r]) ? 1u : 0u;
  }
};
struct FreshOut {
  const uint32_t* runblock;
  uint32_t* newid;
  const uint64_t* scalars;
  uint32_t B;
  __device__ void operator()(uint64_t r, uint32_t excl, uint32_t v) const {
    if (r < scalars[0]) newid[r] = v ? B + excl : runblock[r];
  }
};

__global__ void __launch_bounds__(256) scatter_kernel(uint64_t m, const uint32_t* __restrict__ vals,
                                                      const uint32_t* __restrict__ act,
                                                      const uint32_t* __restrict__ run_of,
                                                      const uint32_t* __restrict__ runstart,
                                                      const uint32_t* __restrict__ newid,
                                                      uint32_t* __restrict__ block,
                                                      uint8_t* __restrict__ flag,
                                                      const uint64_t* scalars) {
  if (scalars[2] != 0) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    const uint32_t r = run_of[j];
    const uint32_t len = runstart[r + 1] - runstart[r];
    const uint32_t pos = vals[j];
    const uint32_t q = act ? act[pos] : pos;
    block[q] = newid[r];
    flag[q] = len >= 2 ? 1 : 0;
  }
}

// Sort-back relabel: instead of scattering each sorted position's new id to its
// state (random 4-byte + 1-byte writes: a DRAM read-modify-write each), pair the
// new id (| run size >= 2 in bit 31) with the active index and radix-sort the pairs
// back into active order — streaming passes — then write block/flag in order.
__global__ void __launch_bounds__(256) unscatter_pairs_kernel(
    uint64_t m, const uint32_t* __restrict__ vals, const uint32_t* __restrict__ run_of,
    const uint32_t* __restrict__ runstart, const uint32_t* __restrict__ newid,
    uint64_t* __restrict__ pkeys, uint32_t* __restrict__ pvals, const uint64_t* scalars) {
  if (scalars[2] != 0) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    const uint32_t r = run_of[j];
    const uint32_t len = runstart[r + 1] - runstart[r];
    pkeys[j] = vals[j];
    pvals[j] = newid[r] | (len >= 2 ? 0x80000000u : 0u);
  }
}
__global__ void __launch_bounds__(256) unscatter_apply_kernel(uint64_t m,
                                                              const uint32_t* __restrict__ pvals,
                                                              const uint32_t* __restrict__ act,
                                                              uint32_t* __restrict__ block,
                                                              uint8_t* __restrict__ flag,
                                                              const uint64_t* scalars) {
  if (scalars[2] != 0) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint32_t v = pvals[i];
    const uint32_t q = act ? act[i] : (uint32_t)i;
    block[q] = v & 0x7FFFFFFFu;
    flag[q] = (uint8_t)(v >> 31);
  }
}

// ---- leader-flag relabel (n < 2^30, >= 2^20 active states).  Every block keeps a
// leader flag on its minimum state (as the hash engine does).  The sort values carry
// it in bit 31, so a run holds its old block's leader iff one of its items has the
// bit: that run keeps the block's id (read from the leader's block entry — one
// gather per old block) and every other run takes a fresh id.  No per-run atomics on
// the old blocks' cells (1e8 singleton runs contending for 3e4 cells took 5.3 ms).
// A fresh run's leader is its head (a stable sort of ascending active states puts
// the minimum state first); a kept run's stays.  The new flags ride the sort back.
__global__ void lead_min_kernel(const uint8_t* __restrict__ acc, uint64_t n,
                                uint32_t* __restrict__ mins) {
  uint32_t la = 0xFFFFFFFFu, lr = 0xFFFFFFFFu;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    if (acc[q]) la = min(la, (uint32_t)q);
    else lr = min(lr, (uint32_t)q);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    la = min(la, __shfl_xor_sync(0xffffffffu, la, o));
    lr = min(lr, __shfl_xor_sync(0xffffffffu, lr, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (la != 0xFFFFFFFFu) atomicMin(&mins[0], la);
    if (lr != 0xFFFFFFFFu) atomicMin(&mins[1], lr);
  }
}
__global__ void lead_init_kernel(uint64_t n, const uint32_t* __restrict__ mins,
                                 uint8_t* __restrict__ lead) {
  const uint32_t a = mins[0], r = mins[1];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride)
    lead[q] = (q == a || q == r) ? 1 : 0;
}
// the sort's input values: active index | leader flag << 31
__global__ void lead_vals_kernel(uint64_t m, const uint32_t* __restrict__ act,
                                 const uint8_t* __restrict__ lead, uint32_t* __restrict__ vals) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
    vals[i] = (uint32_t)i | ((uint32_t)lead[act ? act[i] : (uint32_t)i] << 31);
}
// the run holding an old block's leader keeps the block's id
__global__ void lead_keep_kernel(uint64_t m, const uint32_t* __restrict__ vals,
                                 const uint32_t* __restrict__ act, const uint32_t* __restrict__ run_of,
                                 const uint32_t* __restrict__ block, uint32_t* __restrict__ newid,
                                 uint8_t* __restrict__ kept, const uint64_t* scalars) {
  if (scalars[2] != 0) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    const uint32_t v = vals[j];
    if (!(v >> 31)) continue;
    const uint32_t i = v & 0x7FFFFFFFu;
    const uint32_t r = run_of[j];
    newid[r] = block[act ? act[i] : i];
    kept[r] = 1;
  }
}
struct LeadFreshIn {
  const uint8_t* kept;
  const uint64_t* scalars;
  __device__ uint32_t operator()(uint64_t r) const {
    if (r >= scalars[0] || scalars[2] != 0) return 0u;
    return kept[r] ? 0u : 1u;
  }
};
struct LeadFreshOut {
  uint32_t* newid;
  const uint64_t* scalars;
  uint32_t B;
  __device__ void operator()(uint64_t r, uint32_t excl, uint32_t v) const {
    if (r < scalars[0] && v) newid[r] = B + excl;
  }
};
// pairs (active index, new id | run >= 2 << 31 | new leader << 30) for the sort back
__global__ void __launch_bounds__(256) lead_pairs_kernel(
    uint64_t m, const uint32_t* __restrict__ vals, const uint32_t* __restrict__ run_of,
    const uint32_t* __restrict__ runstart, const uint32_t* __restrict__ newid,
    const uint8_t* __restrict__ kept, uint64_t* __restrict__ pkeys, uint32_t* __restrict__ pvals,
    const uint64_t* scalars) {
  if (scalars[2] != 0) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    const uint32_t v = vals[j];
    const uint32_t r = run_of[j];
    const uint32_t s0 = runstart[r];
    const uint32_t len = runstart[r + 1] - s0;
    const uint32_t nl = kept[r] ? (v >> 31) : ((uint32_t)j == s0 ? 1u : 0u);
    pkeys[j] = v & 0x7FFFFFFFu;
    pvals[j] = newid[r] | (len >= 2 ? 0x80000000u : 0u) | (nl << 30);
  }
}
// The pairs' keys are a permutation of 0..m-1: after a stable sort on bits [11, ..)
// only, window x (positions [2048x, 2048x + 2048)) holds exactly the keys of that
// range, so one CTA per window finishes the order in shared memory and applies the
// values in active order (two digit passes fewer than a full sort at m <= 2^27).
constexpr int kPlaceBits = 11;
__global__ void __launch_bounds__(1024) lead_place_apply_kernel(
    uint64_t m, const uint64_t* __restrict__ pkeys, const uint32_t* __restrict__ pvals,
    const uint32_t* __restrict__ act, uint32_t* __restrict__ block, uint8_t* __restrict__ flag,
    uint8_t* __restrict__ lead, const uint64_t* scalars) {
  __shared__ uint32_t s_v[1u << kPlaceBits];
  if (scalars[2] != 0) return;
  const uint64_t nwin = (m + (1u << kPlaceBits) - 1) >> kPlaceBits;
  for (uint64_t x = blockIdx.x; x < nwin; x += gridDim.x) {
    const uint64_t b = x << kPlaceBits;
    const uint64_t rem = m - b;
    const uint32_t len = rem < (1u << kPlaceBits) ? (uint32_t)rem : (1u << kPlaceBits);
    for (uint32_t t = threadIdx.x; t < len; t += blockDim.x)
      s_v[(uint32_t)(pkeys[b + t] - b)] = pvals[b + t];
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < len; t += blockDim.x) {
      const uint32_t v = s_v[t];
      const uint64_t i = b + t;
      const uint32_t q = act ? act[i] : (uint32_t)i;
      block[q] = v & 0x3FFFFFFFu;
      flag[q] = (uint8_t)(v >> 31);
      lead[q] = (uint8_t)((v >> 30) & 1u);
    }
    __syncthreads();
  }
}

// DFM_RADIX_UNSCATTER=0: the plain scatter (A/B runs)
bool unscatter_enabled() {
  const char* e = getenv("DFM_RADIX_UNSCATTER");
  return !(e && e[0] == '0');
}

struct ActIn {
  const uint32_t* act;
  const uint8_t* flag;
  __device__ uint32_t operator()(uint64_t i) const {
    const uint32_t q = act ? act[i] : (uint32_t)i;
    return flag[q];
  }
};
struct ActOut {
  const uint32_t* act;
  uint32_t* act_next;
  __device__ void operator()(uint64_t i, uint32_t excl, uint32_t v) const {
    if (v) act_next[excl] = act ? act[i] : (uint32_t)i;
  }
};

__global__ void count_accepting_kernel(const uint8_t* __restrict__ acc, uint64_t n,
                                       unsigned long long* out) {
  uint32_t c = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride)
    c += acc[q] != 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

__global__ void init_block_kernel(const uint8_t* __restrict__ acc, uint64_t n, bool split,
                                  uint32_t* __restrict__ block) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride)
    block[q] = (split && acc[q] == 0) ? 1u : 0u;
}

unsigned grid_for(const Ctx& ctx, uint64_t items, int threads = 256) {
  const uint64_t want = ceil_div(std::max<uint64_t>(items, 1), threads);
  return (unsigned)std::min<uint64_t>(want, (uint64_t)ctx.num_sms * 16);
}

int bit_width_u32(uint32_t x) { return x == 0 ? 0 : 32 - __builtin_clz(x); }

}  // namespace

AlgoOut run_sort_pr(Ctx& ctx, const DevDfa& d, const Deadline& dl, const dfm_trace* trace) {
  AlgoOut out;
  const uint64_t n = d.n;
  const uint32_t k = d.k;
  out.peak_memory_estimate = n * (16 + 4ull * k);  // min_sort.hpp:121
  uint32_t* block = ctx.slot_t<uint32_t>("sp.block", n);
  uint8_t* flag = ctx.slot_t<uint8_t>("sp.flag", n);
  uint32_t* act_buf[2] = {ctx.slot_t<uint32_t>("sp.act0", n), ctx.slot_t<uint32_t>("sp.act1", n)};
  uint64_t* keysA = ctx.slot_t<uint64_t>("sp.keysA", n);
  uint64_t* keysB = ctx.slot_t<uint64_t>("sp.keysB", n);
  uint32_t* valsA = ctx.slot_t<uint32_t>("sp.valsA", n);
  uint32_t* valsB = ctx.slot_t<uint32_t>("sp.valsB", n);
  uint32_t* run_of = ctx.slot_t<uint32_t>("sp.runof", n);
  uint32_t* runstart = ctx.slot_t<uint32_t>("sp.runstart", n + 1);
  uint32_t* runblock = ctx.slot_t<uint32_t>("sp.runblock", n);
  uint32_t* newid = ctx.slot_t<uint32_t>("sp.newid", n);
  auto* cells = ctx.slot_t<unsigned long long>("sp.cells", n);
  uint32_t* sig = nullptr;
  uint64_t* sc = ctx.d_scalars;  // [0] runs [1] fresh blocks [2] collision [3] next active [4] acc
  DFM_CUDA(cudaMemsetAsync(cells, 0, n * 8, ctx.stream));
  DFM_CUDA(cudaMemsetAsync(sc, 0, 64 * 8, ctx.stream));

  // init, min_sort.hpp:80-88: two blocks iff both acceptance classes are non-empty
  {
    ProfScope p(ctx, "init");
    count_accepting_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(
        d.acc, n, reinterpret_cast<unsigned long long*>(sc + 4));
    DFM_LAUNCH_CHECK();
  }
  DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars, sc, 64 * 8, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  const uint64_t n_acc = ctx.h_scalars[4];
  const bool split = n_acc > 0 && n_acc < n;
  uint32_t B = split ? 2u : 1u;
  {
    ProfScope p(ctx, "init");
    init_block_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(d.acc, n, split, block);
    DFM_LAUNCH_CHECK();
  }
  // leader flags (the minimum state of each block) for the leader-flag relabel; ids
  // then travel in 30 bits
  const bool lead_ok = n >= (1u << 20) && n < (1ull << 30);
  uint8_t* lead = nullptr;
  uint8_t* kept = nullptr;
  if (lead_ok) {
    lead = ctx.slot_t<uint8_t>("sp.lead", n);
    kept = ctx.slot_t<uint8_t>("sp.kept", n);
    uint32_t* mins = reinterpret_cast<uint32_t*>(sc + 6);
    ProfScope p(ctx, "init", n * 2ull);
    DFM_CUDA(cudaMemsetAsync(mins, 0xFF, 8, ctx.stream));
    lead_min_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(d.acc, n, mins);
    DFM_LAUNCH_CHECK();
    lead_init_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(n, mins, lead);
    DFM_LAUNCH_CHECK();
  }

  const uint32_t* act = nullptr;  // identity: every state active at pass 1
  int act_sel = 0;
  uint64_t m = n;
  uint32_t epoch = 0;
  uint64_t seed = kRadixSeed0;
  {
    sortpr_weak_hash_setup();  // (the blocked builder's keys)
    static unsigned long long mask_set = ~0ull;
    const char* e = getenv("DFM_SORTPR_WEAK_HASH");
    const unsigned long long mask =
        e ? ((1ull << std::min(63ul, strtoul(e, nullptr, 10))) - 1) : ~0ull;
    if (mask != mask_set) {
      DFM_CUDA(cudaMemcpyToSymbol(g_radix_weak_mask, &mask, sizeof(mask)));
      mask_set = mask;
    }
  }
  std::vector<uint32_t> trace_buf;
  struct LayFree {
    void operator()(ShardLayout* s) const { shard_layout_free(s); }
  };
  std::unique_ptr<ShardLayout, LayFree> lay;
  const char* le = getenv("DFM_RADIX_LAYOUT");  // 0: the gather kernel on every pass
  bool lay_enabled = !(le && le[0] == '0');

  while (true) {
    if (dl.expired()) {
      out.status = DFM_STATUS_TIMEOUT;
      return out;
    }
    ++epoch;
    const int w = std::max(1, bit_width_u32(B - 1));
    const bool packed = (uint64_t)(k + 1) * (uint64_t)w <= 64;
    const int bits = packed ? (int)((k + 1) * w) : 64;
    DFM_CUDA(cudaMemsetAsync(sc, 0, 4 * 8, ctx.stream));
    uint32_t* act_next = act_buf[act_sel ^ 1];
    if (m > 0) {
      if (!packed && sig == nullptr) sig = ctx.slot_t<uint32_t>("sp.sig", n * (uint64_t)(k + 1));
      // narrow mirror of the ids for the successor gathers (rebuilt each pass)
      const int mb = B <= 2 ? 1 : B <= 16 ? 4 : B <= 256 ? 8 : B <= 65536 ? 16 : 32;
      uint32_t* mirror = nullptr;
      if (mb < 32) {
        mirror = ctx.slot_t<uint32_t>("sp.mirror", ceil_div(n, 32 / mb));
        ProfScope p(ctx, "mirror", n * 4 + n * mb / 8);
        const unsigned g = grid_for(ctx, ceil_div(n, 32 / mb));
        if (mb == 1) rmirror_kernel<1><<<g, 256, 0, ctx.stream>>>(block, n, mirror);
        else if (mb == 4) rmirror_kernel<4><<<g, 256, 0, ctx.stream>>>(block, n, mirror);
        else if (mb == 8) rmirror_kernel<8><<<g, 256, 0, ctx.stream>>>(block, n, mirror);
        else rmirror_kernel<16><<<g, 256, 0, ctx.stream>>>(block, n, mirror);
        DFM_LAUNCH_CHECK();
      }
      SigParams sp{d.delta, n, k, block, act, m, w, seed, keysA, sig, mirror};
      // ids wider than 4 bits (B > 16) over most states: the blocked builder of
      // the hash engine (no random HBM gathers; built once, delta is pass-invariant)
      if (mb >= 8 && m >= n / 4 && lay_enabled && !lay) {
        lay.reset(radix_layout_build(ctx, d));
        lay_enabled = lay != nullptr;
      }
      if (mb >= 8 && m >= n / 4 && lay) {
        radix_layout_keys(ctx, lay.get(), mb, mb < 32 ? mirror : block, act, m, block, w,
                          !packed, seed, reinterpret_cast<unsigned long long*>(keysA), sig, k + 1);
      } else {
        // delta stream 4k + successor-block gather 4k + own block 4 + active id 4 + key 8
        // (+ signature row 4(k+1) when hashed) per active state
        ProfScope p(ctx, "sig",
                    m * (8ull * k + 4 + (act ? 4 : 0) + 8 + (packed ? 0 : 4ull * (k + 1))));
        const unsigned g = grid_for(ctx, m);
#define DFM_SIG(H)                                                                   \
  switch (mb) {                                                                      \
    case 1: sig_kernel<H, 1><<<g, 256, 0, ctx.stream>>>(sp); break;                  \
    case 4: sig_kernel<H, 4><<<g, 256, 0, ctx.stream>>>(sp); break;                  \
    case 8: sig_kernel<H, 8><<<g, 256, 0, ctx.stream>>>(sp); break;                  \
    case 16: sig_kernel<H, 16><<<g, 256, 0, ctx.stream>>>(sp); break;                \
    default: sig_kernel<H, 32><<<g, 256, 0, ctx.stream>>>(sp); break;                \
  }
        if (packed) {
          DFM_SIG(false)
        } else {
          DFM_SIG(true)
        }
#undef DFM_SIG
        DFM_LAUNCH_CHECK();
      }
      // leader-flag relabel (see lead_keep_kernel) for large active sets
      const bool lead_path = lead_ok && unscatter_enabled() && m >= (1u << 20);
      if (lead_path) {
        ProfScope p(ctx, "relabel", m * 9ull);  // active id 4 + flag 1 + value 4
        lead_vals_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(m, act, lead, valsA);
        DFM_LAUNCH_CHECK();
      }
      const bool alt =
          prims::radix_sort_pairs(ctx, keysA, valsA, keysB, valsB, m, bits, !lead_path);
      const uint64_t* ks = alt ? keysB : keysA;
      const uint32_t* vs = alt ? valsB : valsA;
      {
        ProfScope p(ctx, "scan", m * 16ull);  // key 8 + run_of 4 + runstart 4
        prims::lookback_flags(ctx, "sc.heads", m,
                             HeadIn{ks, vs, packed ? nullptr : sig, k + 1,
                                    reinterpret_cast<unsigned long long*>(sc + 2)},
                             HeadOut{run_of, runstart, m}, sc + 0);
      }
      if (lead_path) {
        // the sorted buffers are dead once the pairs are built: they are the sort's
        // alternates
        uint64_t* pk = alt ? keysA : keysB;
        uint32_t* pv = alt ? valsA : valsB;
        {
          ProfScope p(ctx, "relabel", m * 5ull);  // value 4 + kept flag 1 (+ per old block)
          DFM_CUDA(cudaMemsetAsync(kept, 0, m, ctx.stream));
          lead_keep_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(m, vs, act, run_of, block,
                                                                    newid, kept, sc);
          DFM_LAUNCH_CHECK();
        }
        {
          ProfScope p(ctx, "scan", m * 5ull);  // kept flag 1 + new id 4 per run
          prims::lookback_flags(ctx, "sc.fresh", m, LeadFreshIn{kept, sc},
                               LeadFreshOut{newid, sc, B}, sc + 1);
        }
        {
          // value 4 + run_of 4 + runstart pair 8 + new id 4 + kept 1 + key 8 + value 4
          ProfScope p(ctx, "relabel", m * 33ull);
          lead_pairs_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(m, vs, run_of, runstart, newid,
                                                                     kept, pk, pv, sc);
          DFM_LAUNCH_CHECK();
        }
        // the sort back on the bits above the 2048-key windows, then the windows
        const int hb = bit_width_u32((uint32_t)(m - 1));
        const bool alt2 = prims::radix_sort_pairs_bits(ctx, pk, pv, const_cast<uint64_t*>(ks),
                                                       const_cast<uint32_t*>(vs), m, kPlaceBits,
                                                       hb - kPlaceBits, false);
        // key 8 + value 4 + active id 4 + block 4 + flag 1 + lead 1
        ProfScope p(ctx, "relabel", m * 22ull);
        lead_place_apply_kernel<<<(unsigned)std::min<uint64_t>(
                                      ceil_div(m, 1u << kPlaceBits), (uint64_t)ctx.num_sms * 2),
                                  1024, 0, ctx.stream>>>(m, alt2 ? ks : pk, alt2 ? vs : pv, act,
                                                         block, flag, lead, sc);
        DFM_LAUNCH_CHECK();
      } else {
      {
        ProfScope p(ctx, "relabel");
        keep_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(runstart, vs, act, block, runblock,
                                                              cells, sc, epoch);
        DFM_LAUNCH_CHECK();
      }
      {
        ProfScope p(ctx, "scan");
        prims::lookback_flags(ctx, "sc.fresh", m, FreshIn{runblock, runstart, cells, sc, epoch},
                             FreshOut{runblock, newid, sc, B}, sc + 1);
      }
      if (unscatter_enabled() && n < (1ull << 31) && m >= (1u << 20)) {
        // the sorted buffers are dead once the pairs are built: they are the sort's
        // alternates.  Pairs: run_of 4 + runstart pair 8 + value 4 + new id 4 + key 8 +
        // value 4; the sort back; apply: value 4 + active id 4 + block 4 + flag 1
        uint64_t* pk = alt ? keysA : keysB;
        uint32_t* pv = alt ? valsA : valsB;
        {
          ProfScope p(ctx, "relabel", m * 32ull);
          unscatter_pairs_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(
              m, vs, run_of, runstart, newid, pk, pv, sc);
          DFM_LAUNCH_CHECK();
        }
        const bool alt2 = prims::radix_sort_pairs(ctx, pk, pv, const_cast<uint64_t*>(ks),
                                                  const_cast<uint32_t*>(vs), m,
                                                  bit_width_u32((uint32_t)(m - 1)), false);
        ProfScope p(ctx, "relabel", m * 13ull);
        unscatter_apply_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(
            m, alt2 ? vs : pv, act, block, flag, sc);
        DFM_LAUNCH_CHECK();
      } else {
        // run_of 4 + runstart pair 8 + value 4 + active id 4 + new id 4 + block write 4 + flag 1
        ProfScope p(ctx, "relabel", m * 29ull);
        scatter_kernel<<<grid_for(ctx, m), 256, 0, ctx.stream>>>(m, vs, act, run_of, runstart,
                                                                 newid, block, flag, sc);
        DFM_LAUNCH_CHECK();
      }
      }
      {
        ProfScope p(ctx, "scan", m * 9ull);  // active id 4 + flag 1 + survivor id 4
        prims::lookback_flags(ctx, "sc.act", m, ActIn{act, flag}, ActOut{act, act_next}, sc + 3);
      }
    }
    DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars, sc, 4 * 8, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    if (ctx.h_scalars[2] != 0) {  // hash collision: redo the pass under a new seed
      seed = seed * kGolden + 0x632BE59BD9B4E019ull;
      continue;
    }
    const uint64_t fresh = ctx.h_scalars[1];
    ++out.iterations;
    const uint32_t B_next = B + (uint32_t)fresh;
    if (trace && trace->on_pass) {
      trace_buf.resize(n);
      DFM_CUDA(cudaMemcpyAsync(trace_buf.data(), block, n * 4, cudaMemcpyDeviceToHost, ctx.stream));
      ctx.sync();
      trace->on_pass(trace->user, out.iterations, trace_buf.data(), (uint32_t)n, B_next);
    }
    if (fresh == 0) break;  // fixpoint, min_sort.hpp:111-117
    B = B_next;
    m = ctx.h_scalars[3];
    act = act_next;
    act_sel ^= 1;
  }
  out.canon_dev = ctx.slot_t<uint32_t>("canon", n);
  if (B == n) {  // every block a singleton: the canonical labels are 0..n-1
    ProfScope p(ctx, "canon", n * 4);
    riota_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(out.canon_dev, n);
    DFM_LAUNCH_CHECK();
    out.num_blocks = (uint32_t)n;
  } else {
    out.num_blocks = canonicalize_dev(ctx, block, n, out.canon_dev);
  }
  out.status = DFM_STATUS_OK;
  return out;
}

}  // namespace dfm
