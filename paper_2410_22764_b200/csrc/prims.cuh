// Device-wide primitives used by every minimizer (the B200 replacement of the
// reference substrate, substrate.hpp:124-197):
//   * lookback_scan  — single-pass prefix scan with decoupled look-back
//                      (adjacent_diff + inclusive_scan, substrate.hpp:156-197)
//   * radix_sort     — onesweep LSD radix sort of (u64 key, u32 value) pairs,
//                      stable, 8-bit digits (par_sort, substrate.hpp:124-153)
// Tiles are claimed through an atomic ticket so the look-back never waits on
// a tile that has not been scheduled (forward progress under any residency).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "dfm_internal.cuh"

namespace dfm {
namespace prims {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// look-back status words are single 64-bit words read and written whole: relaxed
// GPU-scope accesses suffice (ld/st.volatile lower to system-scope STRONG.SYS
// accesses, which the look-back spins on)
__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// test-before-set hint: a weak load at L2 (.cg); a stale 0 only costs a redundant
// atomicOr
__device__ __forceinline__ uint32_t ld_hint_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// a flag written by other CTAs before a grid barrier (or polled): GPU scope
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// look-back status word: [63:62] flag, [61:0] value (value + flag in one
// single-copy-atomic 64-bit word, so no fences are needed around it)
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_sum(uint32_t x, uint32_t* s_warp,
                                                        uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < NT / 32 ? s_warp[lane] : 0;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < NT / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == NT / 32 - 1) s_warp[NT / 32] = wi;
  }
  __syncthreads();
  const uint32_t r = s_warp[warp] + incl - x;
  *total = s_warp[NT / 32];
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ scan
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// in(i) -> u32 value, or a payload struct with a u32 member `v` that is carried
// from in() to out(); out(i, exclusive_prefix, item).  Sums must fit in 32 bits.
__device__ __forceinline__ uint32_t scan_value(uint32_t x) { return x; }
template <class T>
__device__ __forceinline__ uint32_t scan_value(const T& x) {
  return x.v;
}

template <class In, class Out>
__global__ void __launch_bounds__(kScanThreads) lookback_scan_kernel(In in, Out out, uint64_t count,
                                                                     uint64_t* status,
                                                                     uint32_t* ticket,
                                                                     uint64_t* total_out) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[kScanThreads / 32 + 1];
  __shared__ uint64_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  using Item = decltype(in(uint64_t{0}));
  Item v[kScanItems];
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + i;
    v[i] = idx < count ? in(idx) : Item{};
    sum += scan_value(v[i]);
  }
  uint32_t agg;
  const uint32_t excl = block_exclusive_sum<kScanThreads>(sum, s_warp, &agg);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint64_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) st_volatile(status, kFlagInc | agg);
    } else {
      if (lane == 0) st_volatile(status + tile, kFlagAgg | agg);
      int64_t pos = (int64_t)tile - 1 - lane;
      while (true) {
        uint64_t s = 0;
        if (pos >= 0) {
          do {
            s = ld_volatile(status + pos);
          } while ((s & ~kValMask) == 0);
        } else {
          s = kFlagInc;  // virtual inclusive zero before tile 0
        }
        const uint32_t inc_mask = __ballot_sync(0xffffffffu, (s & kFlagInc) != 0);
        const int stop = inc_mask ? __ffs(inc_mask) - 1 : 31;
        uint64_t val = (lane <= stop) ? (s & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        if (inc_mask) break;
        pos -= 32;
      }
      if (lane == 0) st_volatile(status + tile, kFlagInc | (prefix + agg));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint32_t run = (uint32_t)s_prefix + excl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + i;
    if (idx < count) out(idx, run, v[i]);
    run += scan_value(v[i]);
  }
  if (total_out != nullptr && threadIdx.x == 0 && (tile + 1) * kScanTile >= count)
    *total_out = s_prefix + agg;
}

// Launch: exclusive scan over [0,count); total written to *total_dev (device).
template <class In, class Out>
void lookback_scan(Ctx& ctx, const char* slot, uint64_t count, In in, Out out,
                   uint64_t* total_dev) {
  if (count == 0) {
    if (total_dev) DFM_CUDA(cudaMemsetAsync(total_dev, 0, 8, ctx.stream));
    return;
  }
  const uint64_t tiles = ceil_div(count, kScanTile);
  uint8_t* scratch = ctx.slot_t<uint8_t>(slot, 16 + tiles * 8);
  uint32_t* ticket = reinterpret_cast<uint32_t*>(scratch);
  uint64_t* status = reinterpret_cast<uint64_t*>(scratch + 16);
  DFM_CUDA(cudaMemsetAsync(scratch, 0, 16 + tiles * 8, ctx.stream));
  lookback_scan_kernel<In, Out><<<(unsigned)tiles, kScanThreads, 0, ctx.stream>>>(
      in, out, count, status, ticket, total_dev);
  DFM_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ flag compaction
// Ordered compaction of 0/1 flags with decoupled look-back: pred(i) -> bool is
// evaluated STRIPED (item u of thread t is tile_base + u*256 + t: every load is
// warp-coalesced) and ranked with ballots; out(i, rank, flag) gets the number of set
// flags before i, so the flagged i leave in ascending order.
template <class Pred, class Out>
__global__ void __launch_bounds__(kScanThreads) lookback_flags_kernel(Pred pred, Out out,
                                                                      uint64_t count,
                                                                      uint64_t* status,
                                                                      uint32_t* ticket,
                                                                      uint64_t* total_out) {
  constexpr int kWarps = kScanThreads / 32;
  static_assert(kScanItems * kWarps == 64, "two (item, warp) counts per lane");
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_cnt[kScanItems * kWarps];
  __shared__ uint32_t s_agg;
  __shared__ uint64_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t tb = tile * kScanTile;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint32_t bal[kScanItems];
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    const uint64_t idx = tb + (uint64_t)u * kScanThreads + threadIdx.x;
    bal[u] = __ballot_sync(0xffffffffu, idx < count && pred(idx));
  }
  if (lane == 0) {
#pragma unroll
    for (int u = 0; u < kScanItems; ++u) s_cnt[u * kWarps + warp] = __popc(bal[u]);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 64 (item, warp) counts, slot-major
    const uint32_t a = s_cnt[2 * lane], b = s_cnt[2 * lane + 1];
    uint32_t incl = a + b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t ex = incl - a - b;
    s_cnt[2 * lane] = ex;
    s_cnt[2 * lane + 1] = ex + a;
    if (lane == 31) s_agg = incl;
  }
  __syncthreads();
  const uint32_t agg = s_agg;
  if (warp == 0) {
    uint64_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) st_volatile(status, kFlagInc | agg);
    } else {
      if (lane == 0) st_volatile(status + tile, kFlagAgg | agg);
      int64_t pos = (int64_t)tile - 1 - lane;
      while (true) {
        uint64_t s = 0;
        if (pos >= 0) {
          do {
            s = ld_volatile(status + pos);
          } while ((s & ~kValMask) == 0);
        } else {
          s = kFlagInc;
        }
        const uint32_t inc_mask = __ballot_sync(0xffffffffu, (s & kFlagInc) != 0);
        const int stop = inc_mask ? __ffs(inc_mask) - 1 : 31;
        uint64_t val = ((int)lane <= stop) ? (s & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        if (inc_mask) break;
        pos -= 32;
      }
      if (lane == 0) st_volatile(status + tile, kFlagInc | (prefix + agg));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    const uint64_t idx = tb + (uint64_t)u * kScanThreads + threadIdx.x;
    if (idx < count)
      out(idx, (uint32_t)s_prefix + s_cnt[u * kWarps + warp] + __popc(bal[u] & lt),
          (bal[u] >> lane) & 1u);
  }
  if (total_out != nullptr && threadIdx.x == 0 && (tile + 1) * kScanTile >= count)
    *total_out = s_prefix + agg;
}

template <class Pred, class Out>
void lookback_flags(Ctx& ctx, const char* slot, uint64_t count, Pred pred, Out out,
                    uint64_t* total_dev) {
  if (count == 0) {
    if (total_dev) DFM_CUDA(cudaMemsetAsync(total_dev, 0, 8, ctx.stream));
    return;
  }
  const uint64_t tiles = ceil_div(count, kScanTile);
  uint8_t* scratch = ctx.slot_t<uint8_t>(slot, 16 + tiles * 8);
  uint32_t* ticket = reinterpret_cast<uint32_t*>(scratch);
  uint64_t* status = reinterpret_cast<uint64_t*>(scratch + 16);
  DFM_CUDA(cudaMemsetAsync(scratch, 0, 16 + tiles * 8, ctx.stream));
  lookback_flags_kernel<Pred, Out><<<(unsigned)tiles, kScanThreads, 0, ctx.stream>>>(
      pred, out, count, status, ticket, total_dev);
  DFM_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ radix sort
constexpr int kRsThreads = 256;   // >= 256: the first 256 threads own one digit each
constexpr int kRsBlocksPerSm = 4;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsItems = 8;
constexpr int kRsTile = kRsThreads * kRsItems;  // 4096
constexpr int kRsSmem = kRsTile * 8 + kRsTile * 4 + kRsWarps * 256 * 4 + 256 * 4 * 2 + 128 + 1024;
static_assert(kRsWarps + 2 <= 32, "s_misc holds the tile id and the warp sums");

// Sorts (keys, vals) of length count on the low `bits` bits.  ident_vals: the
// input values are 0..count-1 and `vals` is not read.  Uses alt_keys/alt_vals
// as ping-pong buffers; returns which buffer set holds the result (false:
// keys/vals, true: alt_*).  count < 2^32.
bool radix_sort_pairs(Ctx& ctx, uint64_t* keys, uint32_t* vals, uint64_t* alt_keys,
                      uint32_t* alt_vals, uint64_t count, int bits, bool ident_vals);
// Same on bits [lo_bit, lo_bit + bits) of the keys (digit passes from lo_bit up):
// a stable partition by that bit field.
bool radix_sort_pairs_bits(Ctx& ctx, uint64_t* keys, uint32_t* vals, uint64_t* alt_keys,
                           uint32_t* alt_vals, uint64_t count, int lo_bit, int bits,
                           bool ident_vals);

}  // namespace prims
}  // namespace dfm
