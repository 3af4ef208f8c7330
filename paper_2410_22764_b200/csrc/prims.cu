// Host side of the device-wide primitives (see prims.cuh).
#include "prims.cuh"

#include <algorithm>
#include <utility>

namespace dfm {
namespace prims {

// per-pass digit histograms of all passes in one read of the keys
__global__ void __launch_bounds__(256) radix_histogram_kernel(const uint64_t* __restrict__ keys,
                                                              uint64_t count, int passes,
                                                              uint32_t* __restrict__ hist,
                                                              int lo_bit) {
  __shared__ uint32_t sh[8 * 256];
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint64_t k = keys[i] >> lo_bit;
    for (int p = 0; p < passes; ++p) atomicAdd(&sh[p * 256 + ((k >> (8 * p)) & 255)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void radix_bucket_scan_kernel(const uint32_t* __restrict__ hist,
                                         uint32_t* __restrict__ base) {
  __shared__ uint32_t s_warp[9];
  const uint32_t x = hist[blockIdx.x * 256 + threadIdx.x];
  uint32_t total;
  const uint32_t e = block_exclusive_sum<256>(x, s_warp, &total);
  base[blockIdx.x * 256 + threadIdx.x] = e;
}

#ifndef DFM_RS_BALLOT_RANK  // digit peers from 9 ballots (1) or match.any (0): sort 28.4 -> 26.7 ms
#define DFM_RS_BALLOT_RANK 1
#endif
// per-(tile, digit) look-back words: 64-bit, or 32-bit (flags in bits 31:30) while the
// item count stays below 2^30 — half the status traffic and memset
template <class S>
struct LbStatus;
template <>
struct LbStatus<uint64_t> {
  static constexpr uint64_t kAgg = kFlagAgg, kInc = kFlagInc, kVal = kValMask;
  __device__ static uint64_t ld(const uint64_t* p) { return ld_volatile(p); }
  __device__ static void st(uint64_t* p, uint64_t v) { st_volatile(p, v); }
};
template <>
struct LbStatus<uint32_t> {
  static constexpr uint32_t kAgg = 1u << 30, kInc = 2u << 30, kVal = (1u << 30) - 1;
  __device__ static uint32_t ld(const uint32_t* p) { return ld_relaxed_u32(p); }
  __device__ static void st(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  }
};

template <bool kIdentVals, class S>
__global__ void __launch_bounds__(kRsThreads, kRsBlocksPerSm) onesweep_kernel(
    const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t count, int shift,
    const uint32_t* __restrict__ bucket_base, S* status, uint32_t* ticket) {
  using St = LbStatus<S>;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(smem);
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + kRsTile);
  uint32_t* s_cnt = s_vals + kRsTile;         // [warp][digit]
  uint32_t* s_start = s_cnt + kRsWarps * 256;  // tile-local digit start
  uint32_t* s_glob = s_start + 256;            // global destination base per digit
  uint32_t* s_misc = s_glob + 256;             // [0] tile id, [1..kRsWarps+1] warp sums
  uint32_t* s_hist = s_misc + 32;              // tile digit histogram (published early)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_misc[0] = atomicAdd(ticket, 1u);
  for (int i = tid; i < kRsWarps * 256; i += kRsThreads) s_cnt[i] = 0;
  if (tid < 256) s_hist[tid] = 0;
  __syncthreads();
  const uint32_t tile = s_misc[0];
  const uint64_t tile_base = (uint64_t)tile * kRsTile;
  const uint64_t warp_base = tile_base + (uint64_t)warp * 32 * kRsItems;

  uint64_t k[kRsItems];
  uint32_t v[kRsItems];
  uint32_t rank[kRsItems];
  uint32_t dig[kRsItems];
#pragma unroll
  for (int j = 0; j < kRsItems; ++j) {
    const uint64_t idx = warp_base + (uint64_t)j * 32 + lane;
    const bool valid = idx < count;
    k[j] = valid ? keys_in[idx] : 0ull;
    if (kIdentVals) v[j] = (uint32_t)idx;
    else v[j] = valid ? vals_in[idx] : 0u;
    dig[j] = valid ? (uint32_t)((k[j] >> shift) & 255) : 256u;
  }
  // the tile's digit counts go out before the ranking, so successors' look-backs
  // rarely wait on this tile
#pragma unroll
  for (int j = 0; j < kRsItems; ++j)
    if (dig[j] < 256) atomicAdd(&s_hist[dig[j]], 1u);
  __syncthreads();
  if (tid < 256) {
    if (tile == 0) St::st(status + tid, St::kInc | (S)s_hist[tid]);
    else St::st(status + (uint64_t)tile * 256 + tid, St::kAgg | (S)s_hist[tid]);
  }
  uint32_t* my_cnt = s_cnt + warp * 256;
#pragma unroll
  for (int j = 0; j < kRsItems; ++j) {
    const uint32_t d = dig[j];
#if DFM_RS_BALLOT_RANK
    // lanes holding the same 9-bit value (digit, or 256 = no item): one ballot per bit
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 9; ++b) {
      const uint32_t m = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? m : ~m;
    }
#else
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
#endif
    const uint32_t lt = __popc(peers & lanemask_lt());
    uint32_t base = 0;
    if (d < 256) base = my_cnt[d];
    rank[j] = base + lt;
    __syncwarp();
    if (d < 256 && lt == 0) my_cnt[d] = base + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix across warps (stability: warp chunks are in order)
  uint32_t total = 0;
  if (tid < 256) {
    const int d = tid;  // one digit per thread of the first 256
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const uint32_t c = s_cnt[w * 256 + d];
      s_cnt[w * 256 + d] = run;
      run += c;
    }
    total = run;
  }
  uint32_t tile_total;
  const uint32_t start = block_exclusive_sum<kRsThreads>(total, s_misc + 1, &tile_total);
  if (tid < 256) s_start[tid] = start;
  // decoupled look-back, one digit per thread
  if (tid < 256) {
    const int d = tid;
    uint64_t prefix = 0;
    if (tile > 0) {
      // kLb predecessors per step: their loads are in flight together (a walk over
      // tiles that published only aggregates costs one L2 round trip per kLb tiles)
      constexpr int kLb = 4;
      int64_t t = (int64_t)tile - 1;
      bool done = false;
      while (!done) {
        S s[kLb];
#pragma unroll
        for (int u = 0; u < kLb; ++u)
          s[u] = t - u >= 0 ? St::ld(status + (uint64_t)(t - u) * 256 + d) : St::kInc;
#pragma unroll
        for (int u = 0; u < kLb; ++u) {
          if (done) break;
          while ((s[u] & ~St::kVal) == 0) s[u] = St::ld(status + (uint64_t)(t - u) * 256 + d);
          prefix += s[u] & St::kVal;
          done = (s[u] & St::kInc) != 0;
        }
        t -= kLb;
      }
      St::st(status + (uint64_t)tile * 256 + d, St::kInc | (S)(prefix + total));
    }
    s_glob[d] = bucket_base[d] + (uint32_t)prefix;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRsItems; ++j) {
    const uint32_t d = dig[j];
    if (d < 256) {
      const uint32_t pos = s_start[d] + my_cnt[d] + rank[j];
      s_keys[pos] = k[j];
      s_vals[pos] = v[j];
    }
  }
  __syncthreads();
  const uint64_t left = count - tile_base;
  const uint32_t valid = left < (uint64_t)kRsTile ? (uint32_t)left : (uint32_t)kRsTile;
  for (uint32_t p = tid; p < valid; p += kRsThreads) {
    const uint64_t key = s_keys[p];
    const uint32_t d = (uint32_t)((key >> shift) & 255);
    const uint32_t o = s_glob[d] + (p - s_start[d]);
    keys_out[o] = key;
    vals_out[o] = s_vals[p];
  }
}


bool radix_sort_pairs(Ctx& ctx, uint64_t* keys, uint32_t* vals, uint64_t* alt_keys,
                      uint32_t* alt_vals, uint64_t count, int bits, bool ident_vals) {
  return radix_sort_pairs_bits(ctx, keys, vals, alt_keys, alt_vals, count, 0, bits, ident_vals);
}

bool radix_sort_pairs_bits(Ctx& ctx, uint64_t* keys, uint32_t* vals, uint64_t* alt_keys,
                           uint32_t* alt_vals, uint64_t count, int lo_bit, int bits,
                           bool ident_vals) {
  if (count == 0) return false;
  if (bits <= 0) bits = 1;  // identity values still need one materialising pass
  if (count >= (1ull << 32)) throw Error(DFM_ERR_INVALID, "radix_sort_pairs: count >= 2^32");
  int dev = 0;
  DFM_CUDA(cudaGetDevice(&dev));
  per_device_memo((const void*)onesweep_kernel<true, uint64_t>, dev, [](const void*) {
    DFM_CUDA(cudaFuncSetAttribute(onesweep_kernel<true, uint64_t>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kRsSmem));
    DFM_CUDA(cudaFuncSetAttribute(onesweep_kernel<false, uint64_t>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kRsSmem));
    DFM_CUDA(cudaFuncSetAttribute(onesweep_kernel<true, uint32_t>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kRsSmem));
    DFM_CUDA(cudaFuncSetAttribute(onesweep_kernel<false, uint32_t>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kRsSmem));
    return 1;
  });
  const int passes = (bits + 7) / 8;
  const uint64_t tiles = ceil_div(count, kRsTile);
  uint32_t* hist = ctx.slot_t<uint32_t>("rs.hist", 2 * 8 * 256 + 16);
  uint32_t* base = hist + 8 * 256;
  uint32_t* tickets = base + 8 * 256;
  const bool narrow = count < (1ull << 30);  // 32-bit look-back words
  const size_t sbytes = tiles * 256 * (narrow ? 4 : 8);
  void* status = ctx.slot("rs.status", sbytes);
  DFM_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (2 * 8 * 256 + 16), ctx.stream));
  {
    ProfScope p(ctx, "sort", count * 8ull);  // one read of the keys for all digit histograms
    const unsigned grid =
        (unsigned)std::min<uint64_t>((uint64_t)ctx.num_sms * 8, ceil_div(count, 256));
    radix_histogram_kernel<<<grid, 256, 0, ctx.stream>>>(keys, count, passes, hist, lo_bit);
    DFM_LAUNCH_CHECK();
    radix_bucket_scan_kernel<<<passes, 256, 0, ctx.stream>>>(hist, base);
    DFM_LAUNCH_CHECK();
  }
  uint64_t* kin = keys;
  uint32_t* vin = vals;
  uint64_t* kout = alt_keys;
  uint32_t* vout = alt_vals;
  for (int p = 0; p < passes; ++p) {
    DFM_CUDA(cudaMemsetAsync(status, 0, sbytes, ctx.stream));
    {
      ProfScope ps(ctx, "sort", count * 24ull);  // (key 8 + value 4) read + written
      const bool iv = p == 0 && ident_vals;
      const int sh = lo_bit + 8 * p;
      if (narrow) {
        auto* st = static_cast<uint32_t*>(status);
        if (iv)
          onesweep_kernel<true, uint32_t><<<(unsigned)tiles, kRsThreads, kRsSmem, ctx.stream>>>(
              kin, nullptr, kout, vout, (uint32_t)count, sh, base + p * 256, st, tickets + p);
        else
          onesweep_kernel<false, uint32_t><<<(unsigned)tiles, kRsThreads, kRsSmem, ctx.stream>>>(
              kin, vin, kout, vout, (uint32_t)count, sh, base + p * 256, st, tickets + p);
      } else {
        auto* st = static_cast<uint64_t*>(status);
        if (iv)
          onesweep_kernel<true, uint64_t><<<(unsigned)tiles, kRsThreads, kRsSmem, ctx.stream>>>(
              kin, nullptr, kout, vout, (uint32_t)count, sh, base + p * 256, st, tickets + p);
        else
          onesweep_kernel<false, uint64_t><<<(unsigned)tiles, kRsThreads, kRsSmem, ctx.stream>>>(
              kin, vin, kout, vout, (uint32_t)count, sh, base + p * 256, st, tickets + p);
      }
      DFM_LAUNCH_CHECK();
    }
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  const bool in_alt = (passes & 1) != 0;
  return in_alt;
}

}  // namespace prims
}  // namespace dfm
