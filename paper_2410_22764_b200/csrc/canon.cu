// K5 canonicalize (reference core.hpp:123-136): relabel raw block ids (< n)
// so that labels are 0..B-1 in order of first occurrence — equivalently, the
// canonical label of a block is the rank of its minimum state index among all
// blocks' minimum indices.  Three passes: atomicMin of the min index per raw
// label, a look-back scan over "q is its block's minimum", and a gather.
// Also: device-side bit-exact random_dfa (generators.hpp:130-145).
#include "prims.cuh"

namespace dfm {
namespace {

__global__ void __launch_bounds__(256) min_index_kernel(const uint32_t* __restrict__ raw,
                                                        uint64_t n, uint32_t* minidx) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    const uint32_t b = raw[q];
    // lanes are in ascending q: only the lowest lane of each label group competes,
    // and a plain read filters labels whose minimum is already smaller
    const uint32_t peers = __match_any_sync(__activemask(), b);
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1) && minidx[b] > (uint32_t)q)
      atomicMin(&minidx[b], (uint32_t)q);
  }
}

struct FirstIn {
  const uint32_t* raw;
  const uint32_t* minidx;
  __device__ uint32_t operator()(uint64_t q) const { return minidx[raw[q]] == (uint32_t)q; }
};
struct FirstOut {
  uint32_t* rank;
  __device__ void operator()(uint64_t q, uint32_t excl, uint32_t v) const {
    if (v) rank[q] = excl;
  }
};

__global__ void __launch_bounds__(256) relabel_kernel(const uint32_t* __restrict__ raw, uint64_t n,
                                                      const uint32_t* __restrict__ minidx,
                                                      const uint32_t* __restrict__ rank,
                                                      uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride)
    out[q] = rank[minidx[raw[q]]];
}

__device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t j) {
  // the j-th (0-based) draw of SplitMix64(seed): state advanced j+1 times
  uint64_t z = seed + (j + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) random_delta_kernel(uint32_t* __restrict__ delta, uint64_t n,
                                                           uint64_t total, uint64_t seed) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += stride)
    delta[j] = (uint32_t)(splitmix_draw(seed, j) % n);  // draw order: row a, state q = a*n+q
}

__global__ void __launch_bounds__(256) random_acc_kernel(uint8_t* __restrict__ acc, uint64_t n,
                                                         uint64_t offset, uint64_t seed, double p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    const double u = (double)(splitmix_draw(seed, offset + q) >> 11) * 0x1.0p-53;
    acc[q] = u < p ? 1 : 0;
  }
}

}  // namespace

uint32_t canonicalize_dev(Ctx& ctx, const uint32_t* raw, uint64_t n, uint32_t* out) {
  if (n == 0) return 0;
  uint32_t* minidx = ctx.slot_t<uint32_t>("cn.min", n);
  uint32_t* rank = ctx.slot_t<uint32_t>("cn.rank", n);
  uint64_t* total = ctx.d_scalars + 8;
  const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(n, 256), (uint64_t)ctx.num_sms * 16);
  // raw 4 (x3 passes) + min index 4 (x3) + rank 4 (x2) + out 4 per state
  ProfScope p(ctx, "canon", n * 36ull);
  DFM_CUDA(cudaMemsetAsync(minidx, 0xFF, n * 4, ctx.stream));
  min_index_kernel<<<grid, 256, 0, ctx.stream>>>(raw, n, minidx);
  DFM_LAUNCH_CHECK();
  prims::lookback_scan(ctx, "sc.canon", n, FirstIn{raw, minidx}, FirstOut{rank}, total);
  relabel_kernel<<<grid, 256, 0, ctx.stream>>>(raw, n, minidx, rank, out);
  DFM_LAUNCH_CHECK();
  DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 8, total, 8, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  return (uint32_t)ctx.h_scalars[8];
}

void random_dfa_dev(Ctx& ctx, DevDfa& d, uint32_t n, uint32_t k, uint64_t seed, double p) {
  const uint64_t total = (uint64_t)n * k;
  const unsigned grid =
      (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(total, 1), 256), ctx.num_sms * 32ull);
  random_delta_kernel<<<grid, 256, 0, ctx.stream>>>(d.delta, n, total, seed);
  DFM_LAUNCH_CHECK();
  random_acc_kernel<<<grid, 256, 0, ctx.stream>>>(d.acc, n, total, seed, p);
  DFM_LAUNCH_CHECK();
}

}  // namespace dfm
