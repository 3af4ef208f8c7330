// Cho–Huynh pair-graph closure (paper Alg. 1; reference min_trans.hpp:81-212).
//
// Pair node (q,r) has index s = q*n + r (|V| = n^2).  Each pass:
//   next  = reach ∨ reach·reach          (boolean squaring, pass-entry reach)
//   apart' = apart ∨ (∃t next[s][t] ∧ apart[t])   (pass-entry apart)
// until apart stops changing; label[q] = min q0 <= q not apart from q.
//
// Two squaring engines behind one driver:
//   * tcgen05 int8 GEMM (trans_tc.cu): 0/1 int8 matrices, int32 TMEM
//     accumulators, epilogue thresholds >0, ORs reach, writes next/nextT and
//     fuses the apartness propagation — the tensor-core path.
//   * bit-broadcast GEMM on CUDA cores (this file): packed 64-bit rows; used
//     for |V| below one tensor tile and as the cross-check engine.
#include <algorithm>
#include <vector>

#include "prims.cuh"
#include "trans_tc.cuh"

namespace dfm {
namespace {

__global__ void pair_init_kernel(const uint32_t* __restrict__ delta, const uint8_t* __restrict__ acc,
                                 uint64_t n, uint32_t k, uint64_t V, uint64_t W,
                                 unsigned long long* __restrict__ reach) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < V; s += stride) {
    const uint64_t q = s / n, r = s % n;
    unsigned long long* row = reach + s * W;
    for (uint32_t a = 0; a < k; ++a) {
      const uint64_t t = (uint64_t)delta[a * n + q] * n + delta[a * n + r];
      row[t >> 6] |= 1ull << (t & 63);
    }
  }
}

__global__ void apart_init_kernel(const uint8_t* __restrict__ acc, uint64_t n, uint64_t V,
                                  uint64_t W, unsigned long long* __restrict__ apart) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < W; w += stride) {
    unsigned long long bits = 0;
    for (int b = 0; b < 64; ++b) {
      const uint64_t s = w * 64 + b;
      if (s < V && acc[s / n] != acc[s % n]) bits |= 1ull << b;
    }
    apart[w] = bits;
  }
}

// next[i][wj] = reach[i][wj] | OR_t bit(reach[i], t) & reach[t][wj]
// CTA tile: 64 rows x 32 words (2048 columns); 8 rows per thread; t in chunks of 64.
constexpr int kBgRows = 64, kBgWords = 32;
__global__ void __launch_bounds__(256) bitgemm_square_kernel(const unsigned long long* __restrict__ reach,
                                                             unsigned long long* __restrict__ next,
                                                             uint64_t V, uint64_t W) {
  __shared__ unsigned long long sA[kBgRows];
  __shared__ unsigned long long sB[64][kBgWords];
  const int tid = threadIdx.x;
  const int word = tid & 31;
  const int rbase = (tid >> 5) * 8;
  const uint64_t i0 = (uint64_t)blockIdx.y * kBgRows;
  const uint64_t j0 = (uint64_t)blockIdx.x * kBgWords;
  unsigned long long acc[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint64_t i = i0 + rbase + r;
    acc[r] = (i < V && j0 + word < W) ? reach[i * W + j0 + word] : 0ull;
  }
  for (uint64_t tw = 0; tw < W; ++tw) {
    __syncthreads();
    if (tid < kBgRows) {
      const uint64_t i = i0 + tid;
      sA[tid] = i < V ? reach[i * W + tw] : 0ull;
    }
    for (int e = tid; e < 64 * kBgWords; e += 256) {
      const int tt = e / kBgWords, ww = e % kBgWords;
      const uint64_t t = tw * 64 + tt;
      sB[tt][ww] = (t < V && j0 + ww < W) ? reach[t * W + j0 + ww] : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      unsigned long long a = sA[rbase + r];
      while (a) {
        const int t = __ffsll((long long)a) - 1;
        a &= a - 1;
        acc[r] |= sB[t][word];
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint64_t i = i0 + rbase + r;
    if (i < V && j0 + word < W) next[i * W + j0 + word] = acc[r];
  }
}

// apart'[s] = apart[s] | any_w(next[s][w] & apart[w]); one warp per row
__global__ void __launch_bounds__(256) propagate_kernel(const unsigned long long* __restrict__ next,
                                                        const unsigned long long* __restrict__ apart,
                                                        unsigned long long* apart_next, uint64_t V,
                                                        uint64_t W) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t s = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < V;
       s += warps) {
    bool hit = (apart[s >> 6] >> (s & 63)) & 1;
    if (!hit) {
      const unsigned long long* row = next + s * W;
      unsigned long long x = 0;
      for (uint64_t w = lane; w < W; w += 32) x |= row[w] & apart[w];
      hit = __any_sync(0xffffffffu, x != 0);
    }
    if (hit && lane == 0) atomicOr(&apart_next[s >> 6], 1ull << (s & 63));
  }
}

__global__ void apart_stats_kernel(const unsigned long long* __restrict__ a,
                                   const unsigned long long* __restrict__ b, uint64_t W,
                                   unsigned long long* out /*[0] diff, [1] popcount(b)*/) {
  unsigned long long diff = 0, pop = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < W; w += stride) {
    diff |= a[w] ^ b[w];
    pop += __popcll(b[w]);
  }
  if (diff) atomicOr(&out[0], 1ull);
  if (pop) atomicAdd(&out[1], pop);
}

__global__ void labels_kernel(const unsigned long long* __restrict__ apart, uint64_t n,
                              uint32_t* __restrict__ label) {
  const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  uint32_t l = (uint32_t)q;
  for (uint64_t q0 = 0; q0 <= q; ++q0) {  // min_trans.hpp:189-197
    const uint64_t i = q0 * n + q;
    if (!((apart[i >> 6] >> (i & 63)) & 1)) {
      l = (uint32_t)q0;
      break;
    }
  }
  label[q] = l;
}

unsigned grid_for(const Ctx& ctx, uint64_t items) {
  return (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(items, 1), 256),
                                      (uint64_t)ctx.num_sms * 16);
}

}  // namespace

AlgoOut run_trans_minimize(Ctx& ctx, const DevDfa& d, const dfm_limits& lim, const Deadline& dl,
                           uint8_t* apart_host, uint64_t* popcounts, uint32_t pop_cap) {
  AlgoOut out;
  const uint64_t n = d.n;
  const uint64_t required = dfm_trans_required_bytes(n);
  if (required > lim.max_memory_bytes) {  // min_trans.hpp:88-95
    out.status = DFM_STATUS_CAPACITY_EXCEEDED;
    out.peak_memory_estimate = required;
    return out;
  }
  const uint64_t V = n * n;
  const uint64_t W = ceil_div(V, 64);
  out.peak_memory_estimate = 2 * V * W * 8 + 2 * W * 8;  // min_trans.hpp:203-205
  auto* apart = ctx.slot_t<unsigned long long>("tr.apart", W);
  auto* apart_next = ctx.slot_t<unsigned long long>("tr.apart2", W);
  auto* stats = reinterpret_cast<unsigned long long*>(ctx.d_scalars + 24);
  const bool use_tc = trans_tc::usable(V, ctx.trans_engine);
  TransTcState tc;
  unsigned long long* reach = nullptr;
  unsigned long long* next = nullptr;
  {
    ProfScope p(ctx, "init");
    if (use_tc) {
      tc = trans_tc::init(ctx, d, V);
    } else {
      reach = ctx.slot_t<unsigned long long>("tr.reach", V * W);
      next = ctx.slot_t<unsigned long long>("tr.next", V * W);
      DFM_CUDA(cudaMemsetAsync(reach, 0, V * W * 8, ctx.stream));
      pair_init_kernel<<<grid_for(ctx, V), 256, 0, ctx.stream>>>(d.delta, d.acc, n, d.k, V, W,
                                                                  reach);
      DFM_LAUNCH_CHECK();
    }
    apart_init_kernel<<<grid_for(ctx, W), 256, 0, ctx.stream>>>(d.acc, n, V, W, apart);
    DFM_LAUNCH_CHECK();
  }
  bool changed = true;
  while (changed) {
    if (dl.expired()) {
      out.status = DFM_STATUS_TIMEOUT;
      return out;
    }
    DFM_CUDA(cudaMemsetAsync(apart_next, 0, W * 8, ctx.stream));
    DFM_CUDA(cudaMemsetAsync(stats, 0, 16, ctx.stream));
    if (use_tc) {
      trans_tc::square_and_propagate(ctx, tc, apart, apart_next);
    } else {
      {
        ProfScope p(ctx, "gemm");
        dim3 g((unsigned)ceil_div(W, kBgWords), (unsigned)ceil_div(V, kBgRows));
        bitgemm_square_kernel<<<g, 256, 0, ctx.stream>>>(reach, next, V, W);
        DFM_LAUNCH_CHECK();
      }
      {
        ProfScope p(ctx, "propagate");
        propagate_kernel<<<grid_for(ctx, V * 32), 256, 0, ctx.stream>>>(next, apart, apart_next, V,
                                                                        W);
        DFM_LAUNCH_CHECK();
      }
      std::swap(reach, next);
    }
    apart_stats_kernel<<<grid_for(ctx, W), 256, 0, ctx.stream>>>(apart, apart_next, W, stats);
    DFM_LAUNCH_CHECK();
    DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 24, stats, 16, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    ++out.iterations;
    changed = ctx.h_scalars[24] != 0;
    if (popcounts && out.iterations <= pop_cap) popcounts[out.iterations - 1] = ctx.h_scalars[25];
    std::swap(apart, apart_next);
  }
  uint32_t* label = ctx.slot_t<uint32_t>("tr.label", n);
  labels_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, ctx.stream>>>(apart, n, label);
  DFM_LAUNCH_CHECK();
  if (apart_host) {
    std::vector<unsigned long long> bits(W);
    DFM_CUDA(cudaMemcpyAsync(bits.data(), apart, W * 8, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    for (uint64_t i = 0; i < V; ++i) apart_host[i] = (bits[i >> 6] >> (i & 63)) & 1;
  }
  out.canon_dev = ctx.slot_t<uint32_t>("canon", n);
  out.num_blocks = canonicalize_dev(ctx, label, n, out.canon_dev);
  out.status = DFM_STATUS_OK;
  return out;
}

}  // namespace dfm
