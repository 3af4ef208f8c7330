// Microbenchmark: cost model of random accesses on B200 as a function of the
// footprint (L2-resident vs HBM): 4-byte gathers, 4-byte scatters, u32 RED,
// u64 CAS, 128-bit CAS, and shared-memory gathers.  1e8 operations each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_bench tools/l2_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// V: 0 gather u32, 1 scatter u32, 2 red.add u32, 3 cas u64 (ret used), 4 cas b128, 5 gather evict_last,
//    6 gather (index from a coalesced stream, like the blocked builder)
template <int V>
__global__ void __launch_bounds__(256) k(uint32_t* tab, uint64_t words, uint64_t m, unsigned* sink,
                                         const uint32_t* idx) {
  unsigned acc = 0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix(i + 12345);
    const uint64_t s = V == 6 ? idx[i] : __umul64hi(h, words);
    if (V == 0 || V == 6) {
      acc += __ldg(tab + s);
    } else if (V == 1) {
      tab[s] = (uint32_t)i;
    } else if (V == 2) {
      atomicAdd(tab + s, 1u);
    } else if (V == 3) {
      acc += (unsigned)atomicCAS(reinterpret_cast<unsigned long long*>(tab) + (s >> 1), 0ull, h | 1);
    } else if (V == 4) {
      unsigned long long lo, hi;
      asm volatile(
          "{\n\t.reg .b128 d, c, v;\n\t"
          "mov.b128 c, {%2, %3};\n\t"
          "mov.b128 v, {%4, %5};\n\t"
          "atom.global.cas.b128 d, [%6], c, v;\n\t"
          "mov.b128 {%0, %1}, d;\n\t}"
          : "=l"(lo), "=l"(hi)
          : "l"(0ull), "l"(0ull), "l"(h | 1), "l"(i), "l"(tab + ((s >> 2) << 2))
          : "memory");
      acc += (unsigned)lo;
    } else if (V == 5) {
      uint32_t v;
      asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(tab + s), "l"(pol));
      acc += v;
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void __launch_bounds__(1024) smem_gather(uint64_t m, unsigned* sink, uint32_t words) {
  extern __shared__ uint32_t s[];
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) s[i] = i;
  __syncthreads();
  unsigned acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc += s[(uint32_t)__umul64hi(mix(i + 99), words)];
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void fill_idx(uint32_t* idx, uint64_t m, uint64_t words) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    idx[i] = (uint32_t)__umul64hi(mix(i + 777), words);
}

template <int V>
float run(uint32_t* tab, uint64_t words, uint64_t m, unsigned* sink, const uint32_t* idx) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<V><<<148 * 8, 256>>>(tab, words, m, sink, idx);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) k<V><<<148 * 8, 256>>>(tab, words, m, sink, idx);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 3;
}

int main() {
  const uint64_t m = 100000000;
  uint32_t* tab;
  uint32_t* idx;
  unsigned* sink;
  cudaMalloc(&tab, 1ull << 31);
  cudaMalloc(&idx, m * 4);
  cudaMalloc(&sink, 4);
  cudaMemset(tab, 0, 1ull << 31);
  const char* names[] = {"gather", "scatter", "red.add", "cas64", "cas128", "gather_evl", "gather_idx"};
  printf("%10s", "footprint");
  for (auto nm : names) printf(" %12s", nm);
  printf("   (G ops/s)\n");
  for (uint64_t mb : {1ull, 16ull, 32ull, 48ull, 56ull, 64ull, 72ull, 80ull, 96ull, 112ull, 128ull, 512ull}) {
    const uint64_t words = (mb << 20) / 4;
    fill_idx<<<148 * 8, 256>>>(idx, m, words);
    float t[7] = {run<0>(tab, words, m, sink, idx), run<1>(tab, words, m, sink, idx),
                  run<2>(tab, words, m, sink, idx), run<3>(tab, words, m, sink, idx),
                  run<4>(tab, words, m, sink, idx), run<5>(tab, words, m, sink, idx),
                  run<6>(tab, words, m, sink, idx)};
    printf("%8llu MB", (unsigned long long)mb);
    for (float x : t) printf(" %12.1f", m / x / 1e6);
    printf("\n");
  }
  for (uint32_t kb : {16u, 64u, 200u}) {
    const uint32_t words = kb * 256;
    cudaFuncSetAttribute(smem_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    smem_gather<<<148, 1024, kb * 1024>>>(m, sink, words);
    cudaEventRecord(a);
    smem_gather<<<148, 1024, kb * 1024>>>(m, sink, words);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("smem gather %u KB: %.1f G ops/s\n", kb, m / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
