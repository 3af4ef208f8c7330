// Microbenchmark: random 4-byte gathers from a >L2 array on B200, by load flavour
// and L2 fetch granularity.  out[i] = tab[idx[i]] for 1e8 random idx into 4e8 B.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ uint32_t ld(const uint32_t* p) {
  uint32_t v;
  if (V == 0) asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (V == 1) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (V == 2) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (V == 3) asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  else asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int V>
__global__ void gather(const uint32_t* __restrict__ idx, const uint32_t* tab, uint32_t* out, uint64_t m) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = ld<V>(tab + idx[i]);
}

__global__ void init(uint32_t* idx, uint64_t m, uint32_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ull + 12345;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    idx[i] = (uint32_t)(z % n);
  }
}

template <int V>
float run(const uint32_t* idx, const uint32_t* tab, uint32_t* out, uint64_t m) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  gather<V><<<148 * 16, 256>>>(idx, tab, out, m);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) gather<V><<<148 * 16, 256>>>(idx, tab, out, m);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}

int main(int argc, char** argv) {
  const uint64_t m = 100000000; const uint32_t n = 100000000;
  uint32_t *idx, *tab, *out;
  cudaMalloc(&idx, m * 4); cudaMalloc(&tab, (uint64_t)n * 4); cudaMalloc(&out, m * 4);
  init<<<148 * 16, 256>>>(idx, m, n); cudaMemset(tab, 1, (uint64_t)n * 4);
  for (int g : {0, 32, 64, 128}) {
    if (g) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
    size_t cur = 0; cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
    const char* names[] = {"ld.global", "ld.global.nc", "ld.global.cg", "L1::no_allocate", "ld.global.cs"};
    float t[5] = {run<0>(idx, tab, out, m), run<1>(idx, tab, out, m), run<2>(idx, tab, out, m),
                  run<3>(idx, tab, out, m), run<4>(idx, tab, out, m)};
    for (int v = 0; v < 5; ++v)
      printf("granularity=%zu %-16s %.3f ms  %.1f Mgathers/s  (%.1f GB/s at 32B/gather)\n", cur, names[v], t[v], m / t[v] / 1e3, m * 32.0 / t[v] / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
