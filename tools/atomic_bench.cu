// Microbenchmark: random-slot atomics on >L2 tables (the sortPR hash-engine insert).
// 1e8 items, slot = hash(i) over `slots` 16-byte slots; variants:
//   red2   : atomicMax(rep) + atomicAdd(info)            (2 fire-and-forget REDs)
//   red1   : atomicAdd(info) only
//   min1   : atomicMin(rep) with the return value used   (1 ATOM)
//   cas    : atomicCAS(key) (return used) + red2          (the hash-table insert)
//   cas1   : atomicCAS(key) only
//   cas128 : one 128-bit CAS of {key, rep} (atom.cas.b128)
//   gather : plain 16-byte load of the slot (reference point)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

struct __align__(16) Slot {
  unsigned long long key;
  unsigned int rep, info;
};

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int V>
__global__ void k(Slot* t, uint64_t slots, uint64_t m, unsigned* sink) {
  unsigned acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix(i + 12345);
    const uint64_t s = __umul64hi(h, slots);
    Slot* p = t + s;
    if (V == 0) {
      atomicMax(&p->rep, ~(unsigned)i);
      atomicAdd(&p->info, 1u);
    } else if (V == 1) {
      atomicAdd(&p->info, 1u);
    } else if (V == 2) {
      acc += atomicMin(&p->rep, (unsigned)i);
    } else if (V == 3) {
      acc += (unsigned)atomicCAS(&p->key, 0ull, h | 1);
      atomicMax(&p->rep, ~(unsigned)i);
      atomicAdd(&p->info, 1u);
    } else if (V == 4) {
      acc += (unsigned)atomicCAS(&p->key, 0ull, h | 1);
    } else if (V == 5) {
      unsigned long long lo, hi;
      const unsigned long long nlo = h | 1, nhi = i;
      asm volatile(
          "{\n\t.reg .b128 d, c, sw;\n\t"
          "mov.b128 c, {%2, %3};\n\t"
          "mov.b128 sw, {%4, %5};\n\t"
          "atom.global.cas.b128 d, [%6], c, sw;\n\t"
          "mov.b128 {%0, %1}, d;\n\t}"
          : "=l"(lo), "=l"(hi)
          : "l"(0ull), "l"(0ull), "l"(nlo), "l"(nhi), "l"(p)
          : "memory");
      acc += (unsigned)lo;
    } else {
      unsigned x, y, z, w;
      asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                   : "l"(p));
      acc += x + z;
    }
  }
  if (acc == 0xFFFFFFFF) *sink = acc;
}

template <int V>
float run(Slot* t, uint64_t slots, uint64_t m, unsigned* sink) {
  cudaMemset(t, 0, slots * sizeof(Slot));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<V><<<148 * 16, 256>>>(t, slots, m, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  const uint64_t m = 100000000;
  Slot* t;
  unsigned* sink;
  cudaMalloc(&t, 150000000ull * sizeof(Slot));
  cudaMalloc(&sink, 4);
  const char* names[] = {"red2", "red1", "min1", "cas+red2", "cas1", "cas128", "load16"};
  for (uint64_t slots : {1ull << 25, 150000000ull}) {
    for (int rep = 0; rep < 2; ++rep) {
      float v[7] = {run<0>(t, slots, m, sink), run<1>(t, slots, m, sink), run<2>(t, slots, m, sink),
                    run<3>(t, slots, m, sink), run<4>(t, slots, m, sink), run<5>(t, slots, m, sink),
                    run<6>(t, slots, m, sink)};
      if (rep == 1)
        for (int i = 0; i < 7; ++i)
          printf("slots=%llu (%5.0f MB) %-9s %7.3f ms  %6.1f Gops/s\n", (unsigned long long)slots,
                 slots * 16 / 1e6, names[i], v[i], m / v[i] / 1e6);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
