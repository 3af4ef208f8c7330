// Grid-barrier cost on B200: cooperative-groups grid.sync() vs a hand-rolled
// generation barrier (one arrival atomic per CTA, acquire polling), as used between
// naivePR passes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gridsync_bench
// tools/cuda/gridsync_bench.cu && build/gridsync_bench
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void cg_kernel(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x ^ i;
    g.sync();
  }
  if (acc == 0xFFFFFFFFu) *sink = acc;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// bar[0] = arrivals, bar[1] = generation
__device__ __forceinline__ void gen_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned n = gridDim.x;
    const unsigned old = atom_add_acqrel(&bar[0], 1u);
    if (old == n - 1) {
      bar[0] = 0;  // ordered before the release below
      st_release(&bar[1], gen + 1);
    } else {
      while (ld_acquire(&bar[1]) == gen) {
      }
    }
  }
  ++gen;
  __syncthreads();
}

__global__ void gen_kernel(int iters, unsigned* bar, unsigned* sink) {
  unsigned gen = 0, acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x ^ i;
    gen_barrier(bar, gen);
  }
  if (acc == 0xFFFFFFFFu) *sink = acc;
}

// monotonic counter: arrival i of pass p waits for count >= (p+1)*n (no reset, no flag)
__device__ __forceinline__ void mono_barrier(unsigned* bar, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    atom_add_acqrel(&bar[0], 1u);
    while (ld_acquire(&bar[0]) < target) {
    }
  }
  __syncthreads();
}
__global__ void mono_kernel(int iters, unsigned* bar, unsigned* sink) {
  unsigned target = 0, acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x ^ i;
    mono_barrier(bar, target);
  }
  if (acc == 0xFFFFFFFFu) *sink = acc;
}

int main() {
  unsigned *bar, *sink;
  cudaMalloc(&bar, 64);
  cudaMalloc(&sink, 4);
  const int iters = 20000;
  for (int blocks : {98, 148, 296}) {
    for (int threads : {256, 1024}) {
      if (blocks * threads > 148 * 2048) continue;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float ms[3] = {0, 0, 0};
      for (int kind = 0; kind < 3; ++kind) {
        cudaMemset(bar, 0, 64);
        int it = iters;
        void* args[] = {&it, kind == 0 ? (void*)&sink : (void*)&bar, &sink};
        cudaEventRecord(a);
        if (kind == 0) {
          void* a0[] = {&it, &sink};
          cudaLaunchCooperativeKernel((void*)cg_kernel, blocks, threads, a0, 0, 0);
        } else if (kind == 1) {
          cudaLaunchCooperativeKernel((void*)gen_kernel, blocks, threads, args, 0, 0);
        } else {
          cudaLaunchCooperativeKernel((void*)mono_kernel, blocks, threads, args, 0, 0);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms[kind], a, b);
      }
      const cudaError_t e = cudaGetLastError();
      printf("blocks %3d x %4d: cg.sync %.3f us  gen-barrier %.3f us  monotonic %.3f us  (%s)\n",
             blocks, threads, 1e3 * ms[0] / iters, 1e3 * ms[1] / iters, 1e3 * ms[2] / iters,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
