// tcgen05 int8 squaring engine for the Cho–Huynh closure (reference
// min_trans.hpp:131-186; paper Alg. 1), sm_100a.
//
// The pair-graph reachability matrix R (|V| x |V|, |V| = n^2, padded to Vp) is
// held as 0/1 bytes.  One pass computes, tile by tile,
//     acc  = R · R                      (tcgen05.mma kind::i8, u8 x u8 -> s32 in TMEM)
//     next = (acc > 0) | R              (epilogue, written as bytes)
//     apart_next[i] |= OR_j next[i][j] & apart[j]     (fused propagation)
// which is exactly the reference's squaring (next = reach ∨ reach², pass-entry
// reach) followed by its propagation (pass-entry apart).
//
// Kernel anatomy (one CTA per 128x256 output tile, 256 threads):
//   warp 0      TMA producer: A = R[m0:m0+128, k:k+128] (K-major, 128B swizzle),
//               B = R[k:k+128, n0:n0+256] (MN-major, two 128-byte swizzle atoms)
//   warp 1      MMA issuer (one elected lane): 4 x (128x256x32) per stage
//   warp 2      TMEM allocator (256 columns of 32-bit accumulators)
//   warps 4..7  epilogue: tcgen05.ld 32x32b.x32 per 32 columns, threshold, OR,
//               store, propagate
// 4-stage smem ring (48 KB/stage) with full/empty mbarriers; tcgen05.commit
// frees a stage and finally signals the accumulator.
#include <cuda.h>

#include <algorithm>

#include "prims.cuh"
#include "trans_tc.cuh"

namespace dfm {
namespace trans_tc {
namespace {

constexpr int kBM = 128, kBN = 256, kBK = 128, kStages = 4;
constexpr int kStageA = kBM * kBK;                 // 16 KB
constexpr int kStageB = kBK * kBN;                 // 32 KB
constexpr int kStageBytes = kStageA + kStageB;     // 48 KB
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr int kThreads = 256;
constexpr int kGroupM = 16;  // rasterisation: 16 M-tiles share the concurrent wave
constexpr uint32_t kMaxKBlocks = 1024;  // Vp <= 131072 (|V| = n^2 <= 65,536 here)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// UMMA shared-memory descriptor (sm100 "version 1"), 128B swizzle
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// instruction descriptor: kind::i8, u8 x u8 -> s32, A K-major, B MN-major, M=128, N=256
constexpr uint32_t kIdesc = (2u << 4)            // D format S32
                            | (0u << 7)          // A u8
                            | (0u << 10)         // B u8
                            | (0u << 15)         // A K-major
                            | (1u << 16)         // B MN-major
                            | ((kBN >> 3) << 17) // N
                            | ((kBM >> 4) << 24);// M

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// tile occupancy bit of the 128x128 tile (mt, ct)
__device__ __forceinline__ bool tile_nz(const uint32_t* nz, uint32_t T, uint32_t mt, uint32_t ct) {
  const uint32_t b = mt * T + ct;
  return (nz[b >> 5] >> (b & 31)) & 1u;
}

__global__ void __launch_bounds__(kThreads, 1)
    square_kernel(const __grid_constant__ CUtensorMap map, const int8_t* __restrict__ reach,
                  int8_t* __restrict__ next, const unsigned long long* __restrict__ apart,
                  unsigned long long* apart_next, uint32_t Vp, uint32_t W,
                  const uint32_t* __restrict__ nz, uint32_t* __restrict__ nz_next,
                  unsigned long long* live_blocks, const uint32_t* __restrict__ tile_list) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // rasterised tile order: groups of kGroupM M-tiles sweep all N-tiles together
  const uint32_t tiles_m = Vp / kBM, tiles_n = Vp / kBN;
  const uint32_t tid = tile_list[blockIdx.x];  // a tile with live K blocks
  const uint32_t group = tid / (kGroupM * tiles_n);
  const uint32_t first_m = group * kGroupM;
  const uint32_t gm = min((uint32_t)kGroupM, tiles_m - first_m);
  const uint32_t in_group = tid - group * kGroupM * tiles_n;
  const uint32_t m0 = (first_m + in_group % gm) * kBM;
  const uint32_t n0 = (in_group / gm) * kBN;
  const uint32_t kblocks = Vp / kBK;
  // K block kb contributes only if the A tile (m0, kb) and one of the B tiles
  // (kb, n0) / (kb, n0 + 128) hold a one (producer and MMA warp skip the same ones)
  const uint32_t T = Vp / 128, mt = m0 / 128, nt = n0 / 128;
  __shared__ uint32_t s_live[kMaxKBlocks / 32];  // live K blocks of this tile, one bit each
  for (uint32_t w = threadIdx.x; w < kMaxKBlocks / 32; w += blockDim.x) s_live[w] = 0;
  __syncthreads();
  for (uint32_t kb = threadIdx.x; kb < kblocks; kb += blockDim.x)
    if (tile_nz(nz, T, mt, kb) && (tile_nz(nz, T, kb, nt) || tile_nz(nz, T, kb, nt + 1)))
      atomicOr(&s_live[kb >> 5], 1u << (kb & 31));
  auto live = [&](uint32_t kb) { return (s_live[kb >> 5] >> (kb & 31)) & 1u; };
  // (tiles without a live K block never get here: dead_copy_kernel handles them;
  // the __syncthreads below — after the TMEM allocation — publishes s_live)

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      uint32_t j = 0;  // live blocks so far
      for (uint32_t kb = 0; kb < kblocks; ++kb) {
        if (!live(kb)) continue;
        const int s = j % kStages;
        const uint32_t round = j / kStages;
        if (j >= (uint32_t)kStages) mbar_wait(&empty[s], (round - 1) & 1);
        ++j;
        uint8_t* a = smem + s * kStageBytes;
        uint8_t* b = a + kStageA;
        mbar_expect_tx(&full[s], kStageBytes);
        tma_load_2d(a, &map, &full[s], (int)(kb * kBK), (int)m0);         // A: {k, m}
        tma_load_2d(b, &map, &full[s], (int)n0, (int)(kb * kBK));         // B: {n, k} lo
        tma_load_2d(b + kStageB / 2, &map, &full[s], (int)(n0 + 128), (int)(kb * kBK));  // hi
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      uint32_t j = 0;
      for (uint32_t kb = 0; kb < kblocks; ++kb) {
        if (!live(kb)) continue;
        const int s = j % kStages;
        mbar_wait(&full[s], (j / kStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a = smem_u32(smem + s * kStageBytes);
        const uint32_t b = a + kStageA;
#pragma unroll
        for (int kk = 0; kk < kBK / 32; ++kk) {
          // A K-major: +32 bytes along K; B MN-major: +32 rows of 128 bytes
          const uint64_t da = smem_desc(a + kk * 32, 16, 1024);
          const uint64_t db = smem_desc(b + kk * 32 * 128, kStageB / 2, 1024);
          umma_i8(tmem, da, db, (j | kk) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);  // frees the stage once these MMAs retire
        ++j;
      }
      if (j) atomicAdd(live_blocks, (unsigned long long)j);  // (the executed ops, for the roofline)
      umma_commit(acc_full);
    }
  } else if (warp >= 4) {  // epilogue: one accumulator row per thread
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    bool any_mma = false;  // no live K block: the accumulator was never written (zero)
    for (uint32_t kb = 0; kb < kblocks && !any_mma; ++kb) any_mma = live(kb);
    const uint32_t quarter = warp - 4;  // TMEM lanes [32*quarter, 32*quarter+32)
    const uint32_t row = m0 + quarter * 32 + lane;
    const int8_t* rrow = reach + (uint64_t)row * Vp;
    int8_t* nrow = next + (uint64_t)row * Vp;
    bool hit = false;
    // an R half whose occupancy bit is clear is zero (and may be unwritten: dead_copy
    // skips all-zero tiles)
    const bool r_lo = tile_nz(nz, T, mt, nt), r_hi = tile_nz(nz, T, mt, nt + 1);
#pragma unroll 1
    for (int c = 0; c < kBN / 32; ++c) {
      uint32_t v[32];
      if (any_mma) {
        tmem_ld32(tmem + ((quarter * 32) << 16) + c * 32, v);
      } else {
#pragma unroll
        for (int b = 0; b < 32; ++b) v[b] = 0;
      }
      const uint32_t j0 = n0 + c * 32;
      uint32_t rw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (c < 4 ? r_lo : r_hi) {
        const uint4* rp = reinterpret_cast<const uint4*>(rrow + j0);
        const uint4 r0 = rp[0], r1 = rp[1];
        rw[0] = r0.x; rw[1] = r0.y; rw[2] = r0.z; rw[3] = r0.w;
        rw[4] = r1.x; rw[5] = r1.y; rw[6] = r1.z; rw[7] = r1.w;
      }
      uint32_t mask = 0;
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        const uint32_t rb = (rw[b >> 2] >> ((b & 3) * 8)) & 0xFFu;
        mask |= ((v[b] != 0u) | (rb != 0u) ? 1u : 0u) << b;
      }
      uint32_t ow[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const uint32_t nib = (mask >> (w * 4)) & 0xFu;
        ow[w] = (nib & 1u) | ((nib >> 1) & 1u) << 8 | ((nib >> 2) & 1u) << 16 |
                ((nib >> 3) & 1u) << 24;
      }
      uint4* op = reinterpret_cast<uint4*>(nrow + j0);
      op[0] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
      op[1] = make_uint4(ow[4], ow[5], ow[6], ow[7]);
      const uint32_t abits = (j0 >> 6) < W ? (uint32_t)(apart[j0 >> 6] >> (j0 & 63)) : 0u;
      hit |= (mask & abits) != 0u;
      // occupancy of next for the following pass: tile (mt, j0 / 128)
      if (__any_sync(0xffffffffu, mask != 0u) && lane == 0) {
        const uint32_t b = mt * T + j0 / 128;
        atomicOr(&nz_next[b >> 5], 1u << (b & 31));
      }
    }
    if (hit) atomicOr(&apart_next[row >> 6], 1ull << (row & 63));
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

// ---------------------------------------------------------------------------
// Persistent variant: one CTA per SM walks the live-tile list (static round robin),
// so the TMEM allocation, barrier setup and tensormap prefetch happen once per pass
// instead of once per tile; TMEM holds TWO 256-column accumulators, so the
// epilogue of tile i (warps 4..7) overlaps the TMA loads and MMAs of tile i+1
// (acc_full / acc_empty mbarrier pairs per buffer); the smem ring's stage counter
// runs across tiles.  The producer and MMA warps find a tile's live K blocks
// warp-cooperatively (one ballot per 32 K blocks) in the same order.  The epilogue
// skips reading R where both 128x128 halves of the R tile are zero (occupancy
// bits), and dead_copy skips all-zero tiles: a tile whose occupancy bit is clear
// is never read by anyone (TMA loads, epilogue, copy), so it need not be written.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tile_coords(uint32_t tid, uint32_t Vp, uint32_t& m0, uint32_t& n0) {
  const uint32_t tiles_m = Vp / kBM, tiles_n = Vp / kBN;
  const uint32_t group = tid / (kGroupM * tiles_n);
  const uint32_t first_m = group * kGroupM;
  const uint32_t gm = min((uint32_t)kGroupM, tiles_m - first_m);
  const uint32_t in_group = tid - group * kGroupM * tiles_n;
  m0 = (first_m + in_group % gm) * kBM;
  n0 = (in_group / gm) * kBN;
}

// live K blocks kb0..kb0+31 of output tile (mt, nt..nt+1), one bit per lane
__device__ __forceinline__ uint32_t live_mask32(const uint32_t* nz, uint32_t T, uint32_t mt,
                                                uint32_t nt, uint32_t kb0, uint32_t kblocks,
                                                uint32_t lane) {
  const uint32_t kb = kb0 + lane;
  const bool lv = kb < kblocks && tile_nz(nz, T, mt, kb) &&
                  (tile_nz(nz, T, kb, nt) || tile_nz(nz, T, kb, nt + 1));
  return __ballot_sync(0xffffffffu, lv);
}

__global__ void __launch_bounds__(kThreads, 1)
    square_persistent_kernel(const __grid_constant__ CUtensorMap map,
                             const int8_t* __restrict__ reach, int8_t* __restrict__ next,
                             const unsigned long long* __restrict__ apart,
                             unsigned long long* apart_next, uint32_t Vp, uint32_t W,
                             const uint32_t* __restrict__ nz, uint32_t* __restrict__ nz_next,
                             unsigned long long* live_blocks,
                             const uint32_t* __restrict__ tile_list, uint32_t n_tiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t kblocks = Vp / kBK, T = Vp / 128;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // TMA producer (whole warp finds the live blocks, lane 0 issues)
    uint32_t j = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      uint32_t m0, n0;
      tile_coords(tile_list[t], Vp, m0, n0);
      const uint32_t mt = m0 / 128, nt = n0 / 128;
      for (uint32_t kb0 = 0; kb0 < kblocks; kb0 += 32) {
        uint32_t mask = live_mask32(nz, T, mt, nt, kb0, kblocks, lane);
        while (mask) {
          const uint32_t kb = kb0 + __ffs(mask) - 1;
          mask &= mask - 1;
          if (lane == 0) {
            const int s = j % kStages;
            if (j >= (uint32_t)kStages) mbar_wait(&empty[s], ((j / kStages) - 1) & 1);
            uint8_t* a = smem + s * kStageBytes;
            uint8_t* b = a + kStageA;
            mbar_expect_tx(&full[s], kStageBytes);
            tma_load_2d(a, &map, &full[s], (int)(kb * kBK), (int)m0);
            tma_load_2d(b, &map, &full[s], (int)n0, (int)(kb * kBK));
            tma_load_2d(b + kStageB / 2, &map, &full[s], (int)(n0 + 128), (int)(kb * kBK));
          }
          ++j;
        }
      }
    }
  } else if (warp == 1) {  // MMA issuer
    uint32_t j = 0, tl = 0;
    unsigned long long done = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      uint32_t m0, n0;
      tile_coords(tile_list[t], Vp, m0, n0);
      const uint32_t mt = m0 / 128, nt = n0 / 128;
      const uint32_t buf = tl & 1, use = tl >> 1;
      if (tl >= 2) mbar_wait(&acc_empty[buf], (use - 1) & 1);  // epilogue drained it
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dacc = tmem + buf * kBN;
      bool first = true;
      for (uint32_t kb0 = 0; kb0 < kblocks; kb0 += 32) {
        uint32_t mask = live_mask32(nz, T, mt, nt, kb0, kblocks, lane);
        while (mask) {
          mask &= mask - 1;
          if (lane == 0) {
            const int s = j % kStages;
            mbar_wait(&full[s], (j / kStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a = smem_u32(smem + s * kStageBytes);
            const uint32_t b = a + kStageA;
#pragma unroll
            for (int kk = 0; kk < kBK / 32; ++kk) {
              const uint64_t da = smem_desc(a + kk * 32, 16, 1024);
              const uint64_t db = smem_desc(b + kk * 32 * 128, kStageB / 2, 1024);
              umma_i8(dacc, da, db, (!first || kk != 0) ? 1u : 0u);
            }
            umma_commit(&empty[s]);
          }
          first = false;
          ++j;
          ++done;
        }
      }
      if (lane == 0) umma_commit(&acc_full[buf]);  // (every listed tile has a live block)
    }
    if (lane == 0 && done) atomicAdd(live_blocks, done);
  } else if (warp >= 4) {  // epilogue
    const uint32_t quarter = warp - 4;
    uint32_t tl = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      uint32_t m0, n0;
      tile_coords(tile_list[t], Vp, m0, n0);
      const uint32_t mt = m0 / 128;
      const uint32_t buf = tl & 1, use = tl >> 1;
      const bool r_lo = tile_nz(nz, T, mt, n0 / 128), r_hi = tile_nz(nz, T, mt, n0 / 128 + 1);
      mbar_wait(&acc_full[buf], use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t row = m0 + quarter * 32 + lane;
      const int8_t* rrow = reach + (uint64_t)row * Vp;
      int8_t* nrow = next + (uint64_t)row * Vp;
      bool hit = false;
#pragma unroll 1
      for (int c = 0; c < kBN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + ((quarter * 32) << 16) + buf * kBN + c * 32, v);
        const uint32_t j0 = n0 + c * 32;
        uint32_t rw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (c < 4 ? r_lo : r_hi) {
          const uint4* rp = reinterpret_cast<const uint4*>(rrow + j0);
          const uint4 r0 = rp[0], r1 = rp[1];
          rw[0] = r0.x; rw[1] = r0.y; rw[2] = r0.z; rw[3] = r0.w;
          rw[4] = r1.x; rw[5] = r1.y; rw[6] = r1.z; rw[7] = r1.w;
        }
        uint32_t mask = 0;
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          const uint32_t rb = (rw[b >> 2] >> ((b & 3) * 8)) & 0xFFu;
          mask |= ((v[b] != 0u) | (rb != 0u) ? 1u : 0u) << b;
        }
        uint32_t ow[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const uint32_t nib = (mask >> (w * 4)) & 0xFu;
          ow[w] = (nib & 1u) | ((nib >> 1) & 1u) << 8 | ((nib >> 2) & 1u) << 16 |
                  ((nib >> 3) & 1u) << 24;
        }
        uint4* op = reinterpret_cast<uint4*>(nrow + j0);
        op[0] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        op[1] = make_uint4(ow[4], ow[5], ow[6], ow[7]);
        const uint32_t abits = (j0 >> 6) < W ? (uint32_t)(apart[j0 >> 6] >> (j0 & 63)) : 0u;
        hit |= (mask & abits) != 0u;
        if (__any_sync(0xffffffffu, mask != 0u) && lane == 0) {
          const uint32_t b = mt * T + j0 / 128;
          atomicOr(&nz_next[b >> 5], 1u << (b & 31));
        }
      }
      if (hit) atomicOr(&apart_next[row >> 6], 1ull << (row & 63));
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

bool persist_enabled() {
  const char* e = getenv("DFM_TRANS_PERSIST");
  return e == nullptr || e[0] != '0';
}

// Output tiles (in square_kernel's rasterised order) with / without a live K block;
// the live ones go to the tensor kernel, the others to the copy kernel below, so
// the 197 KB-smem tensor CTAs run only where there is something to multiply
__global__ void tile_classify_kernel(const uint32_t* __restrict__ nz, uint32_t Vp,
                                     uint32_t* __restrict__ live_list,
                                     uint32_t* __restrict__ dead_list, uint32_t* counts) {
  const uint32_t tiles_m = Vp / kBM, tiles_n = Vp / kBN, T = Vp / 128;
  const uint32_t tiles = tiles_m * tiles_n;
  for (uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x; tid - (threadIdx.x & 31) < tiles;
       tid += gridDim.x * blockDim.x) {
    bool live = false;
    if (tid < tiles) {
      const uint32_t group = tid / (kGroupM * tiles_n);
      const uint32_t first_m = group * kGroupM;
      const uint32_t gm = min((uint32_t)kGroupM, tiles_m - first_m);
      const uint32_t in_group = tid - group * kGroupM * tiles_n;
      const uint32_t mt = first_m + in_group % gm, nt = (in_group / gm) * 2;
      for (uint32_t kb = 0; kb < T && !live; ++kb)
        live = tile_nz(nz, T, mt, kb) && (tile_nz(nz, T, kb, nt) || tile_nz(nz, T, kb, nt + 1));
    }
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t vm = __ballot_sync(0xffffffffu, tid < tiles && live);
    const uint32_t dm = __ballot_sync(0xffffffffu, tid < tiles && !live);
    uint32_t lb = 0, db = 0;
    if (lane == 0) {
      if (vm) lb = atomicAdd(&counts[0], (uint32_t)__popc(vm));
      if (dm) db = atomicAdd(&counts[1], (uint32_t)__popc(dm));
    }
    lb = __shfl_sync(0xffffffffu, lb, 0);
    db = __shfl_sync(0xffffffffu, db, 0);
    const uint32_t below = (1u << lane) - 1u;
    if ((vm >> lane) & 1u) live_list[lb + __popc(vm & below)] = tid;
    if ((dm >> lane) & 1u) dead_list[db + __popc(dm & below)] = tid;
  }
}

// next = R on a tile without live K blocks, with the apartness propagation and the
// occupancy bits (one 256-thread CTA per tile, small footprint: many CTAs per SM)
__global__ void __launch_bounds__(256) dead_copy_kernel(const int8_t* __restrict__ reach,
                                                        int8_t* __restrict__ next, uint32_t Vp,
                                                        const uint32_t* __restrict__ dead_list,
                                                        const unsigned long long* __restrict__ apart,
                                                        unsigned long long* apart_next, uint32_t W,
                                                        const uint32_t* __restrict__ nz,
                                                        uint32_t* __restrict__ nz_next) {
  __shared__ uint32_t s_occ[2];
  const uint32_t tiles_m = Vp / kBM, tiles_n = Vp / kBN, T = Vp / 128;
  const uint32_t tid = dead_list[blockIdx.x];
  const uint32_t group = tid / (kGroupM * tiles_n);
  const uint32_t first_m = group * kGroupM;
  const uint32_t gm = min((uint32_t)kGroupM, tiles_m - first_m);
  const uint32_t in_group = tid - group * kGroupM * tiles_n;
  const uint32_t m0 = (first_m + in_group % gm) * kBM;
  const uint32_t n0 = (in_group / gm) * kBN;
  // an all-zero R tile stays unwritten: its occupancy bit stays clear, so no reader
  // (TMA, epilogue, this copy) touches the stale bytes there
  if (!tile_nz(nz, T, m0 / 128, n0 / 128) && !tile_nz(nz, T, m0 / 128, n0 / 128 + 1)) return;
  if (threadIdx.x < 2) s_occ[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t idx = threadIdx.x; idx < kBM * (kBN / 16); idx += blockDim.x) {
    const uint32_t r = idx / (kBN / 16), c = (idx % (kBN / 16)) * 16;
    const uint64_t off = (uint64_t)(m0 + r) * Vp + n0 + c;
    const uint4 v = *reinterpret_cast<const uint4*>(reach + off);
    *reinterpret_cast<uint4*>(next + off) = v;
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
    uint32_t mask = 0;
#pragma unroll
    for (int b = 0; b < 16; ++b) mask |= (((w4[b >> 2] >> ((b & 3) * 8)) & 0xFFu) ? 1u : 0u) << b;
    const uint32_t j0 = n0 + c;
    const uint32_t abits = (j0 >> 6) < W ? (uint32_t)(apart[j0 >> 6] >> (j0 & 63)) & 0xFFFFu : 0u;
    if (mask & abits) atomicOr(&apart_next[(m0 + r) >> 6], 1ull << ((m0 + r) & 63));
    if (mask) atomicOr(&s_occ[c >> 7], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 2 && s_occ[threadIdx.x]) {
    const uint32_t b = (m0 / 128) * T + n0 / 128 + threadIdx.x;
    atomicOr(&nz_next[b >> 5], 1u << (b & 31));
  }
}

// 0/1 byte matrix init: row s = (q,r) gets 1 at (delta_a(q), delta_a(r)) for every a
__global__ void init_bytes_kernel(const uint32_t* __restrict__ delta, uint64_t n, uint32_t k,
                                  uint64_t V, uint64_t Vp, int8_t* __restrict__ R,
                                  uint32_t* __restrict__ nz) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < V; s += stride) {
    const uint64_t q = s / n, r = s % n;
    for (uint32_t a = 0; a < k; ++a) {
      const uint64_t c = (uint64_t)delta[a * n + q] * n + delta[a * n + r];
      R[s * Vp + c] = 1;
      const uint64_t b = (s / 128) * (Vp / 128) + c / 128;
      atomicOr(&nz[b >> 5], 1u << (b & 31));
    }
  }
}

// apart_next starts as apart (the reference ORs the pass-entry flag in)
__global__ void copy_words_kernel(const unsigned long long* a, unsigned long long* b, uint64_t W) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < W) b[i] = a[i];
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    DFM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (p == nullptr || q != cudaDriverEntryPointSuccess)
      throw Error(DFM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

CUtensorMap make_map(int8_t* base, uint64_t Vp) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {Vp, Vp};
  const cuuint64_t strides[1] = {Vp};
  const cuuint32_t box[2] = {128, 128};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(DFM_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

}  // namespace

bool usable(uint64_t V, int engine) {
  if (engine == DFM_TRANS_BIT) return false;
  if (engine == DFM_TRANS_TENSOR) return true;
  return V >= 1024;  // below one wave of tiles the bit engine is already latency-bound
}

TransTcState init(Ctx& ctx, const DevDfa& d, uint64_t V) {
  per_device_memo((const void*)square_kernel, ctx.device, [](const void*) {
    DFM_CUDA(cudaFuncSetAttribute(square_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemBytes));
    DFM_CUDA(cudaFuncSetAttribute(square_persistent_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    return 1;
  });
  TransTcState st;
  st.V = V;
  st.Vp = std::max<uint64_t>(256, ceil_div(V, 256) * 256);
  const uint64_t bytes = st.Vp * st.Vp;
  st.reach = ctx.slot_t<int8_t>("tc.R0", bytes);
  st.next = ctx.slot_t<int8_t>("tc.R1", bytes);
  DFM_CUDA(cudaMemsetAsync(st.reach, 0, bytes, ctx.stream));
  const uint64_t T = st.Vp / 128, nzw = ceil_div(T * T, 32);
  st.nz = ctx.slot_t<uint32_t>("tc.nz0", nzw);
  st.nz_next = ctx.slot_t<uint32_t>("tc.nz1", nzw);
  // DFM_TRANS_DENSE=1: every tile treated as occupied (the dense squaring; tests)
  const char* dense = getenv("DFM_TRANS_DENSE");
  DFM_CUDA(cudaMemsetAsync(st.nz, (dense && dense[0] == '1') ? 0xFF : 0x00, nzw * 4, ctx.stream));
  const unsigned grid =
      (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(V, 1), 256), ctx.num_sms * 16ull);
  init_bytes_kernel<<<grid, 256, 0, ctx.stream>>>(d.delta, d.n, d.k, V, st.Vp, st.reach, st.nz);
  DFM_LAUNCH_CHECK();
  return st;
}

void square_and_propagate(Ctx& ctx, TransTcState& st, const unsigned long long* apart,
                          unsigned long long* apart_next) {
  const uint64_t W = ceil_div(st.V, 64);
  copy_words_kernel<<<(unsigned)ceil_div(W, 256), 256, 0, ctx.stream>>>(apart, apart_next, W);
  DFM_LAUNCH_CHECK();
  const CUtensorMap map = make_map(st.reach, st.Vp);
  const uint64_t tiles = (st.Vp / kBM) * (st.Vp / kBN);
  const uint64_t T = st.Vp / 128, nzw = ceil_div(T * T, 32);
  const char* dense = getenv("DFM_TRANS_DENSE");
  DFM_CUDA(cudaMemsetAsync(st.nz_next, (dense && dense[0] == '1') ? 0xFF : 0x00, nzw * 4,
                           ctx.stream));
  {
    // int8 ops executed: 2 * 128 * 256 * 128 per live (output tile, K block) — the
    // dense pass would be 2 * Vp^3; K blocks of all-zero tiles are skipped
    auto* live = reinterpret_cast<unsigned long long*>(ctx.d_scalars + 56);
    uint32_t* counts = reinterpret_cast<uint32_t*>(ctx.d_scalars + 57);
    uint32_t* live_list = ctx.slot_t<uint32_t>("tc.live", tiles);
    uint32_t* dead_list = ctx.slot_t<uint32_t>("tc.dead", tiles);
    DFM_CUDA(cudaMemsetAsync(live, 0, 16, ctx.stream));  // live blocks + the two counts
    ProfScope p(ctx, "gemm", 0);
    tile_classify_kernel<<<(unsigned)std::min<uint64_t>(ceil_div(tiles, 256), ctx.num_sms * 8ull),
                           256, 0, ctx.stream>>>(st.nz, (uint32_t)st.Vp, live_list, dead_list,
                                                 counts);
    DFM_LAUNCH_CHECK();
    DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 57, counts, 8, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    const uint32_t n_live = (uint32_t)(ctx.h_scalars[57] & 0xFFFFFFFFu);
    const uint32_t n_dead = (uint32_t)(ctx.h_scalars[57] >> 32);
    if (n_dead)
      dead_copy_kernel<<<n_dead, 256, 0, ctx.stream>>>(st.reach, st.next, (uint32_t)st.Vp,
                                                      dead_list, apart, apart_next, (uint32_t)W,
                                                      st.nz, st.nz_next);
    DFM_LAUNCH_CHECK();
    if (n_live && persist_enabled())
      square_persistent_kernel<<<std::min<uint32_t>(n_live, (uint32_t)ctx.num_sms), kThreads,
                                 kSmemBytes, ctx.stream>>>(
          map, st.reach, st.next, apart, apart_next, (uint32_t)st.Vp, (uint32_t)W, st.nz,
          st.nz_next, live, live_list, n_live);
    else if (n_live)
      square_kernel<<<n_live, kThreads, kSmemBytes, ctx.stream>>>(
          map, st.reach, st.next, apart, apart_next, (uint32_t)st.Vp, (uint32_t)W, st.nz,
          st.nz_next, live, live_list);
    DFM_LAUNCH_CHECK();
    p.stop();
    DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 56, live, 8, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    p.bytes = ctx.h_scalars[56] * 2ull * kBM * kBN * kBK;
  }
  std::swap(st.reach, st.next);
  std::swap(st.nz, st.nz_next);
}

}  // namespace trans_tc
}  // namespace dfm
