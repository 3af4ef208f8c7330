// Blocked signature builder for sortPR (included by sortpr_hash.cu inside its
// anonymous namespace: uses ld_stream, load_id, mix64, the L2 policies).
//
// Problem: a pass needs, for every active state q, the ids of its k successors
// — n*k random 4-byte gathers.  Measured on B200 (tools/l2_bench.cu): random
// gathers are capped at ~285 G/s even when L2-resident (one L1 tag lookup per
// request per SM clock) and fall to ~40-50 G/s once the id array exceeds L2;
// shared-memory gathers run at ~700 G/s.
//
// Design (propagation blocking; delta is iteration-invariant, so the layout is
// built once per minimization and reused by every pass):
//   * target RANGES of kRs = 49152 states: a range's id slice (<= 192 KB even
//     at 32 bits) fits in shared memory; a transition's target is stored as a
//     16-bit offset inside its range (tgt, bucket order: range-major, then
//     source window);
//   * source WINDOWS of W states (W*k = 32768 transitions, one CTA tile);
//   * per pass, G (one CTA per group of ranges) loads the id slice into shared
//     memory and resolves every transition into that range with a shared-
//     memory gather, writing the id straight to the transition's position in
//     WINDOW-FLATTENED order (v, runs of ~16 consecutive positions);
//   * P (one CTA per window) streams the window's ids and tile slots (lsf) —
//     pure coalesced reads — into a shared-memory k x W tile and emits the
//     exact packed key (or hash + signature row) of every active state.
// HBM traffic per transition per pass: 2 (tgt) + 2 (lsf) + 2 x id width bytes;
// no random HBM access.  Layout: tgt/lsf u16 [T], off u32 [R*nW+1] (bucket
// start of sub-run (range j, window w), range-major), pre u16 [nW*R] (start of
// sub-run (j, w) inside window w's flattened order, window-major).
#pragma once

constexpr uint32_t kRs = 49152;          // states per target range (16-bit offsets)
constexpr uint32_t kMaxRanges = 4096;    // n <= 2.01e8 on the blocked path
#ifndef DFM_WIN_ELEMS  // (build-variant experiments: tools/build_variant.sh)
#define DFM_WIN_ELEMS 32768
#endif
constexpr uint32_t kWinElems = DFM_WIN_ELEMS;  // transitions per source window (u16 tile slots)
constexpr uint32_t kSliceBytes = 192u << 10;

struct Layout {
  uint32_t R = 0, W = 0, nW = 0, E = 0;  // E = W*k
  // bucket order is chunk-major: chunks of Wc windows (the first Wc*W states, ...)
  // each hold their transitions range-major, so a chunk's layout can be built as
  // soon as its rows are in HBM (pipelined upload); one chunk = plain range-major
  uint32_t Wc = 0, nC = 0;
  uint64_t n = 0, T = 0;
  uint32_t k = 0;
  // target states: == n on one GPU; the global count for a shard's rows (u32: fills
  // the padding after k, so the struct — a kernel parameter — keeps its size)
  uint32_t nt = 0;
  uint16_t* tgt = nullptr;
  uint16_t* lsf = nullptr;
  uint32_t* eidx = nullptr;    // [T] bucket position of each window-flattened transition
  uint32_t* off = nullptr;     // [nW][R] (+1): bucket start of sub-run (window w, range j)
  uint32_t* gb = nullptr;      // [nC][R]: bucket start of range j inside chunk c
  uint16_t* pre = nullptr;
  uint32_t* wstart = nullptr;  // [nW + 1] first active index of each window
  void* v = nullptr;           // [T] ids in window-flattened order (id bytes)
};

__device__ __forceinline__ uint32_t lanemask_lt_() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- layout build: per-window range histogram (w-major) + in-window prefix
__global__ void __launch_bounds__(512) lay_count_kernel(const uint32_t* __restrict__ delta, Layout L,
                                                        uint32_t* __restrict__ cnt_w,
                                                        uint32_t w_begin, uint32_t w_end) {
  extern __shared__ uint32_t s_h[];  // [R]
  __shared__ uint32_t s_warp[512 / 32 + 1];
  const uint64_t pol = policy_evict_first();
  for (uint32_t w = w_begin + blockIdx.x; w < w_end; w += gridDim.x) {
    for (uint32_t j = threadIdx.x; j < L.R; j += blockDim.x) s_h[j] = 0;
    __syncthreads();
    const uint64_t q0 = (uint64_t)w * L.W;
    const uint32_t wn = (uint32_t)(L.n - q0 < L.W ? L.n - q0 : L.W);
    // the window's k x wn transitions as one flat range (rows of wn coalesced
    // states): 16-byte loads when rows are 16-byte aligned, 4 in flight per thread
    const uint32_t ew = wn * L.k;
    if ((L.n & 3) == 0) {
      const uint32_t w4 = wn / 4, ew4 = ew / 4;
      for (uint32_t e0 = 0; e0 < ew4; e0 += 4 * blockDim.x) {
        uint4 t[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t e = e0 + u * blockDim.x + threadIdx.x;
          const uint32_t a = e / w4;
          if (e < ew4)
            asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                : "=r"(t[u].x), "=r"(t[u].y), "=r"(t[u].z), "=r"(t[u].w)
                : "l"(delta + a * L.n + q0 + 4 * (e - a * w4)), "l"(pol));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e0 + u * blockDim.x + threadIdx.x < ew4) {
            atomicAdd(&s_h[t[u].x / kRs], 1u);
            atomicAdd(&s_h[t[u].y / kRs], 1u);
            atomicAdd(&s_h[t[u].z / kRs], 1u);
            atomicAdd(&s_h[t[u].w / kRs], 1u);
          }
      }
    } else {
      for (uint32_t e0 = 0; e0 < ew; e0 += 8 * blockDim.x) {
        uint32_t t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t e = e0 + u * blockDim.x + threadIdx.x;
          const uint32_t a = e / wn;
          t[u] = e < ew ? ld_stream(delta + a * L.n + q0 + (e - a * wn), pol) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e0 + u * blockDim.x + threadIdx.x < ew) atomicAdd(&s_h[t[u] / kRs], 1u);
      }
    }
    __syncthreads();
    // counts (w-major, transposed later for the bucket scan) + in-window prefix
    constexpr uint32_t kPer = kMaxRanges / 512;
    const uint32_t j0 = threadIdx.x * kPer;
    uint32_t c[kPer], sum = 0;
#pragma unroll
    for (uint32_t u = 0; u < kPer; ++u) {
      c[u] = j0 + u < L.R ? s_h[j0 + u] : 0u;
      sum += c[u];
    }
    uint32_t tot;
    uint32_t run = prims::block_exclusive_sum<512>(sum, s_warp, &tot);
    // stage the in-window prefixes in shared memory (after the counts in s_h) so that
    // both rows leave with coalesced stores (a thread's 8 consecutive entries would
    // touch 8 sectors per warp instruction)
    uint16_t* s_pre_w = reinterpret_cast<uint16_t*>(s_h + L.R);
#pragma unroll
    for (uint32_t u = 0; u < kPer; ++u)
      if (j0 + u < L.R) {
        s_pre_w[j0 + u] = (uint16_t)run;
        run += c[u];
      }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < L.R; j += blockDim.x) {
      cnt_w[(uint64_t)w * L.R + j] = s_h[j];
      L.pre[(uint64_t)w * L.R + j] = s_pre_w[j];
    }
    __syncthreads();
  }
}

// [rows][cols] -> [cols][rows], 32x32 tiles
__global__ void lay_transpose_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                     uint32_t rows, uint32_t cols) {
  __shared__ uint32_t t[32][33];
  const uint32_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y) {
    const uint32_t r = r0 + y, c = c0 + threadIdx.x;
    if (r < rows && c < cols) t[y][threadIdx.x] = in[(uint64_t)r * cols + c];
  }
  __syncthreads();
  for (uint32_t y = threadIdx.y; y < 32; y += blockDim.y) {
    const uint32_t c = c0 + y, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[(uint64_t)c * rows + r] = t[threadIdx.x][y];
  }
}

struct LayOffIn {
  const uint32_t* cnt;
  __device__ uint32_t operator()(uint64_t i) const { return cnt[i]; }
};
// one chunk's cells in (range j, window w0 + x) order, x < wc -> off(w, j), absolute
// (window-major, so the per-window kernels read a window's R starts coalesced), and
// the chunk's range starts for the gather kernel
struct LayOffOut {
  uint32_t* off;
  uint32_t* gb;
  uint32_t R, wc, w0, ch;
  uint32_t base;     // transitions of the chunks before
  uint64_t count;    // cells of this chunk (R * wc)
  uint64_t total;    // final chunk: off[nW * R] = T (else ~0)
  __device__ void operator()(uint64_t i, uint32_t excl, uint32_t v) const {
    const uint64_t j = i / wc, x = i - j * wc;
    off[(w0 + x) * (uint64_t)R + j] = base + excl;
    if (x == 0) gb[(uint64_t)ch * R + j] = base + excl;
    if (total != ~0ull && i + 1 == count) off[total] = base + excl + v;
  }
};

// ---- layout build: bucket every transition (tgt) and its tile slot (lsf).
// Both are staged in shared memory in the window's flattened order (sub-run j
// at pre(w, j)); lsf and the bucket positions (eidx) leave as coalesced chunks and
// every tgt goes to its bucket position off(w, j) + rank.
__device__ __forceinline__ void lay_stage(uint32_t t, uint32_t a, uint32_t x, uint32_t W,
                                          uint32_t* s_cur, const uint32_t* s_pre,
                                          uint32_t* s_tj, uint16_t* s_lsf) {
  const uint32_t j = t / kRs;
  const uint32_t f = s_pre[j] + atomicAdd(&s_cur[j], 1u);
  s_tj[f] = (t - j * kRs) | (j << 16);  // target offset (16 bits) and range (< 4096)
  s_lsf[f] = (uint16_t)(a * W + x);
}

__global__ void __launch_bounds__(1024) lay_scatter_kernel(const uint32_t* __restrict__ delta,
                                                           Layout L, uint32_t w_begin,
                                                           uint32_t w_end) {
  // s_cur[R], s_off[R], s_pre[R+1], then u32 s_tj[E] (target offset | range << 16),
  // u16 s_lsf[E]: two shared stores per staged transition
  extern __shared__ uint32_t s_lay[];
  uint32_t* s_cur = s_lay;
  uint32_t* s_off = s_lay + L.R;
  uint32_t* s_pre = s_lay + 2 * L.R;
  uint32_t* s_tj = s_lay + 3 * L.R + 1;
  uint16_t* s_lsf = reinterpret_cast<uint16_t*>(s_tj + L.E);
  const uint64_t pol = policy_evict_first();
  // the next window's sub-run starts are loaded while the current one is written out
  constexpr uint32_t kPf = kMaxRanges / 1024;
  uint32_t pf_off[kPf], pf_pre[kPf];
  auto prefetch = [&](uint32_t w) {
#pragma unroll
    for (uint32_t u = 0; u < kPf; ++u) {
      const uint32_t j = threadIdx.x + u * blockDim.x;
      if (w < w_end && j < L.R) {
        pf_off[u] = L.off[(uint64_t)w * L.R + j];
        pf_pre[u] = L.pre[(uint64_t)w * L.R + j];
      }
    }
  };
  prefetch(w_begin + blockIdx.x);
  for (uint32_t w = w_begin + blockIdx.x; w < w_end; w += gridDim.x) {
    const uint64_t q0 = (uint64_t)w * L.W;
    const uint32_t wn = (uint32_t)(L.n - q0 < L.W ? L.n - q0 : L.W);
    const uint32_t ew = wn * L.k;
#pragma unroll
    for (uint32_t u = 0; u < kPf; ++u) {
      const uint32_t j = threadIdx.x + u * blockDim.x;
      if (j < L.R) {
        s_cur[j] = 0;
        s_off[j] = pf_off[u];
        s_pre[j] = pf_pre[u];
      }
    }
    if (threadIdx.x == 0) s_pre[L.R] = ew;
    __syncthreads();
    if ((L.n & 3) == 0) {  // 16-byte row loads
      const uint32_t w4 = wn / 4, ew4 = ew / 4;
      for (uint32_t e0 = 0; e0 < ew4; e0 += 2 * blockDim.x) {
        uint4 t[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t e = e0 + u * blockDim.x + threadIdx.x;
          const uint32_t a = e / w4;
          if (e < ew4)
            asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                : "=r"(t[u].x), "=r"(t[u].y), "=r"(t[u].z), "=r"(t[u].w)
                : "l"(delta + a * L.n + q0 + 4 * (e - a * w4)), "l"(pol));
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t e = e0 + u * blockDim.x + threadIdx.x;
          if (e < ew4) {
            const uint32_t a = e / w4, x = 4 * (e - a * w4);
            lay_stage(t[u].x, a, x, L.W, s_cur, s_pre, s_tj, s_lsf);
            lay_stage(t[u].y, a, x + 1, L.W, s_cur, s_pre, s_tj, s_lsf);
            lay_stage(t[u].z, a, x + 2, L.W, s_cur, s_pre, s_tj, s_lsf);
            lay_stage(t[u].w, a, x + 3, L.W, s_cur, s_pre, s_tj, s_lsf);
          }
        }
      }
    } else {
      for (uint32_t e0 = 0; e0 < ew; e0 += 8 * blockDim.x) {
        uint32_t t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t e = e0 + u * blockDim.x + threadIdx.x;
          const uint32_t a = e / wn;
          t[u] = e < ew ? ld_stream(delta + a * L.n + q0 + (e - a * wn), pol) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t e = e0 + u * blockDim.x + threadIdx.x;
          if (e < ew) {
            const uint32_t a = e / wn;
            lay_stage(t[u], a, e - a * wn, L.W, s_cur, s_pre, s_tj, s_lsf);
          }
        }
      }
    }
    __syncthreads();
    prefetch(w + gridDim.x);
    // bucket position of flattened slot f of sub-run j = off(j, w) - pre(w, j) + f
    for (uint32_t j = threadIdx.x; j < L.R; j += blockDim.x) s_off[j] -= s_pre[j];
    __syncthreads();
    const uint64_t fb = (uint64_t)w * L.E;
    for (uint32_t f = threadIdx.x; f < ew; f += blockDim.x) {
      const uint32_t tj = s_tj[f];
      const uint32_t e = s_off[tj >> 16] + f;
      L.lsf[fb + f] = s_lsf[f];
      L.eidx[fb + f] = e;
      L.tgt[e] = (uint16_t)(tj & 0xFFFFu);
    }
    __syncthreads();
  }
}

// first active index of every window (act ascending); wstart[nW] = m
__global__ void lay_wstart_kernel(const uint32_t* __restrict__ act, uint64_t m, uint32_t W,
                                  uint32_t nW, uint32_t* __restrict__ wstart) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += stride) {
    const int64_t w = i < m ? (int64_t)(act[i] / W) : (int64_t)nW;
    const int64_t wp = i > 0 ? (int64_t)(act[i - 1] / W) : -1;
    for (int64_t x = wp + 1; x <= w; ++x) wstart[x] = (uint32_t)i;
  }
}

// id bytes in the flattened buffer: 1 for mirrors of <= 8 bits
template <int kIdBits>
struct IdT {
  using type = uint8_t;
};
template <>
struct IdT<16> {
  using type = uint16_t;
};
template <>
struct IdT<32> {
  using type = uint32_t;
};

template <int kIdBits>
__device__ __forceinline__ uint32_t slice_id(const uint32_t* s, uint32_t x) {
  if (kIdBits == 1) return (s[x >> 5] >> (x & 31)) & 1u;
  if (kIdBits == 4) return (s[x >> 3] >> ((x & 7) * 4)) & 0xFu;
  if (kIdBits == 8) return reinterpret_cast<const uint8_t*>(s)[x];
  if (kIdBits == 16) return reinterpret_cast<const uint16_t*>(s)[x];
  return s[x];
}

// ---- per pass G: shared-memory gathers, one CTA per group of c ranges; ids
// are written in bucket order (coalesced)
template <int kIdBits>
__global__ void __launch_bounds__(1024) lay_gather_kernel(Layout L, const uint32_t* __restrict__ ids,
                                                          uint32_t c) {
  using V = typename IdT<kIdBits>::type;
  extern __shared__ uint4 s_slice4[];
  __shared__ uint32_t s_bound[33];
  uint32_t* s_slice = reinterpret_cast<uint32_t*>(s_slice4);
  V* __restrict__ vout = static_cast<V*>(L.v);
  const uint64_t pol = policy_evict_first();
  const uint32_t groups = (L.R + c - 1) / c;
  for (uint32_t g = blockIdx.x; g < groups; g += gridDim.x) {
    const uint32_t j0 = g * c, j1 = min(L.R, j0 + c);
    // id slice of states [j0*kRs, min(n, j1*kRs)): words of the packed mirror
    const uint64_t st0 = (uint64_t)j0 * kRs;
    const uint64_t st1 = min((uint64_t)L.nt, (uint64_t)j1 * kRs);
    const uint64_t w0 = st0 * kIdBits / 32, w1 = (st1 * kIdBits + 31) / 32;
    const uint32_t nwords = (uint32_t)(w1 - w0);
    const uint4* src4 = reinterpret_cast<const uint4*>(ids + w0);  // 16-byte aligned: kRs*bits/8
    for (uint32_t i = threadIdx.x; i < nwords / 4; i += blockDim.x) s_slice4[i] = __ldg(src4 + i);
    for (uint32_t i = (nwords / 4) * 4 + threadIdx.x; i < nwords; i += blockDim.x)
      s_slice[i] = __ldg(ids + w0 + i);
    for (uint32_t ch = 0; ch < L.nC; ++ch) {
      // bucket starts of ranges j0..j1 inside chunk ch (its end after the last range)
      if (threadIdx.x <= j1 - j0) {
        const uint32_t j = j0 + threadIdx.x;
        s_bound[threadIdx.x] =
            j < L.R ? L.gb[(uint64_t)ch * L.R + j]
                    : (ch + 1 < L.nC ? (ch + 1) * L.Wc * L.E : (uint32_t)L.T);
      }
      __syncthreads();
      // range by range (no per-element range search).  The aligned body moves 8
      // targets per 16-byte load and 8 ids per vector store (two groups in flight
      // per thread); the unaligned head and tail go element by element
      for (uint32_t r = 0; r < j1 - j0; ++r) {
        const uint32_t start = s_bound[r], end = s_bound[r + 1];
        const uint32_t* sl = s_slice;
        const uint32_t sb = r * kRs;
        const uint32_t g0 = (start + 7) / 8, g1 = end / 8;  // whole 8-element groups
        const uint32_t head_end = g0 < g1 ? g0 * 8 : end;
        for (uint32_t e = start + threadIdx.x; e < head_end; e += blockDim.x)
          vout[e] = (V)slice_id<kIdBits>(sl, sb + L.tgt[e]);
        if (g0 < g1) {
          for (uint32_t e = g1 * 8 + threadIdx.x; e < end; e += blockDim.x)
            vout[e] = (V)slice_id<kIdBits>(sl, sb + L.tgt[e]);
          const uint4* t4 = reinterpret_cast<const uint4*>(L.tgt);
          for (uint32_t g = g0 + threadIdx.x; g < g1; g += 2 * blockDim.x) {
            uint4 tv[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint32_t gg = g + u * blockDim.x;
              if (gg < g1)
                asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                    : "=r"(tv[u].x), "=r"(tv[u].y), "=r"(tv[u].z), "=r"(tv[u].w)
                    : "l"(t4 + gg), "l"(pol));
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint32_t gg = g + u * blockDim.x;
              if (gg >= g1) continue;
              const uint32_t w4[4] = {tv[u].x, tv[u].y, tv[u].z, tv[u].w};
              uint32_t id[8];
#pragma unroll
              for (int b = 0; b < 8; ++b)
                id[b] = slice_id<kIdBits>(sl, sb + ((w4[b >> 1] >> ((b & 1) * 16)) & 0xFFFFu));
              if (sizeof(V) == 4) {
                uint4* o = reinterpret_cast<uint4*>(vout) + 2 * (uint64_t)gg;
                o[0] = make_uint4(id[0], id[1], id[2], id[3]);
                o[1] = make_uint4(id[4], id[5], id[6], id[7]);
              } else if (sizeof(V) == 2) {
                reinterpret_cast<uint4*>(vout)[gg] =
                    make_uint4(id[0] | id[1] << 16, id[2] | id[3] << 16, id[4] | id[5] << 16,
                               id[6] | id[7] << 16);
              } else {
                reinterpret_cast<uint2*>(vout)[gg] =
                    make_uint2(id[0] | id[1] << 8 | id[2] << 16 | id[3] << 24,
                               id[4] | id[5] << 8 | id[6] << 16 | id[7] << 24);
              }
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

struct SigParams {
  Layout L;
  const uint32_t* wstart;  // nullptr: every state active (act == identity)
  const uint32_t* act;
  const uint32_t* block;
  int w;
  uint64_t seed;
  unsigned long long* keys;
  uint32_t* sig;  // hashed: signature rows (stride row), else nullptr
  uint32_t row;
  // partitioned grouping (sortpr_group.cuh): packed keys leave as a bijective mix,
  // and vals[i] = i | lead << 31
  uint32_t* vals;
  const uint8_t* lead;
  uint32_t* present;  // direct keys: bitmap of the keys present, words interleaved with
                      // their exclusive popcounts (rank-compacted table)
  uint32_t tile_bytes;  // shared tile size (16-byte multiple)
};

// ---- per pass P: one CTA per window, streamed ids -> smem tile -> keys
// narrow tiles (<= 64 KB) fit two CTAs per SM: cap registers at 32 for that
// kTile24: 32-bit ids below 2^24 kept as 3 bytes per tile entry (96 KB instead of
// 128 KB: two CTAs per SM, so one window's loads overlap the other's key phase)
template <int kIdBits, int kK, bool kHashed, bool kTile24 = false>
__global__ void __launch_bounds__(1024, (kIdBits <= 16 || kTile24) ? 2 : 1)
    lay_sig_kernel(SigParams p) {
  using V = typename IdT<kIdBits>::type;
  extern __shared__ uint4 s_tile4[];
  V* s_tile = reinterpret_cast<V*>(s_tile4);  // [k][W]
  uint8_t* s_t8 = reinterpret_cast<uint8_t*>(s_tile4);
  auto tput = [&](uint32_t slot, V x) {
    if (kTile24) {
      s_t8[3 * slot] = (uint8_t)x;
      s_t8[3 * slot + 1] = (uint8_t)(x >> 8);
      s_t8[3 * slot + 2] = (uint8_t)(x >> 16);
    } else {
      s_tile[slot] = x;
    }
  };
  auto tget = [&](uint32_t slot) -> uint32_t {
    if (kTile24)
      return (uint32_t)s_t8[3 * slot] | (uint32_t)s_t8[3 * slot + 1] << 8 |
             (uint32_t)s_t8[3 * slot + 2] << 16;
    return (uint32_t)s_tile[slot];
  };
  const Layout& L = p.L;
  const uint32_t k = kK > 0 ? (uint32_t)kK : L.k;
  const V* __restrict__ vin = static_cast<const V*>(L.v);
  const uint64_t pol = policy_evict_first();
  for (uint32_t w = blockIdx.x; w < L.nW; w += gridDim.x) {
    const uint64_t q0 = (uint64_t)w * L.W;
    const uint32_t wn = (uint32_t)(L.n - q0 < L.W ? L.n - q0 : L.W);
    const uint32_t ew = wn * k;
    const uint64_t fb = (uint64_t)w * L.E;
    // lane-consecutive transitions (coalesced slot / position loads; the ids come
    // in runs of ~16 per sub-run), U in flight per thread (fewer under the 32-register
    // cap of the two-CTA narrow tiles)
    constexpr int U = (kIdBits <= 16 || kTile24) ? 4 : 8;
    for (uint32_t f0 = threadIdx.x; f0 < ew; f0 += U * blockDim.x) {
      uint32_t sl[U], ee[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t f = f0 + u * blockDim.x;
        sl[u] = 0;
        ee[u] = 0;
        if (f < ew) {
          asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
              : "=r"(sl[u]) : "l"(L.lsf + fb + f), "l"(pol));
          asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
              : "=r"(ee[u]) : "l"(L.eidx + fb + f), "l"(pol));
        }
      }
      V x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = (f0 + u * blockDim.x < ew) ? vin[ee[u]] : (V)0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (f0 + u * blockDim.x < ew) tput(sl[u], x[u]);
    }
    __syncthreads();
    const uint64_t i0 = p.wstart ? p.wstart[w] : q0;
    const uint64_t i1 = p.wstart ? p.wstart[w + 1] : q0 + wn;
    // KU states per thread: their own-block loads are in flight together (one state
    // at a time left every warp waiting a full memory latency per state)
    constexpr int KU = kHashed ? 1 : 4;
    for (uint64_t ib = i0 + threadIdx.x; ib < i1; ib += KU * blockDim.x) {
      uint32_t qq[KU], bb[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const uint64_t i = ib + (uint64_t)u * blockDim.x;
        qq[u] = i < i1 ? (p.act ? p.act[i] : (uint32_t)i) : 0u;
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) bb[u] = ib + (uint64_t)u * blockDim.x < i1 ? p.block[qq[u]] : 0u;
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const uint64_t i = ib + (uint64_t)u * blockDim.x;
        if (i >= i1) break;
        const uint32_t q = qq[u];
        const uint32_t x = (uint32_t)(q - q0);
        const uint32_t b = bb[u];
        if (!kHashed) {
          unsigned long long key = b;
#pragma unroll
          for (uint32_t a = 0; a < (kK > 0 ? (uint32_t)kK : k); ++a)
            key = (key << p.w) | tget(a * L.W + x);
          p.keys[i] = p.vals ? mix64(key ^ p.seed) : key;
          if (p.present) {  // test before set: most keys of a dense pass are repeats
            const uint32_t bit = 1u << (key & 31);
            uint32_t* word = p.present + 2 * (key >> 5);  // (interleaved with the prefixes)
            if (!(prims::ld_hint_u32(word) & bit)) atomicOr(word, bit);
          }
        } else {
          uint32_t* row = p.sig + i * (uint64_t)p.row;
          row[0] = b;
          unsigned long long h = mix64(p.seed * kGolden + b);
#pragma unroll
          for (uint32_t a = 0; a < (kK > 0 ? (uint32_t)kK : k); ++a) {
            const uint32_t s = tget(a * L.W + x);
            row[a + 1] = s;
            h = mix64(h + kGolden + s);
          }
          p.keys[i] = weak(h, p.seed);
        }
        if (p.vals) p.vals[i] = (uint32_t)i | ((uint32_t)p.lead[q] << 31);
      }
    }
    __syncthreads();
  }
}
