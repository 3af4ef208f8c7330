// Post-/pre-processing next to the minimize path, on
// the device:
//   quotient           core.hpp:256-290  — the automaton induced on the blocks of a
//                                           canonical partition, with the reference's
//                                           validation and error messages;
//   remove_unreachable core.hpp:152-187  — breadth-first reachability from the initial
//                                           state, dense renumbering in ascending order.
#include <algorithm>
#include <string>

#include <cooperative_groups.h>

#include "prims.cuh"

namespace cg = cooperative_groups;

namespace dfm {
namespace {

unsigned grid_for(const Ctx& ctx, uint64_t items) {
  return (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(items, 1), 256),
                                      (uint64_t)ctx.num_sms * 16);
}

// ------------------------------------------------------------------ quotient
// representative of every block = its minimum state (the first state of the block in
// the reference's ascending scan, core.hpp:270); labels >= nb flag a non-canonical input
__global__ void q_rep_kernel(const uint32_t* __restrict__ block, uint64_t n, uint32_t nb,
                             uint32_t* __restrict__ rep, unsigned long long* flags) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t qb = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); qb < n;
       qb += stride) {
    const uint64_t q = qb + (threadIdx.x & 31);
    const bool inr = q < n;
    const uint32_t b = inr ? block[q] : 0u;
    const bool ok = inr && b < nb;
    if (inr && !ok) atomicOr(flags, 1ull);
    // lanes hold ascending states: the lowest lane of each label group is its minimum
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      const uint32_t peers = __match_any_sync(m, b);
      if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicMin(&rep[b], (uint32_t)q);
    }
  }
}

// canonical (core.hpp:259-262) <=> every label used and first occurrences ascending
__global__ void q_canon_kernel(const uint32_t* __restrict__ rep, uint32_t nb,
                               unsigned long long* flags) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride)
    if (rep[b] == 0xFFFFFFFFu || (b > 0 && rep[b - 1] >= rep[b])) atomicOr(flags, 1ull);
}

// quotient rows from the representatives (core.hpp:270-277)
__global__ void q_rows_kernel(const uint32_t* __restrict__ delta, const uint8_t* __restrict__ acc,
                              uint64_t n, uint32_t k, const uint32_t* __restrict__ block,
                              const uint32_t* __restrict__ rep, uint32_t nb,
                              uint32_t* __restrict__ out_delta, uint8_t* __restrict__ out_acc) {
  const uint64_t total = (uint64_t)nb * (k + 1);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const uint64_t a = i / nb, b = i - a * nb;
    const uint32_t r = rep[b];
    if (a < k) out_delta[i] = block[delta[a * n + r]];
    else out_acc[b] = acc[r];
  }
}

// every other state must agree (core.hpp:279-286): the first violation in ascending
// state order, acceptance before letters, as (q << 32 | code), code 0 = acceptance,
// a + 1 = letter a
__global__ void q_check_kernel(const uint32_t* __restrict__ delta, const uint8_t* __restrict__ acc,
                               uint64_t n, uint32_t k, const uint32_t* __restrict__ block,
                               const uint32_t* __restrict__ out_delta,
                               const uint8_t* __restrict__ out_acc, uint32_t nb,
                               unsigned long long* first_bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    const uint32_t b = block[q];
    uint32_t code = 0xFFFFFFFFu;
    if (acc[q] != out_acc[b]) {
      code = 0;
    } else {
      for (uint32_t a = 0; a < k; ++a)
        if (block[delta[(uint64_t)a * n + q]] != out_delta[(uint64_t)a * nb + b]) {
          code = a + 1;
          break;
        }
    }
    if (code != 0xFFFFFFFFu) atomicMin(first_bad, (q << 32) | code);
  }
}

// ------------------------------------------------------------------ remove_unreachable
// Level-synchronous BFS in one cooperative launch: each level expands the frontier,
// claims unseen targets in a bitmap (atomicOr) and appends them with one atomic per
// warp; counters rotate over three slots so a single grid barrier per level suffices.
struct BfsArgs {
  const uint32_t* rows;
  uint64_t n, letters;
  uint32_t* seen;  // bitmap
  uint32_t* f0;
  uint32_t* f1;
  uint32_t* cnt;  // [3]
  uint64_t level0;
  uint32_t max_levels;
  uint32_t* out;  // [0] levels run, [1] finished
};

__global__ void __launch_bounds__(512) bfs_kernel(BfsArgs a) {
  cg::grid_group g = cg::this_grid();
  const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t L = 0;
  bool done = false;
  for (; L < a.max_levels; ++L) {
    const uint64_t lvl = a.level0 + L;
    const uint32_t cur_c = (uint32_t)(lvl % 3), nxt_c = (uint32_t)((lvl + 1) % 3),
                   clr_c = (uint32_t)((lvl + 2) % 3);
    const uint32_t* cur_f = (lvl & 1) ? a.f1 : a.f0;
    uint32_t* nxt_f = (lvl & 1) ? a.f0 : a.f1;
    const uint32_t size = prims::ld_relaxed_u32(&a.cnt[cur_c]);
    if (size == 0) {
      done = true;
      break;
    }
    if (gt == 0) a.cnt[clr_c] = 0;
    for (uint64_t ib = gt - lane; ib < size; ib += nth) {
      const uint64_t i = ib + lane;
      const bool valid = i < size;
      const uint32_t q = valid ? cur_f[i] : 0u;
      for (uint64_t c = 0; c < a.letters; ++c) {
        bool claim = false;
        uint32_t t = 0;
        if (valid) {
          t = a.rows[c * a.n + q];
          const uint32_t bit = 1u << (t & 31);
          claim = (atomicOr(&a.seen[t >> 5], bit) & bit) == 0u;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, claim);
        if (m) {
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(&a.cnt[nxt_c], (uint32_t)__popc(m));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (claim) nxt_f[base + __popc(m & ((1u << lane) - 1u))] = t;
        }
      }
    }
    g.sync();
  }
  if (gt == 0) {
    a.out[0] = L;
    a.out[1] = done ? 1u : 0u;
  }
}

struct SeenIn {
  const uint32_t* seen;
  __device__ uint32_t operator()(uint64_t q) const { return (seen[q >> 5] >> (q & 31)) & 1u; }
};
struct SeenOut {
  uint32_t* ren;
  __device__ void operator()(uint64_t q, uint32_t excl, uint32_t) const { ren[q] = excl; }
};

// induced rows on the kept states (core.hpp:172-186)
__global__ void keep_rows_kernel(const uint32_t* __restrict__ delta, const uint8_t* __restrict__ acc,
                                 uint64_t n, uint32_t k, const uint32_t* __restrict__ seen,
                                 const uint32_t* __restrict__ ren, uint32_t kept,
                                 uint32_t* __restrict__ out_delta, uint8_t* __restrict__ out_acc) {
  const uint64_t total = n * (k + 1);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const uint64_t a = i / n, q = i - a * n;
    if (!((seen[q >> 5] >> (q & 31)) & 1u)) continue;
    if (a < k) out_delta[a * kept + ren[q]] = ren[delta[i]];
    else out_acc[ren[q]] = acc[q];
  }
}

}  // namespace

DevDfa quotient_dev(Ctx& ctx, const DevDfa& d, const uint32_t* block, uint32_t nb) {
  const uint64_t n = d.n;
  const uint32_t k = d.k;
  auto* flags = reinterpret_cast<unsigned long long*>(ctx.d_scalars + 44);
  auto* first_bad = reinterpret_cast<unsigned long long*>(ctx.d_scalars + 45);
  DFM_CUDA(cudaMemsetAsync(flags, 0, 8, ctx.stream));
  DFM_CUDA(cudaMemsetAsync(first_bad, 0xFF, 8, ctx.stream));
  uint32_t* rep = ctx.slot_t<uint32_t>("qt.rep", std::max<uint32_t>(nb, 1));
  DFM_CUDA(cudaMemsetAsync(rep, 0xFF, (uint64_t)std::max<uint32_t>(nb, 1) * 4, ctx.stream));
  {
    ProfScope p(ctx, "quotient", n * 4 + nb * 8ull);
    q_rep_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(block, n, nb, rep, flags);
    DFM_LAUNCH_CHECK();
    q_canon_kernel<<<grid_for(ctx, nb), 256, 0, ctx.stream>>>(rep, nb, flags);
    DFM_LAUNCH_CHECK();
  }
  DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 44, flags, 8, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  if (ctx.h_scalars[44] != 0 || (n > 0 && nb == 0))
    throw Error(DFM_ERR_INVALID, "partition is not in canonical form");
  DevDfa out;
  out.n = nb;
  out.k = k;
  out.owns = true;
  DFM_CUDA(cudaMalloc(&out.delta, std::max<uint64_t>((uint64_t)nb * k, 1) * 4));
  DFM_CUDA(cudaMalloc(&out.acc, std::max<uint32_t>(nb, 1)));
  try {
    {
      // rows: rep 4 + delta gather 4 + block gather 4 + write 4 per entry
      ProfScope p(ctx, "quotient", (uint64_t)nb * (k + 1) * 16 + n * (4ull * k + 2));
      q_rows_kernel<<<grid_for(ctx, (uint64_t)nb * (k + 1)), 256, 0, ctx.stream>>>(
          d.delta, d.acc, n, k, block, rep, nb, out.delta, out.acc);
      DFM_LAUNCH_CHECK();
      q_check_kernel<<<grid_for(ctx, n), 256, 0, ctx.stream>>>(d.delta, d.acc, n, k, block,
                                                                out.delta, out.acc, nb, first_bad);
      DFM_LAUNCH_CHECK();
    }
    DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 45, first_bad, 8, cudaMemcpyDeviceToHost, ctx.stream));
    uint32_t init_label = 0;
    DFM_CUDA(cudaMemcpyAsync(&init_label, block + d.initial, 4, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    const unsigned long long fb = ctx.h_scalars[45];
    if (fb != ~0ull) {
      const uint32_t q = (uint32_t)(fb >> 32), code = (uint32_t)fb;
      uint32_t b = 0;
      DFM_CUDA(cudaMemcpy(&b, block + q, 4, cudaMemcpyDeviceToHost));
      if (code == 0)
        throw Error(DFM_ERR_INVALID, "inconsistent partition: block " + std::to_string(b) +
                                         " mixes accepting and rejecting states");
      throw Error(DFM_ERR_INVALID, "inconsistent partition: block " + std::to_string(b) +
                                       " splits on letter " + std::to_string(code - 1));
    }
    out.initial = init_label;
  } catch (...) {
    cudaFree(out.delta);
    cudaFree(out.acc);
    throw;
  }
  return out;
}

DevDfa remove_unreachable_dev(Ctx& ctx, const DevDfa& d) {
  const uint64_t n = d.n;
  const uint32_t k = d.k;
  const uint64_t words = ceil_div(std::max<uint64_t>(n, 1), 32);
  uint32_t* seen = ctx.slot_t<uint32_t>("ur.seen", words);
  uint32_t* f0 = ctx.slot_t<uint32_t>("ur.f0", std::max<uint64_t>(n, 1));
  uint32_t* f1 = ctx.slot_t<uint32_t>("ur.f1", std::max<uint64_t>(n, 1));
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ctx.d_scalars + 46);   // [3]
  uint32_t* bout = reinterpret_cast<uint32_t*>(ctx.d_scalars + 48);  // [2]
  DFM_CUDA(cudaMemsetAsync(seen, 0, words * 4, ctx.stream));
  // seed the search: seen[initial], frontier {initial}, cnt = {1, 0, 0}
  const uint32_t init = d.initial;
  const uint32_t seed_bits = 1u << (init & 31);
  DFM_CUDA(cudaMemcpyAsync(seen + (init >> 5), &seed_bits, 4, cudaMemcpyHostToDevice, ctx.stream));
  DFM_CUDA(cudaMemcpyAsync(f0, &init, 4, cudaMemcpyHostToDevice, ctx.stream));
  const uint32_t c3[3] = {1, 0, 0};
  DFM_CUDA(cudaMemcpyAsync(cnt, c3, 12, cudaMemcpyHostToDevice, ctx.stream));
  int per_sm = 0;
  DFM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_kernel, 512, 0));
  const unsigned grid = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>((uint64_t)per_sm * ctx.num_sms, ceil_div(n, 512)));
  const uint32_t* rows = d.delta;
  uint64_t letters = k;
  uint64_t level = 0;
  bool expanded = false;
  // deep searches (chains, combs) switch to the doubled alphabet a^(2^j) of
  // min_transpr.hpp:59-85 after kDeep levels: the reachable set is the same, the
  // number of levels drops to ~log2(n) for single-letter paths
  constexpr uint32_t kDeep = 64;
  while (true) {
    BfsArgs ba{rows, n, letters, seen, f0, f1, cnt, level, expanded ? (1u << 20) : kDeep, bout};
    void* args[] = {&ba};
    {
      ProfScope p(ctx, "bfs", 0);
      if (letters > 0)
        DFM_CUDA(cudaLaunchCooperativeKernel((const void*)bfs_kernel, grid, 512, args, 0,
                                             ctx.stream));
      DFM_LAUNCH_CHECK();
    }
    uint32_t h[2] = {0, 1};
    if (letters > 0) {
      DFM_CUDA(cudaMemcpyAsync(h, bout, 8, cudaMemcpyDeviceToHost, ctx.stream));
      ctx.sync();
    }
    level += h[0];
    if (h[1]) break;
    if (!expanded) {
      expanded = true;
      size_t free_b = 0, total_b = 0;
      DFM_CUDA(cudaMemGetInfo(&free_b, &total_b));
      if (dfm_expand_required_bytes(d.n, d.k) < free_b / 2) {  // else: plain levels to the end
        const uint32_t levels = dfm_power_levels(d.n);
        rows = expand_alphabet_dev(ctx, d, levels);
        letters = (uint64_t)levels * k;
      }
    }
  }
  // dense renumbering in ascending original order (core.hpp:167-171)
  uint32_t* ren = ctx.slot_t<uint32_t>("ur.ren", std::max<uint64_t>(n, 1));
  auto* total = ctx.d_scalars + 50;
  prims::lookback_scan(ctx, "sc.ur", n, SeenIn{seen}, SeenOut{ren}, total);
  DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 50, total, 8, cudaMemcpyDeviceToHost, ctx.stream));
  uint32_t init_ren = 0;
  DFM_CUDA(cudaMemcpyAsync(&init_ren, ren + init, 4, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  const uint32_t kept = (uint32_t)ctx.h_scalars[50];
  DevDfa out;
  out.n = kept;
  out.k = k;
  out.initial = init_ren;
  out.owns = true;
  DFM_CUDA(cudaMalloc(&out.delta, std::max<uint64_t>((uint64_t)kept * k, 1) * 4));
  DFM_CUDA(cudaMalloc(&out.acc, std::max<uint32_t>(kept, 1)));
  {
    ProfScope p(ctx, "keep", n * (k + 1) * 12ull);
    keep_rows_kernel<<<grid_for(ctx, n * (k + 1)), 256, 0, ctx.stream>>>(
        d.delta, d.acc, n, k, seen, ren, kept, out.delta, out.acc);
    DFM_LAUNCH_CHECK();
  }
  ctx.sync();
  return out;
}

}  // namespace dfm
