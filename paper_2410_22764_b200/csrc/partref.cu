// naivePR (paper Alg. 2/3; reference min_partref.hpp:42-176) and transPR
// (paper Alg. 5; reference min_transpr.hpp:21-122), B200 edition.
//
// Leader election: block[q] holds the id of q's block leader.  A pass reads
// the pass-entry labels `cur` (the reference's frozen copy, :85) and writes
// `nxt` (ping-pong, no copy).  Election cells are 64-bit epoch-tagged words
// (pass number in the high half, candidate in the low half), so the
// reference's O(n) cell reset per pass (:136-138) disappears:
//   deterministic_min -> atomicMin on (~pass<<32 | q)   (cells start at ~0)
//   deterministic_max -> atomicMax on ( pass<<32 | q)   (cells start at 0)
//   arbitrary_winner  -> plain 64-bit store
//   fused CAS         -> atomicCAS; a stale epoch counts as kNoLeader
// Passes are launched in batches without host round trips: a pass after the
// fixpoint is a no-op, so the host reads the per-pass "changed" flags once
// per batch and the iteration count is the first unchanged pass.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include <cooperative_groups.h>

#include "prims.cuh"

namespace cg = cooperative_groups;

namespace dfm {
namespace {

__global__ void leaders_kernel(const uint8_t* __restrict__ acc, uint64_t n, uint32_t* out2) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t la = kNoLeader, lr = kNoLeader;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    if (acc[q]) la = min(la, (uint32_t)q);
    else lr = min(lr, (uint32_t)q);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    la = min(la, __shfl_xor_sync(0xffffffffu, la, o));
    lr = min(lr, __shfl_xor_sync(0xffffffffu, lr, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (la != kNoLeader) atomicMin(&out2[0], la);
    if (lr != kNoLeader) atomicMin(&out2[1], lr);
  }
}

__global__ void init_leaders_kernel(const uint8_t* __restrict__ acc, uint64_t n,
                                    const uint32_t* __restrict__ l2, uint32_t* __restrict__ cur) {
  uint32_t la = l2[0], lr = l2[1];
  if (la == kNoLeader) la = lr;  // min_partref.hpp:62-63
  if (lr == kNoLeader) lr = la;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride)
    cur[q] = acc[q] ? la : lr;
}

// split condition (min_partref.hpp:90-99): some letter's successor lies in a
// different pass-entry block than the leader's successor on that letter
// (letters in groups of 4: the 8 successor loads, then the 8 label loads, are in
// flight together — two dependent round trips per group instead of two per letter)
__device__ __forceinline__ bool splits(const uint32_t* __restrict__ rows, uint64_t n,
                                       uint64_t letters, const uint32_t* __restrict__ cur,
                                       uint32_t q, uint32_t leader) {
  if (q == leader) return false;
  for (uint64_t a0 = 0; a0 < letters; a0 += 4) {
    uint32_t tq[4], tl[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (a0 + u < letters) {
        tq[u] = rows[(a0 + u) * n + q];
        tl[u] = rows[(a0 + u) * n + leader];
      }
    bool diff = false;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (a0 + u < letters) diff |= cur[tq[u]] != cur[tl[u]];
    if (diff) return true;
  }
  return false;
}

// Warp-aggregated election.  In early passes a few huge blocks receive tens of
// thousands of candidates each, and same-address atomics serialise at one L2
// slice; lanes of a warp hold consecutive states, so among a warp's splitting
// lanes with the same leader only the policy's candidate touches the cell —
// the lowest q for min / arbitrary / CAS, the highest for max.  The cell value
// is the one the per-state atomics would leave.
template <int kPolicy>
__device__ __forceinline__ void elect_cell(unsigned long long* cells, uint32_t leader, uint32_t q,
                                           uint32_t pass, bool sp, uint32_t vmask) {
  const uint32_t spm = __ballot_sync(vmask, sp);
  if (!sp) return;
  const uint32_t peers = __match_any_sync(spm, leader);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t src = kPolicy == DFM_POLICY_MAX ? 31 - __clz(peers) : __ffs(peers) - 1;
  if (lane != src) return;
  if (kPolicy == DFM_POLICY_MIN)
    atomicMin(&cells[leader], ((unsigned long long)(~pass) << 32) | q);
  else if (kPolicy == DFM_POLICY_MAX)
    atomicMax(&cells[leader], ((unsigned long long)pass << 32) | q);
  else
    *reinterpret_cast<volatile unsigned long long*>(&cells[leader]) =
        ((unsigned long long)pass << 32) | q;
}

// fused CAS (min_partref.hpp:116-132): the group's lowest lane competes for the
// cell; the first CAS wins and every lane of the group adopts the winner
__device__ __forceinline__ uint32_t cas_cell(unsigned long long* cells, uint32_t leader, uint32_t q,
                                             uint32_t pass, bool sp, uint32_t vmask) {
  const uint32_t spm = __ballot_sync(vmask, sp);
  if (!sp) return leader;
  const uint32_t peers = __match_any_sync(spm, leader);
  const uint32_t src = __ffs(peers) - 1;
  uint32_t winner = 0;
  if ((threadIdx.x & 31) == src) {
    const unsigned long long mine = ((unsigned long long)pass << 32) | q;
    unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(&cells[leader]);
    while (true) {
      if ((uint32_t)(old >> 32) == pass) {
        winner = (uint32_t)old;
        break;
      }
      const unsigned long long prev = atomicCAS(&cells[leader], old, mine);
      if (prev == old) {
        winner = q;
        break;
      }
      old = prev;
    }
  }
  return __shfl_sync(peers, winner, src);
}

template <int kPolicy>
__global__ void __launch_bounds__(256) elect_kernel(const uint32_t* __restrict__ rows, uint64_t n,
                                                    uint64_t letters,
                                                    const uint32_t* __restrict__ cur,
                                                    unsigned long long* cells,
                                                    uint8_t* __restrict__ split_flag,
                                                    uint32_t pass) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t qb = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); qb < n;
       qb += stride) {
    const uint64_t qi = qb + (threadIdx.x & 31);
    const uint32_t vmask = __ballot_sync(0xffffffffu, qi < n);
    if (qi >= n) continue;
    const uint32_t q = (uint32_t)qi;
    const uint32_t leader = cur[q];
    const bool s = splits(rows, n, letters, cur, q, leader);
    split_flag[q] = s;
    elect_cell<kPolicy>(cells, leader, q, pass, s, vmask);
  }
}

__global__ void __launch_bounds__(256) split_kernel(uint64_t n, const uint32_t* __restrict__ cur,
                                                    const unsigned long long* __restrict__ cells,
                                                    const uint8_t* __restrict__ split_flag,
                                                    uint32_t* __restrict__ nxt,
                                                    uint32_t* __restrict__ changed) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  bool any = false;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    const uint32_t c = cur[q];
    if (split_flag[q]) {
      nxt[q] = (uint32_t)cells[c];
      any = true;
    } else {
      nxt[q] = c;
    }
  }
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *changed = 1u;
}

// fused pass (min_partref.hpp:116-132): first CAS on the block's cell wins
__global__ void __launch_bounds__(256) cas_kernel(const uint32_t* __restrict__ rows, uint64_t n,
                                                  uint64_t letters, const uint32_t* __restrict__ cur,
                                                  unsigned long long* cells,
                                                  uint32_t* __restrict__ nxt,
                                                  uint32_t* __restrict__ changed, uint32_t pass) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  bool any = false;
  for (uint64_t qb = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); qb < n;
       qb += stride) {
    const uint64_t qi = qb + (threadIdx.x & 31);
    const uint32_t vmask = __ballot_sync(0xffffffffu, qi < n);
    if (qi >= n) continue;
    const uint32_t q = (uint32_t)qi;
    const uint32_t leader = cur[q];
    const bool sp = splits(rows, n, letters, cur, q, leader);
    any |= sp;
    nxt[q] = cas_cell(cells, leader, q, pass, sp, vmask);
  }
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) *changed = 1u;
}

// pointer doubling (min_transpr.hpp:76-83): level lvl row a = prev∘prev, all letters
__global__ void __launch_bounds__(256) double_kernel(const uint32_t* __restrict__ prev,
                                                     uint32_t* __restrict__ cur, uint64_t n,
                                                     uint64_t total) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const uint64_t row = (i / n) * n;
    cur[i] = prev[row + prev[i]];
  }
}

// ---------------------------------------------------------------------------
// Persistent cooperative variant: all passes of a run in one launch, passes
// separated by grid-wide barriers instead of kernel boundaries — for inputs
// whose pass count, not per-pass work, dominates (C1: 16,474 passes on 1e5
// states; rings and chains: n-1 passes).  Same per-pass semantics as
// elect/split/cas_kernel above.
constexpr int kPersistThreads = 1024;

struct PersistentArgs {
  const uint32_t* rows;
  uint64_t n, letters;
  uint32_t* lab0;
  uint32_t* lab1;
  unsigned long long* cells;
  uint8_t* split;
  uint32_t* changed;  // one flag per pass of this launch (zeroed by the host)
  uint32_t pass0;     // epoch of the pass before this launch
  uint32_t max_passes;
  int start_sel;
  uint32_t* out;      // [0] passes executed, [1] stable, [2] buffer holding the labels
};

template <int kPolicy, bool kCas>
__global__ void __launch_bounds__(kPersistThreads) persistent_kernel(PersistentArgs a) {
  cg::grid_group g = cg::this_grid();
  const uint64_t first = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  int sel = a.start_sel;
  uint32_t p = 0;
  bool stable = false;
  while (p < a.max_passes) {
    const uint32_t pass = a.pass0 + p + 1;
    const uint32_t* cur = sel ? a.lab1 : a.lab0;
    uint32_t* nxt = sel ? a.lab0 : a.lab1;
    // the previous pass's "changed" flag is read here and tested after this pass's
    // election, off the critical path: a pass after a stable one changes nothing
    const uint32_t prev_changed =
        p > 0 ? *reinterpret_cast<volatile uint32_t*>(&a.changed[p - 1]) : 1u;
    bool any = false;
    if (kCas) {
      for (uint64_t qb = first - (threadIdx.x & 31); qb < a.n; qb += nth) {
        const uint64_t qi = qb + (threadIdx.x & 31);
        const uint32_t vmask = __ballot_sync(0xffffffffu, qi < a.n);
        if (qi >= a.n) continue;
        const uint32_t q = (uint32_t)qi;
        const uint32_t leader = cur[q];
        const bool sp = splits(a.rows, a.n, a.letters, cur, q, leader);
        any |= sp;
        nxt[q] = cas_cell(a.cells, leader, q, pass, sp, vmask);
      }
      if (prev_changed == 0u) {  // pass p was stable; this one rewrote identical labels
        stable = true;
        break;
      }
    } else {
      for (uint64_t qb = first - (threadIdx.x & 31); qb < a.n; qb += nth) {
        const uint64_t qi = qb + (threadIdx.x & 31);
        const uint32_t vmask = __ballot_sync(0xffffffffu, qi < a.n);
        if (qi >= a.n) continue;
        const uint32_t q = (uint32_t)qi;
        const uint32_t leader = cur[q];
        const bool sp = splits(a.rows, a.n, a.letters, cur, q, leader);
        a.split[q] = sp;
        elect_cell<kPolicy>(a.cells, leader, q, pass, sp, vmask);
      }
      if (prev_changed == 0u) {  // pass p was stable; election cells are epoch-tagged
        stable = true;
        break;
      }
      g.sync();
      for (uint64_t qi = first; qi < a.n; qi += nth) {
        const uint32_t c = cur[qi];
        if (a.split[qi]) {
          nxt[qi] = (uint32_t)a.cells[c];
          any = true;
        } else {
          nxt[qi] = c;
        }
      }
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) a.changed[p] = 1u;
    g.sync();
    sel ^= 1;
    ++p;
  }
  if (!stable && p > 0 && *reinterpret_cast<volatile uint32_t*>(&a.changed[p - 1]) == 0u)
    stable = true;
  if (first == 0) {
    a.out[0] = p;
    a.out[1] = stable ? 1u : 0u;
    a.out[2] = (uint32_t)sel;
  }
}

unsigned grid_for(const Ctx& ctx, uint64_t items) {
  return (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(items, 1), 256),
                                      (uint64_t)ctx.num_sms * 16);
}

}  // namespace

constexpr uint64_t kPersistentMaxStates = 1ull << 22;

AlgoOut run_leader_election(Ctx& ctx, const DevDfa& d, const uint32_t* rows, uint64_t letters,
                            int policy, bool fused_cas, const Deadline& dl,
                            const dfm_trace* trace) {
  AlgoOut out;
  const uint64_t n = d.n;
  out.peak_memory_estimate = n * 12;  // min_partref.hpp:145
  uint32_t* lab[2] = {ctx.slot_t<uint32_t>("pr.lab0", n), ctx.slot_t<uint32_t>("pr.lab1", n)};
  auto* cells = ctx.slot_t<unsigned long long>("pr.cells", n);
  uint8_t* split_flag = fused_cas ? nullptr : ctx.slot_t<uint8_t>("pr.split", n);
  const uint32_t kBatchMax = 256;
  uint32_t* changed = ctx.slot_t<uint32_t>("pr.changed", kBatchMax);
  uint32_t* lead2 = reinterpret_cast<uint32_t*>(ctx.d_scalars + 16);
  const unsigned grid = grid_for(ctx, n);

  // algorithmic bytes per pass: own label 4, one letter's delta(q) and
  // delta(leader) 8 and their two labels 8, split flag 1, then the split phase's label,
  // flag, cell and new label 13 — the reference's early exit (min_partref.hpp:93-97)
  // means most states read one letter; the SURVEY 8(d) figure n(16k'+8) is the bound
  const uint64_t pass_bytes = n * (fused_cas ? 4ull + 16 + 8 + 4 : 4ull + 16 + 1 + 13);
  DFM_CUDA(cudaMemsetAsync(lead2, 0xFF, 8, ctx.stream));
  DFM_CUDA(cudaMemsetAsync(cells, (!fused_cas && policy == DFM_POLICY_MIN) ? 0xFF : 0x00, n * 8,
                           ctx.stream));
  {
    ProfScope p(ctx, "init");
    leaders_kernel<<<grid, 256, 0, ctx.stream>>>(d.acc, n, lead2);
    DFM_LAUNCH_CHECK();
    init_leaders_kernel<<<grid, 256, 0, ctx.stream>>>(d.acc, n, lead2, lab[0]);
    DFM_LAUNCH_CHECK();
  }
  int sel = 0;
  uint32_t pass = 0;
  const bool tracing_ = trace && trace->on_pass;
  if (!tracing_ && n <= kPersistentMaxStates) {
    // one cooperative launch per chunk of passes; the deadline is checked between
    // chunks (the reference checks it before every pass, min_partref.hpp:78-83), so
    // chunks start small and double: a run that overruns its deadline is reported as
    // a timeout within ~2x of it
    const uint32_t kChunkMax = 8192;
    uint32_t chunk = 16;
    uint32_t* chg = ctx.slot_t<uint32_t>("pr.pchanged", kChunkMax);
    uint32_t* pout = reinterpret_cast<uint32_t*>(ctx.d_scalars + 20);
    void (*kern)(PersistentArgs) =
        fused_cas ? persistent_kernel<DFM_POLICY_ARBITRARY, true>
        : policy == DFM_POLICY_MIN ? persistent_kernel<DFM_POLICY_MIN, false>
        : policy == DFM_POLICY_MAX ? persistent_kernel<DFM_POLICY_MAX, false>
                                   : persistent_kernel<DFM_POLICY_ARBITRARY, false>;
    int per_sm = 0;
    DFM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPersistThreads, 0));
    const unsigned pgrid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)per_sm * ctx.num_sms, ceil_div(n, kPersistThreads)));
    while (true) {
      if (dl.expired()) {
        out.status = DFM_STATUS_TIMEOUT;
        return out;
      }
      DFM_CUDA(cudaMemsetAsync(chg, 0, chunk * 4, ctx.stream));
      PersistentArgs pa{rows, n, letters, lab[0], lab[1], cells, split_flag, chg, pass, chunk,
                        sel, pout};
      chunk = std::min(kChunkMax, chunk * 2);
      void* args[] = {&pa};
      ProfScope prof(ctx, "elect", 0);
      DFM_CUDA(cudaLaunchCooperativeKernel((const void*)kern, pgrid, kPersistThreads, args, 0,
                                           ctx.stream));
      DFM_LAUNCH_CHECK();
      prof.stop();
      DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 20, pout, 12, cudaMemcpyDeviceToHost, ctx.stream));
      ctx.sync();
      const uint32_t* h = reinterpret_cast<const uint32_t*>(ctx.h_scalars + 20);
      prof.bytes = (uint64_t)h[0] * pass_bytes;
      pass += h[0];
      sel = (int)h[2];
      if (h[1]) break;
    }
    out.iterations = pass;
    out.canon_dev = ctx.slot_t<uint32_t>("canon", n);
    out.num_blocks = canonicalize_dev(ctx, lab[sel], n, out.canon_dev);
    out.status = DFM_STATUS_OK;
    return out;
  }
  uint32_t batch = 1;
  std::vector<uint32_t> h_changed(kBatchMax);
  std::vector<uint32_t> trace_buf;
  const bool tracing = trace && trace->on_pass;
  while (true) {
    if (dl.expired()) {
      out.status = DFM_STATUS_TIMEOUT;
      return out;
    }
    if (tracing) batch = 1;
    DFM_CUDA(cudaMemsetAsync(changed, 0, batch * 4, ctx.stream));
    // with a batch in flight the final labels sit in the buffer after the last
    // CHANGED pass; remember where each pass wrote
    int sel_after[kBatchMax];
    for (uint32_t b = 0; b < batch; ++b) {
      ++pass;
      const uint32_t* cur = lab[sel];
      uint32_t* nxt = lab[sel ^ 1];
      if (fused_cas) {
        ProfScope p(ctx, "elect", pass_bytes);
        cas_kernel<<<grid, 256, 0, ctx.stream>>>(rows, n, letters, cur, cells, nxt, changed + b,
                                                 pass);
        DFM_LAUNCH_CHECK();
      } else {
        {
          ProfScope p(ctx, "elect", n * (4ull + 16 + 1));
          if (policy == DFM_POLICY_MIN)
            elect_kernel<DFM_POLICY_MIN><<<grid, 256, 0, ctx.stream>>>(rows, n, letters, cur, cells,
                                                                       split_flag, pass);
          else if (policy == DFM_POLICY_MAX)
            elect_kernel<DFM_POLICY_MAX><<<grid, 256, 0, ctx.stream>>>(rows, n, letters, cur, cells,
                                                                       split_flag, pass);
          else
            elect_kernel<DFM_POLICY_ARBITRARY><<<grid, 256, 0, ctx.stream>>>(
                rows, n, letters, cur, cells, split_flag, pass);
          DFM_LAUNCH_CHECK();
        }
        {
          ProfScope p(ctx, "split", n * 13ull);  // label 4 + flag 1 + cell 4 + write 4
          split_kernel<<<grid, 256, 0, ctx.stream>>>(n, cur, cells, split_flag, nxt, changed + b);
          DFM_LAUNCH_CHECK();
        }
      }
      sel ^= 1;
      sel_after[b] = sel;
    }
    DFM_CUDA(cudaMemcpyAsync(h_changed.data(), changed, batch * 4, cudaMemcpyDeviceToHost,
                             ctx.stream));
    ctx.sync();
    uint32_t first_stable = batch;
    for (uint32_t b = 0; b < batch; ++b)
      if (h_changed[b] == 0) {
        first_stable = b;
        break;
      }
    if (tracing) {
      trace_buf.resize(n);
      DFM_CUDA(cudaMemcpyAsync(trace_buf.data(), lab[sel], n * 4, cudaMemcpyDeviceToHost,
                               ctx.stream));
      ctx.sync();
      trace->on_pass(trace->user, pass, trace_buf.data(), (uint32_t)n, 0);
    }
    if (first_stable < batch) {
      // passes after the first stable one were no-ops (labels unchanged)
      out.iterations = pass - batch + first_stable + 1;
      sel = sel_after[first_stable];
      break;
    }
    batch = std::min(kBatchMax, batch * 2);
  }
  out.canon_dev = ctx.slot_t<uint32_t>("canon", n);
  out.num_blocks = canonicalize_dev(ctx, lab[sel], n, out.canon_dev);
  out.status = DFM_STATUS_OK;
  return out;
}

uint32_t* expand_alphabet_dev(Ctx& ctx, const DevDfa& d, uint32_t levels) {
  const uint64_t n = d.n, k = d.k;
  uint32_t* rows = ctx.slot_t<uint32_t>("tp.rows", std::max<uint64_t>(levels * k * n, 1));
  if (k == 0 || n == 0) return rows;
  DFM_CUDA(cudaMemcpyAsync(rows, d.delta, k * n * 4, cudaMemcpyDeviceToDevice, ctx.stream));
  for (uint32_t lvl = 1; lvl < levels; ++lvl) {
    ProfScope p(ctx, "double", 12ull * k * n);  // 12 n per (level, letter)
    double_kernel<<<grid_for(ctx, k * n), 256, 0, ctx.stream>>>(
        rows + (uint64_t)(lvl - 1) * k * n, rows + (uint64_t)lvl * k * n, n, k * n);
    DFM_LAUNCH_CHECK();
  }
  return rows;
}

AlgoOut run_trans_pr(Ctx& ctx, const DevDfa& d, int policy, const dfm_limits& lim,
                     const Deadline& dl) {
  AlgoOut out;
  const uint32_t levels = dfm_power_levels(d.n);
  const uint64_t required = dfm_expand_required_bytes(d.n, d.k);
  if (required > lim.max_memory_bytes) {  // min_transpr.hpp:95-101
    out.status = DFM_STATUS_CAPACITY_EXCEEDED;
    out.peak_memory_estimate = required;
    return out;
  }
  const uint32_t* rows = expand_alphabet_dev(ctx, d, levels);
  out = run_leader_election(ctx, d, rows, (uint64_t)levels * d.k, policy, false, dl, nullptr);
  out.closure_steps = levels - 1;  // min_transpr.hpp:108
  out.peak_memory_estimate += required;
  return out;
}

}  // namespace dfm
