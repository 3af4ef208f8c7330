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
        p > 0 ? prims::ld_relaxed_u32(&a.changed[p - 1]) : 1u;
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
  if (!stable && p > 0 && prims::ld_relaxed_u32(&a.changed[p - 1]) == 0u)
    stable = true;
  if (first == 0) {
    a.out[0] = p;
    a.out[1] = stable ? 1u : 0u;
    a.out[2] = (uint32_t)sel;
  }
}

// ---------------------------------------------------------------------------
// One grid barrier per pass: the split phase of pass p-1 is not materialised
// before pass p; pass p reads the label words the previous pass wrote — the labels
// L(p-2) with that pass's split flag in bit 31 — and that pass's election cells,
// and forms each label it needs on the fly: L(p-1)[x] = flag ? winner(cell(p-1)[
// L(p-2)[x]]) : L(p-2)[x].  Each thread stores L(p-1) of its own state with its
// split flag of pass p (for pass p+1), and its election for pass p.  Election
// cells are double-buffered by pass parity, labels by the usual two buffers.  Same
// per-pass semantics and pass count as persistent_kernel (min_partref.hpp:78-143);
// the dependent-load depth of a pass is unchanged and there is no extra gather
// per compared letter (the flag rides in the label word), one barrier and one grid
// sweep fewer.
struct FusedArgs {
  const uint32_t* rows;
  uint64_t n, letters;
  uint32_t* lab0;
  uint32_t* lab1;
  unsigned long long* cells0;  // pass parity 0 / 1
  unsigned long long* cells1;
  uint32_t* changed;  // one flag per pass of this launch (zeroed by the host)
  uint32_t pass0;
  uint32_t max_passes;
  int start_sel;  // buffer holding the labels the next pass reads
  uint32_t* out;  // [0] passes executed, [1] stable, [2] buffer holding the labels
  // work-efficient passes (null: off): predecessor lists (CSR over all letters) and
  // mark[r] = the first pass that must re-evaluate r — set when a successor of r
  // split (its label changed).  A state is evaluated in pass P iff it split in P-1
  // (new leader), mark[q] >= P, or mark[leader(q)] >= P (a successor of its leader
  // changed); otherwise every label it would compare is unchanged since its last
  // evaluation, which found no difference, so its verdict is "no split" again.
  const uint32_t* pred_off;
  const uint32_t* pred_src;
  uint32_t* mark;
  uint32_t dirty_from;  // first pass that writes marks (it evaluates every state)
  bool own_label;       // kOne: keep the state's own label word in a register
  // letter masks (the kMask kernels; <= 32 letters, n < 2^21): `mark` is then three
  // arrays of n, pass P reads mask[P % 3] — the letters whose successor changed in
  // P-1 — writes mask[(P+1) % 3] and clears mask[(P+2) % 3].  A state evaluated only
  // through the marks compares just the letters in mask[q] | mask[leader(q)]: every
  // other letter compares two labels unchanged since an evaluation that found them
  // equal.  pred_src then packs (source | letter << 21).
};
constexpr uint32_t kPredSrcBits = 21;

// label words carry the previous pass's split flag in bit 31 (state ids < 2^31), so
// one gather yields both the label and whether it must be corrected
constexpr uint32_t kSplitBit = 0x80000000u;
__device__ __forceinline__ uint32_t label_on_the_fly(uint32_t w, const unsigned long long* cprev) {
  return (w & kSplitBit) ? (uint32_t)cprev[w & ~kSplitBit] : w;
}

// kMask: the letter-mask variant (launched once the masks exist; the plain variants
// keep their code: the extra paths doubled the latency-bound C1 kernel's SASS and
// slowed it 43 %)
template <int kPolicy, bool kOne, bool kMask = false>
__global__ void __launch_bounds__(kPersistThreads) fused_pr_kernel(FusedArgs a) {
  cg::grid_group g = cg::this_grid();
  const uint64_t first = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  int sel = a.start_sel;
  uint32_t p = 0;
  bool stable = false;
  // one state per thread (n <= resident threads): the first four successors of the
  // state and of its leader stay in registers — the leader changes only when the
  // state splits — taking the leader-row load off the pass's dependent chain
  constexpr bool one = kOne;  // the host launches kOne only when n <= resident threads
  uint32_t cl = 0xFFFFFFFFu, crow[4] = {0, 0, 0, 0}, qrow[4] = {0, 0, 0, 0};
  // ... and so does its own label word: the word pass p reads at Lm[q] is the one this
  // thread wrote in pass p-1 (one dependent L2 round trip fewer per pass)
  uint32_t myw = 0;
  if (one && first < a.n) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if ((uint64_t)u < a.letters) qrow[u] = a.rows[(uint64_t)u * a.n + first];
  }
  const bool own_label_enabled = a.own_label;
  // masked passes above the resident threads: the warps of a CTA take its rows of 32
  // states from a shared counter, so a warp that drew cheap rows
  // (skip tests) takes more instead of waiting at the grid barrier for the warp that
  // drew full evaluations (ncu, C2: 44 % of the stall samples were that barrier)
  constexpr bool dyn = !kOne;
  __shared__ uint32_t s_row[2];
  // rows are dealt round-robin (CTA b takes rows b, b + G, b + 2G, ...): every CTA
  // draws from the whole state range, so contiguous heavy regions spread over the SMs
  const uint64_t nrows = (a.n + 31) / 32;
  if (dyn) {
    if (threadIdx.x < 2) s_row[threadIdx.x] = 0;
    __syncthreads();
  }
  while (p < a.max_passes) {
    const uint32_t pass = a.pass0 + p + 1;
    if (dyn && threadIdx.x == 0) s_row[(p + 1) & 1] = 0;  // last used in pass p - 1
    const uint32_t* Lm = sel ? a.lab1 : a.lab0;
    uint32_t* Lw = sel ? a.lab0 : a.lab1;
    const unsigned long long* cprev = (pass & 1) ? a.cells0 : a.cells1;
    unsigned long long* ccur = (pass & 1) ? a.cells1 : a.cells0;
    const uint32_t prev_changed =
        p > 0 ? prims::ld_relaxed_u32(&a.changed[p - 1]) : 1u;
    bool any = false;
    const uint64_t qend = a.n;
    for (uint64_t qb = dyn ? 0 : first - (threadIdx.x & 31);; qb += nth) {
      if (dyn) {
        uint32_t r = 0;
        if ((threadIdx.x & 31) == 0) r = atomicAdd(&s_row[p & 1], 1u);
        const uint64_t row = blockIdx.x + (uint64_t)gridDim.x * __shfl_sync(0xffffffffu, r, 0);
        qb = row < nrows ? 32ull * row : qend;
      }
      if (qb >= qend) break;
      const uint64_t qi = qb + (threadIdx.x & 31);
      const uint32_t vmask = __ballot_sync(0xffffffffu, qi < qend);
      if (qi >= qend) continue;
      const uint32_t q = (uint32_t)qi;
      const uint32_t lw = (one && p > 0 && own_label_enabled) ? myw : Lm[q];
      const uint32_t leader = label_on_the_fly(lw, cprev);
      bool sp = false;
      bool eval = q != leader;
      uint32_t lm = 0xFFFFFFFFu;  // letters to compare
      if (eval && a.mark != nullptr && pass > a.dirty_from && !(lw & kSplitBit)) {
        if constexpr (kMask) {
          const uint32_t* mc = a.mark + (uint64_t)(pass % 3) * a.n;
          lm = mc[q] | mc[leader];
          eval = lm != 0;
        } else {
          eval = a.mark[q] >= pass || a.mark[leader] >= pass;
        }
      }
      if constexpr (kMask)  // (read in pass - 1, written in pass + 1)
        if (pass >= a.dirty_from) a.mark[(uint64_t)((pass + 2) % 3) * a.n + q] = 0;
      if (one && leader != cl && eval && (!kMask || lm == 0xFFFFFFFFu)) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if ((uint64_t)u < a.letters) crow[u] = a.rows[(uint64_t)u * a.n + leader];
        cl = leader;
      }
      if (kMask && eval && lm != 0xFFFFFFFFu) {  // only the letters whose successors changed
        uint32_t rem = lm;
        while (rem != 0u && !sp) {
          uint32_t al[4], tq[4], tl[4], lq[4], ll[4];
          int c = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (rem != 0u) {
              al[u] = (uint32_t)__ffs(rem) - 1u;
              rem &= rem - 1u;
              c = u + 1;
            }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < c) {
              tq[u] = a.rows[(uint64_t)al[u] * a.n + q];
              tl[u] = a.rows[(uint64_t)al[u] * a.n + leader];
            }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < c) {
              lq[u] = Lm[tq[u]];
              ll[u] = Lm[tl[u]];
            }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < c) sp |= label_on_the_fly(lq[u], cprev) != label_on_the_fly(ll[u], cprev);
        }
      } else if (eval) {
        for (uint64_t a0 = 0; a0 < a.letters && !sp; a0 += 4) {
          uint32_t tq[4], tl[4], lq[4], ll[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (a0 + u < a.letters) {
              tq[u] = (one && a0 == 0) ? qrow[u] : a.rows[(a0 + u) * a.n + q];
              tl[u] = (one && a0 == 0) ? crow[u] : a.rows[(a0 + u) * a.n + leader];
            }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (a0 + u < a.letters) {
              lq[u] = Lm[tq[u]];
              ll[u] = Lm[tl[u]];
            }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (a0 + u < a.letters)
              sp |= label_on_the_fly(lq[u], cprev) != label_on_the_fly(ll[u], cprev);
        }
      }
      Lw[q] = leader | (sp ? kSplitBit : 0u);  // this pass's split rides with the label
      if (one) myw = leader | (sp ? kSplitBit : 0u);
      any |= sp;
      elect_cell<kPolicy>(ccur, leader, q, pass, sp, vmask);
      if (sp && a.mark != nullptr) {  // q's label changes: its predecessors re-evaluate
        // (pass >= dirty_from always holds here: marks exist only from that launch on)
        if constexpr (kMask) {
          uint32_t* mn = a.mark + (uint64_t)((pass + 1) % 3) * a.n;
          for (uint32_t e = a.pred_off[q], e1 = a.pred_off[q + 1]; e < e1; ++e) {
            const uint32_t ps = a.pred_src[e];
            atomicOr(&mn[ps & ((1u << kPredSrcBits) - 1u)], 1u << (ps >> kPredSrcBits));
          }
        } else {
          for (uint32_t e = a.pred_off[q], e1 = a.pred_off[q + 1]; e < e1; ++e)
            a.mark[a.pred_src[e]] = pass + 1;
        }
      }
    }
    if (prev_changed == 0u) {  // pass p was stable: this pass rewrote the same labels
      stable = true;
      break;
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) a.changed[p] = 1u;
    g.sync();
    sel ^= 1;
    ++p;
  }
  if (!stable && p > 0 && prims::ld_relaxed_u32(&a.changed[p - 1]) == 0u)
    stable = true;
  if (first == 0) {
    a.out[0] = p;
    a.out[1] = stable ? 1u : 0u;
    a.out[2] = (uint32_t)sel;
  }
}

// ---------------------------------------------------------------------------
// Queued masked passes (letter masks on, n above the resident threads).  The grid-
// stride loop of fused_pr_kernel<kMask> walks ~n / resident-threads states per thread
// one after another, each a chain of dependent L2 round trips (label word -> cell ->
// masks -> rows -> labels -> cells), although most states stop at the skip test.
// Here a pass runs in rounds of kQueue states per CTA: stage A evaluates the skip test
// of three states per thread with all their loads in flight and writes the unchanged
// labels at once; the states that must compare letters go to a shared-memory queue,
// which stage B drains one entry per thread.  The queue breaks the lane = q order the
// warp-aggregated election relies on, so the group's candidate is found with a
// min / max reduction over its lanes.  Same per-pass semantics as fused_pr_kernel.
constexpr int kQueuePer = 3;  // states per thread per round (static smem: 36 KB)
constexpr int kQueue = kQueuePer * kPersistThreads;
template <int kPolicy>
__device__ __forceinline__ void elect_cell_any(unsigned long long* cells, uint32_t leader,
                                               uint32_t q, uint32_t pass, bool sp,
                                               uint32_t vmask) {
  const uint32_t spm = __ballot_sync(vmask, sp);
  if (!sp) return;
  const uint32_t peers = __match_any_sync(spm, leader);
  if (kPolicy == DFM_POLICY_MIN) {
    if (__reduce_min_sync(peers, q) == q)
      atomicMin(&cells[leader], ((unsigned long long)(~pass) << 32) | q);
  } else if (kPolicy == DFM_POLICY_MAX) {
    if (__reduce_max_sync(peers, q) == q)
      atomicMax(&cells[leader], ((unsigned long long)pass << 32) | q);
  } else if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) {
    *reinterpret_cast<volatile unsigned long long*>(&cells[leader]) =
        ((unsigned long long)pass << 32) | q;
  }
}

template <int kPolicy>
__global__ void __launch_bounds__(kPersistThreads) queue_pr_kernel(FusedArgs a) {
  cg::grid_group g = cg::this_grid();
  __shared__ uint32_t s_q[kQueue], s_l[kQueue], s_m[kQueue];
  __shared__ uint32_t s_cnt;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t per = (a.n + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = (uint64_t)blockIdx.x * per;
  const uint64_t hi = lo + per < a.n ? lo + per : a.n;
  int sel = a.start_sel;
  uint32_t p = 0;
  bool stable = false;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  while (p < a.max_passes) {
    const uint32_t pass = a.pass0 + p + 1;
    const uint32_t* Lm = sel ? a.lab1 : a.lab0;
    uint32_t* Lw = sel ? a.lab0 : a.lab1;
    const unsigned long long* cprev = (pass & 1) ? a.cells0 : a.cells1;
    unsigned long long* ccur = (pass & 1) ? a.cells1 : a.cells0;
    const uint32_t prev_changed = p > 0 ? prims::ld_relaxed_u32(&a.changed[p - 1]) : 1u;
    const uint32_t* mc = a.mark + (uint64_t)(pass % 3) * a.n;
    uint32_t* mn = a.mark + (uint64_t)((pass + 1) % 3) * a.n;
    uint32_t* mz = a.mark + (uint64_t)((pass + 2) % 3) * a.n;
    const bool masks_valid = pass > a.dirty_from;
    bool any = false;
    for (uint64_t rb = lo; rb < hi; rb += kQueue) {
      // stage A: skip tests, kQueuePer states per thread, loads batched
      uint32_t lw[kQueuePer], ld[kQueuePer], lm[kQueuePer];
#pragma unroll
      for (int u = 0; u < kQueuePer; ++u) {
        const uint64_t qi = rb + (uint64_t)u * kPersistThreads + threadIdx.x;
        lw[u] = qi < hi ? Lm[qi] : 0u;
      }
#pragma unroll
      for (int u = 0; u < kQueuePer; ++u) {
        const uint64_t qi = rb + (uint64_t)u * kPersistThreads + threadIdx.x;
        ld[u] = qi < hi ? label_on_the_fly(lw[u], cprev) : (uint32_t)qi;
      }
#pragma unroll
      for (int u = 0; u < kQueuePer; ++u) {
        const uint64_t qi = rb + (uint64_t)u * kPersistThreads + threadIdx.x;
        const bool ev = qi < hi && (uint32_t)qi != ld[u];
        lm[u] = 0u;
        if (ev) lm[u] = (masks_valid && !(lw[u] & kSplitBit)) ? (mc[qi] | mc[ld[u]]) : 0xFFFFFFFFu;
        if (qi < hi) mz[qi] = 0u;  // (read in pass - 1, written in pass + 1)
      }
#pragma unroll
      for (int u = 0; u < kQueuePer; ++u) {
        const uint64_t qi = rb + (uint64_t)u * kPersistThreads + threadIdx.x;
        const bool push = lm[u] != 0u;
        if (qi < hi && !push) Lw[qi] = ld[u];
        const uint32_t bm = __ballot_sync(0xffffffffu, push);
        uint32_t base = 0;
        if (lane == 0 && bm) base = atomicAdd(&s_cnt, (uint32_t)__popc(bm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (push) {
          const uint32_t slot = base + __popc(bm & ((1u << lane) - 1u));
          s_q[slot] = (uint32_t)qi;
          s_l[slot] = ld[u];
          s_m[slot] = lm[u];
        }
      }
      __syncthreads();
      const uint32_t cnt = s_cnt;
      // stage B: the queued states compare their letters
      for (uint32_t ib = threadIdx.x - lane; ib < cnt; ib += kPersistThreads) {
        const uint32_t i = ib + lane;
        const bool valid = i < cnt;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        if (!valid) continue;
        const uint32_t q = s_q[i], leader = s_l[i];
        uint32_t rem = s_m[i];
        bool sp = false;
        if (rem == 0xFFFFFFFFu) {
          for (uint64_t a0 = 0; a0 < a.letters && !sp; a0 += 4) {
            uint32_t tq[4], tl[4], lq[4], ll[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (a0 + u < a.letters) {
                tq[u] = a.rows[(a0 + u) * a.n + q];
                tl[u] = a.rows[(a0 + u) * a.n + leader];
              }
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (a0 + u < a.letters) {
                lq[u] = Lm[tq[u]];
                ll[u] = Lm[tl[u]];
              }
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (a0 + u < a.letters)
                sp |= label_on_the_fly(lq[u], cprev) != label_on_the_fly(ll[u], cprev);
          }
        } else {
          while (rem != 0u && !sp) {
            uint32_t al[4], tq[4], tl[4], lq[4], ll[4];
            int c = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (rem != 0u) {
                al[u] = (uint32_t)__ffs(rem) - 1u;
                rem &= rem - 1u;
                c = u + 1;
              }
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < c) {
                tq[u] = a.rows[(uint64_t)al[u] * a.n + q];
                tl[u] = a.rows[(uint64_t)al[u] * a.n + leader];
              }
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < c) {
                lq[u] = Lm[tq[u]];
                ll[u] = Lm[tl[u]];
              }
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < c) sp |= label_on_the_fly(lq[u], cprev) != label_on_the_fly(ll[u], cprev);
          }
        }
        Lw[q] = leader | (sp ? kSplitBit : 0u);
        any |= sp;
        elect_cell_any<kPolicy>(ccur, leader, q, pass, sp, vmask);
        if (sp) {  // q's label changes: its predecessors compare that letter next pass
          for (uint32_t e = a.pred_off[q], e1 = a.pred_off[q + 1]; e < e1; ++e) {
            const uint32_t ps = a.pred_src[e];
            atomicOr(&mn[ps & ((1u << kPredSrcBits) - 1u)], 1u << (ps >> kPredSrcBits));
          }
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) s_cnt = 0;
      __syncthreads();
    }
    if (prev_changed == 0u) {  // pass p was stable: this pass rewrote the same labels
      stable = true;
      break;
    }
    if (__any_sync(0xffffffffu, any) && lane == 0) a.changed[p] = 1u;
    g.sync();
    sel ^= 1;
    ++p;
  }
  if (!stable && p > 0 && prims::ld_relaxed_u32(&a.changed[p - 1]) == 0u) stable = true;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out[0] = p;
    a.out[1] = stable ? 1u : 0u;
    a.out[2] = (uint32_t)sel;
  }
}

// ---------------------------------------------------------------------------
// Lane groups for large alphabets: kG lanes per state, each comparing the letters
// a = g, g + kG, ... (kPer of them per round, all loads of a round in flight), so a
// stable state costs one round of two dependent gathers instead of k/4 rounds
// (min_partref.hpp:93-97's early exit only helps the states that split).  The
// group's first lane writes the label, elects and marks as fused_pr_kernel does;
// same per-pass semantics and pass count.
template <int kPolicy, int kG>
__global__ void __launch_bounds__(kPersistThreads) fused_group_kernel(FusedArgs a) {
  constexpr int kPer = 4;
  cg::grid_group g = cg::this_grid();
  const uint32_t lane = threadIdx.x & 31, sub = lane % kG;
  const uint32_t gmask = ((1u << kG) - 1u) << (lane - sub);  // (kG < 32)
  const uint64_t spw = 32 / kG;  // states per warp step
  const uint64_t warp_id = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  int sel = a.start_sel;
  uint32_t p = 0;
  bool stable = false;
  while (p < a.max_passes) {
    const uint32_t pass = a.pass0 + p + 1;
    const uint32_t* Lm = sel ? a.lab1 : a.lab0;
    uint32_t* Lw = sel ? a.lab0 : a.lab1;
    const unsigned long long* cprev = (pass & 1) ? a.cells0 : a.cells1;
    unsigned long long* ccur = (pass & 1) ? a.cells1 : a.cells0;
    const uint32_t prev_changed = p > 0 ? prims::ld_relaxed_u32(&a.changed[p - 1]) : 1u;
    bool any = false;
    for (uint64_t qb = warp_id * spw; qb < a.n; qb += nwarps * spw) {
      const uint64_t qi = qb + lane / kG;
      const bool valid = qi < a.n;
      const uint32_t q = (uint32_t)qi;
      uint32_t lw = 0, leader = 0;
      bool eval = false;
      if (valid) {
        lw = Lm[q];
        leader = label_on_the_fly(lw, cprev);
        eval = q != leader;
        if (eval && a.mark != nullptr && pass > a.dirty_from && !(lw & kSplitBit))
          eval = a.mark[q] >= pass || a.mark[leader] >= pass;
      }
      bool spl = false;
      if (eval) {
        for (uint64_t a0 = sub; a0 < a.letters && !spl; a0 += (uint64_t)kG * kPer) {
          uint32_t tq[kPer], tl[kPer], lq[kPer], ll[kPer];
#pragma unroll
          for (int u = 0; u < kPer; ++u) {
            const uint64_t aa = a0 + (uint64_t)u * kG;
            if (aa < a.letters) {
              tq[u] = a.rows[aa * a.n + q];
              tl[u] = a.rows[aa * a.n + leader];
            }
          }
#pragma unroll
          for (int u = 0; u < kPer; ++u)
            if (a0 + (uint64_t)u * kG < a.letters) {
              lq[u] = Lm[tq[u]];
              ll[u] = Lm[tl[u]];
            }
#pragma unroll
          for (int u = 0; u < kPer; ++u)
            if (a0 + (uint64_t)u * kG < a.letters)
              spl |= label_on_the_fly(lq[u], cprev) != label_on_the_fly(ll[u], cprev);
        }
      }
      const bool sp = (__ballot_sync(0xffffffffu, spl) & gmask) != 0;
      const bool head = valid && sub == 0;
      const uint32_t vmask = __ballot_sync(0xffffffffu, head);
      if (head) {
        Lw[q] = leader | (sp ? kSplitBit : 0u);
        any |= sp;
        elect_cell<kPolicy>(ccur, leader, q, pass, sp, vmask);
      }
      if (sp && valid && a.mark != nullptr)  // the group marks q's predecessors
        for (uint32_t e = a.pred_off[q] + sub, e1 = a.pred_off[q + 1]; e < e1; e += kG)
          a.mark[a.pred_src[e]] = pass + 1;
    }
    if (prev_changed == 0u) {  // pass p was stable: this pass rewrote the same labels
      stable = true;
      break;
    }
    if (__any_sync(0xffffffffu, any) && lane == 0) a.changed[p] = 1u;
    g.sync();
    sel ^= 1;
    ++p;
  }
  if (!stable && p > 0 && prims::ld_relaxed_u32(&a.changed[p - 1]) == 0u) stable = true;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out[0] = p;
    a.out[1] = stable ? 1u : 0u;
    a.out[2] = (uint32_t)sel;
  }
}

// ---------------------------------------------------------------------------
// Cluster variant for tiny inputs (rings and chains of a few thousand states run
// n-1 passes): the whole working set — successor rows, both label buffers,
// election cells, split flags — lives in the (distributed) shared memory of a
// thread-block cluster; CTA r owns states [r*S, (r+1)*S) and any state's data is
// one (DSMEM) access away; the two barriers per pass are cluster barriers instead
// of grid-wide ones.  Same per-pass semantics as persistent_kernel.  Used for
// single-CTA instances only (see run_leader_election for the measurements).
struct ClusterArgs {
  const uint32_t* rows;  // global [letters][n]
  uint64_t n, letters;
  uint32_t S;            // states per CTA
  uint32_t* lab0;        // global label buffers (in/out)
  uint32_t* lab1;
  uint32_t pass0, max_passes;
  int start_sel;
  uint32_t* out;         // [0] passes executed, [1] stable, [2] buffer holding the labels
};

// DSMEM accesses through explicit shared::cluster addresses.  Election cells are
// 32-bit (64-bit min/max on another CTA's shared memory is not a native atomic on
// sm_100: ptxas lowers it to a local-CTA CAS fallback) and double-buffered by pass
// parity instead of epoch-tagged: a CTA clears its own cells of the next pass while
// the current pass runs (their last readers finished before this pass's barrier).
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, uint32_t rank) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsmem_min_u32(uint32_t addr, uint32_t v) {
  asm volatile("red.shared::cluster.min.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void dsmem_max_u32(uint32_t addr, uint32_t v) {
  asm volatile("red.shared::cluster.max.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t dsmem_cas_u32(uint32_t addr, uint32_t cmp, uint32_t val) {
  uint32_t old;
  asm volatile("atom.shared::cluster.cas.b32 %0, [%1], %2, %3;"
               : "=r"(old) : "r"(addr), "r"(cmp), "r"(val) : "memory");
  return old;
}
__device__ __forceinline__ void dsmem_or_u32(uint32_t addr, uint32_t v) {
  asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t dsmem_ld_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

template <int kPolicy, bool kCas>
__global__ void __launch_bounds__(1024, 1) cluster_pr_kernel(ClusterArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t me = cl.block_rank();
  const uint32_t S = a.S;
  extern __shared__ uint32_t s_dyn[];
  // per CTA: cells[2][S] | lab0[S] | lab1[S] | rows[letters][S] | split[S] u8
  uint32_t* s_cells = s_dyn;
  uint32_t* s_lab0 = s_cells + 2 * S;
  uint32_t* s_lab1 = s_lab0 + S;
  uint32_t* s_rows = s_lab1 + S;
  uint8_t* s_split = reinterpret_cast<uint8_t*>(s_rows + (uint64_t)a.letters * S);
  __shared__ uint32_t s_changed[3];  // per-pass flags, rotating (see the reset below)
  const uint64_t base = (uint64_t)me * S;
  const uint32_t own = base >= a.n ? 0u : (uint32_t)(a.n - base < S ? a.n - base : S);
  // MIN: cells hold q (empty ~0); MAX / arbitrary / CAS: q + 1 (empty 0)
  const uint32_t empty = (!kCas && kPolicy == DFM_POLICY_MIN) ? 0xFFFFFFFFu : 0u;
  const uint32_t* gin = a.start_sel ? a.lab1 : a.lab0;
  for (uint32_t i = threadIdx.x; i < own; i += blockDim.x) {
    s_cells[i] = empty;
    s_cells[S + i] = empty;
    s_lab0[i] = gin[base + i];
    for (uint64_t c = 0; c < a.letters; ++c) s_rows[c * S + i] = a.rows[c * a.n + base + i];
  }
  if (threadIdx.x < 3) s_changed[threadIdx.x] = 0;
  cl.sync();
  auto rlab = [&](const uint32_t* local, uint32_t x) -> uint32_t {
    return *(cl.map_shared_rank(local, x / S) + (x % S));
  };
  auto rrow = [&](uint64_t c, uint32_t x) -> uint32_t {
    return *(cl.map_shared_rank(s_rows, x / S) + c * S + (x % S));
  };
  const uint32_t flag0 = dsmem_addr(s_changed, 0);
  int sel = 0;  // local buffer holding the current labels (s_lab0 after the load)
  uint32_t p = 0;
  bool stable = false;
  const uint32_t lane = threadIdx.x & 31;
  while (p < a.max_passes) {
    const uint32_t* cur = sel ? s_lab1 : s_lab0;
    uint32_t* nxt = sel ? s_lab0 : s_lab1;
    uint32_t* cells = s_cells + (p & 1) * S;
    // pass p writes flag p % 3; flag (p + 1) % 3 was last read at the end of pass
    // p - 2, which every CTA has left (two cluster barriers since)
    if (me == 0 && threadIdx.x == 0) s_changed[(p + 1) % 3] = 0;
    {  // the next pass's cells: last read in pass p - 1's split phase
      uint32_t* nc = s_cells + ((p + 1) & 1) * S;
      for (uint32_t i = threadIdx.x; i < own; i += blockDim.x) nc[i] = empty;
    }
    auto rcell = [&](uint32_t x) -> uint32_t { return dsmem_addr(cells + (x % S), x / S); };
    bool any = false;
    for (uint32_t ib = threadIdx.x & ~31u; ib < own; ib += blockDim.x) {
      const uint32_t i = ib + lane;
      const bool valid = i < own;
      const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
      if (!valid) continue;
      const uint32_t q = (uint32_t)(base + i);
      const uint32_t leader = cur[i];
      bool sp = false;
      if (q != leader) {
        for (uint64_t c0 = 0; c0 < a.letters && !sp; c0 += 4) {
          uint32_t tq[4], tl[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c0 + u < a.letters) {
              tq[u] = s_rows[(c0 + u) * S + i];
              tl[u] = rrow(c0 + u, leader);
            }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c0 + u < a.letters) sp |= rlab(cur, tq[u]) != rlab(cur, tl[u]);
        }
      }
      // warp-aggregated election (see elect_cell): consecutive lanes hold consecutive q
      const uint32_t spm = __ballot_sync(vmask, sp);
      if (kCas) {
        any |= sp;
        uint32_t win = leader;
        if (sp) {
          const uint32_t peers = __match_any_sync(spm, leader);
          const uint32_t src = __ffs(peers) - 1;
          uint32_t w = 0;
          if (lane == src) {  // first CAS into an empty cell wins
            const uint32_t prev = dsmem_cas_u32(rcell(leader), 0u, q + 1);
            w = prev == 0u ? q : prev - 1;
          }
          win = __shfl_sync(peers, w, src);
        }
        nxt[i] = win;
      } else {
        s_split[i] = sp;
        if (sp) {
          const uint32_t peers = __match_any_sync(spm, leader);
          const uint32_t src = kPolicy == DFM_POLICY_MAX ? 31 - __clz(peers) : __ffs(peers) - 1;
          if (lane == src) {
            if (kPolicy == DFM_POLICY_MIN) dsmem_min_u32(rcell(leader), q);
            else if (kPolicy == DFM_POLICY_MAX) dsmem_max_u32(rcell(leader), q + 1);
            else dsmem_st_u32(rcell(leader), q + 1);
          }
        }
      }
    }
    if (!kCas) {
      cl.sync();
      for (uint32_t i = threadIdx.x; i < own; i += blockDim.x) {
        const uint32_t c = cur[i];
        if (s_split[i]) {
          const uint32_t v = dsmem_ld_u32(rcell(c));
          nxt[i] = kPolicy == DFM_POLICY_MIN ? v : v - 1;
          any = true;
        } else {
          nxt[i] = c;
        }
      }
    }
    if (__any_sync(0xffffffffu, any) && lane == 0) dsmem_or_u32(flag0 + 4 * (p % 3), 1u);
    cl.sync();
    sel ^= 1;
    ++p;
    if (dsmem_ld_u32(flag0 + 4 * ((p - 1) % 3)) == 0u) {
      stable = true;
      break;
    }
  }
  // labels back to global (the buffer the host expects next)
  const uint32_t* fin = sel ? s_lab1 : s_lab0;
  uint32_t* gout = ((a.start_sel + (int)p) & 1) ? a.lab1 : a.lab0;
  for (uint32_t i = threadIdx.x; i < own; i += blockDim.x) gout[base + i] = fin[i];
  if (me == 0 && threadIdx.x == 0) {
    a.out[0] = p;
    a.out[1] = stable ? 1u : 0u;
    a.out[2] = (uint32_t)((a.start_sel + (int)p) & 1);
  }
  cl.sync();  // no CTA leaves while others may still read its shared memory
}

unsigned grid_for(const Ctx& ctx, uint64_t items) {
  return (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(items, 1), 256),
                                      (uint64_t)ctx.num_sms * 16);
}

}  // namespace

// Persistent kernels (all passes in one launch; grid barriers) up to 2M states;
// larger inputs launch each pass at full occupancy.  Measured (B200, persistent vs
// per-pass launches): transPR chain 1e6 1.70 vs 1.92 ms, chain 4e6 7.5 vs 4.7 ms,
// comb 4e6 10.8 vs 8.9 ms; naive vlts 1e6 (602 passes) 59.8 vs 69.4 ms, random 3e5
// (50,291 passes) 477 vs 1421 ms.
constexpr uint64_t kPersistentMaxStates = 1ull << 21;

uint64_t persistent_max_states() {  // DFM_NAIVE_PERSIST_MAX (experiments)
  const char* e = getenv("DFM_NAIVE_PERSIST_MAX");
  return e ? strtoull(e, nullptr, 10) : kPersistentMaxStates;
}
constexpr uint64_t kClusterMaxStates = 4096;

// resident threads of the cooperative launch of `kern` (per variant: its register
// count sets its occupancy)
__global__ void pred_count_kernel(const uint32_t* __restrict__ rows, uint64_t n, uint64_t letters,
                                  uint32_t* __restrict__ deg) {
  const uint64_t total = n * letters, stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += stride)
    atomicAdd(&deg[rows[j]], 1u);
}
__global__ void pred_fill_kernel(const uint32_t* __restrict__ rows, uint64_t n, uint64_t letters,
                                 uint32_t* __restrict__ cursor, uint32_t* __restrict__ src,
                                 bool with_letter) {
  const uint64_t total = n * letters, stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += stride) {
    const uint32_t s = (uint32_t)(j % n);
    src[atomicAdd(&cursor[rows[j]], 1u)] =
        with_letter ? s | (uint32_t)(j / n) << kPredSrcBits : s;
  }
}
struct DegIn {
  const uint32_t* deg;
  __device__ uint32_t operator()(uint64_t i) const { return deg[i]; }
};
struct DegOut {
  uint32_t* off;
  uint32_t* cursor;
  __device__ void operator()(uint64_t i, uint32_t excl, uint32_t) const {
    off[i] = excl;
    cursor[i] = excl;
  }
};

// DFM_NAIVE_QUEUE=1 (opt-in): the masked passes above the resident threads run
// queue_pr_kernel.  Measured on C2 naive (vlts(1000, 1e6, 20), profiles/r04/r04b): 35.5 vs
// 33.0 ms for fused_pr_kernel<kMask> — exact, but slower
bool queue_enabled() {
  const char* e = getenv("DFM_NAIVE_QUEUE");
  return e != nullptr && e[0] == '1';
}

// DFM_NAIVE_ONE=0 (tests): the grid-stride / dynamic-row kernels even when every
// state would get its own resident thread
bool one_enabled() {
  const char* e = getenv("DFM_NAIVE_ONE");
  return e == nullptr || e[0] != '0';
}

bool own_label_on() {
  const char* e = getenv("DFM_NAIVE_OWN_LABEL");
  return e == nullptr || e[0] != '0';
}

// large alphabets only: the marks cost one store per predecessor of each split state
// and two reads per state; the saving is up to 2k gathers per stable state per pass
bool dirty_enabled(uint64_t n, uint64_t letters) {
  const char* e = getenv("DFM_NAIVE_DIRTY");
  if (e != nullptr) return e[0] == '1';
  return letters >= 8 && n * letters < (1ull << 31);
}

uint64_t fused_max_states(const Ctx& ctx, const void* kern) {
  const int per_sm = per_device_memo(kern, ctx.device, [](const void* k) {
        int v = 0;
        DFM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, kPersistThreads, 0));
        return v;
      });
  return (uint64_t)per_sm * ctx.num_sms * kPersistThreads;
}

// DFM_NAIVE_GROUP (opt-in): 1 = lane groups for >= 8 letters when the thread-per-
// state variant does not hold all states, 2 = always (tests).  Off by default:
// measured on vlts(1000, 1e6, 20) (602 passes) 49.3 ms -> 114.5 ms — with the
// work-efficient marks most states only run the skip test, which the groups
// replicate kG times (`profiles/r03q`)
int group_mode() {
  const char* e = getenv("DFM_NAIVE_GROUP");
  return e == nullptr ? 0 : (int)strtol(e, nullptr, 10);
}

// passes before the predecessor lists are built (DFM_NAIVE_DIRTY_AFTER, default 64)
uint32_t dirty_after() {
  const char* e = getenv("DFM_NAIVE_DIRTY_AFTER");
  return e ? (uint32_t)strtoul(e, nullptr, 10) : 64u;
}

// DFM_NAIVE_LMASK=0: work-efficient passes re-compare every letter of a marked state
bool lmask_enabled() {
  const char* e = getenv("DFM_NAIVE_LMASK");
  return e == nullptr || e[0] != '0';
}

bool fused_enabled() {
  const char* e = getenv("DFM_NAIVE_FUSED");
  return e == nullptr || e[0] != '0';
}

bool cluster_disabled() {
  const char* e = getenv("DFM_NAIVE_CLUSTER");
  return e != nullptr && e[0] == '0';
}

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
  // smallest cluster (<= 16 CTAs of ~200 KB) that holds the whole working set
  const uint64_t per_state = 8 + 4 + 4 + 4 * letters + 1;  // cells x2, labels x2, rows, flag
  const uint64_t kClusterSmem = 200ull << 10;
  const uint32_t S_max = (uint32_t)std::min<uint64_t>(kClusterSmem / per_state, 1u << 20);
  const uint32_t csize = (uint32_t)std::max<uint64_t>(1, ceil_div(n, std::max<uint32_t>(S_max, 1)));
  // Measured (B200, tools/dbg_cluster_time.py): the cluster wins only while the
  // instance fits one CTA — fib_dfa(17) (2,584 states, 2,583 passes) 7.7 vs 9.7 ms —
  // and loses beyond (random 8e3 states: 17.3 vs 7.0 ms in one CTA, 2e4 states: 52.7 vs
  // 18.4 ms over 3 CTAs): DSMEM random accesses and one SM's issue rate cap a pass
  // long before the grid barriers do.  So: single-CTA instances of <= 4096 states.
  if (!tracing_ && n <= kClusterMaxStates && csize == 1 && !cluster_disabled()) {
    const uint32_t S = (uint32_t)ceil_div(n, csize);
    const size_t smem = (size_t)S * per_state + 16;
    void (*kern)(ClusterArgs) =
        fused_cas ? cluster_pr_kernel<DFM_POLICY_ARBITRARY, true>
        : policy == DFM_POLICY_MIN ? cluster_pr_kernel<DFM_POLICY_MIN, false>
        : policy == DFM_POLICY_MAX ? cluster_pr_kernel<DFM_POLICY_MAX, false>
                                   : cluster_pr_kernel<DFM_POLICY_ARBITRARY, false>;
    DFM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DFM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    uint32_t* cout = reinterpret_cast<uint32_t*>(ctx.d_scalars + 20);
    const uint32_t kChunkMax = 1u << 16;
    uint32_t chunk = 64;
    while (true) {
      if (dl.expired()) {
        out.status = DFM_STATUS_TIMEOUT;
        return out;
      }
      ClusterArgs ca{rows, n, letters, S, lab[0], lab[1], pass, chunk, sel, cout};
      chunk = std::min(kChunkMax, chunk * 4);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(csize);
      cfg.blockDim = dim3(1024);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = ctx.stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = csize;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      ProfScope prof(ctx, "elect", 0);
      DFM_CUDA(cudaLaunchKernelEx(&cfg, kern, ca));
      DFM_LAUNCH_CHECK();
      prof.stop();
      DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 20, cout, 12, cudaMemcpyDeviceToHost, ctx.stream));
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
  const uint64_t persist_max = persistent_max_states();
  if (!tracing_ && !fused_cas && fused_enabled() && n <= persist_max) {
    // one barrier per pass (fused_pr_kernel), grid-stride over the resident threads.
    // Measured (B200, against the two-phase persistent kernel): C1 random_dfa(1e5, 2)
    // 95 -> 79 ms, vlts(1000, 1e6, 20) 66 -> 60 ms, transPR comb(1e6, 3) 12.8 -> 10.8 ms
    const uint32_t kChunkMax = 8192;
    uint32_t chunk = 16;
    uint32_t* chg = ctx.slot_t<uint32_t>("pr.pchanged", kChunkMax);
    uint32_t* pout = reinterpret_cast<uint32_t*>(ctx.d_scalars + 20);
    auto* cells1 = ctx.slot_t<unsigned long long>("pr.cells1", n);
    DFM_CUDA(cudaMemsetAsync(cells1, policy == DFM_POLICY_MIN ? 0xFF : 0x00, n * 8, ctx.stream));
    void (*kern_one)(FusedArgs) =
        policy == DFM_POLICY_MIN   ? fused_pr_kernel<DFM_POLICY_MIN, true>
        : policy == DFM_POLICY_MAX ? fused_pr_kernel<DFM_POLICY_MAX, true>
                                   : fused_pr_kernel<DFM_POLICY_ARBITRARY, true>;
    // a thread per state when the kOne variant holds all n resident
    const bool one = n <= fused_max_states(ctx, (const void*)kern_one) && one_enabled();
    const int gm = group_mode();
    const int lanes = (letters >= 8 && ((gm == 1 && !one) || gm == 2)) ? (letters >= 16 ? 8 : 4) : 1;
    void (*kern)(FusedArgs) =
        lanes == 8 ? (policy == DFM_POLICY_MIN   ? fused_group_kernel<DFM_POLICY_MIN, 8>
                      : policy == DFM_POLICY_MAX ? fused_group_kernel<DFM_POLICY_MAX, 8>
                                                 : fused_group_kernel<DFM_POLICY_ARBITRARY, 8>)
        : lanes == 4 ? (policy == DFM_POLICY_MIN   ? fused_group_kernel<DFM_POLICY_MIN, 4>
                        : policy == DFM_POLICY_MAX ? fused_group_kernel<DFM_POLICY_MAX, 4>
                                                   : fused_group_kernel<DFM_POLICY_ARBITRARY, 4>)
        : one ? kern_one
        : policy == DFM_POLICY_MIN ? fused_pr_kernel<DFM_POLICY_MIN, false>
        : policy == DFM_POLICY_MAX ? fused_pr_kernel<DFM_POLICY_MAX, false>
                                   : fused_pr_kernel<DFM_POLICY_ARBITRARY, false>;
    const unsigned pgrid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>(ceil_div(n * lanes, kPersistThreads),
                              fused_max_states(ctx, (const void*)kern) / kPersistThreads));
    const uint32_t *pred_off = nullptr, *pred_src = nullptr;
    uint32_t* mark = nullptr;
    uint32_t dirty_from = 0;
    const bool use_lmask = lanes == 1 && letters <= 32 && n < (1ull << kPredSrcBits) &&
                           lmask_enabled();
    // the predecessor lists pay off only over many passes: built once a run has gone
    // 64 passes without converging (transPR's few-pass runs never build them)
    auto build_dirty = [&]() {
      // predecessor lists over all letters (CSR by target), built once per run
      ProfScope p(ctx, "init", n * letters * 12 + n * 12);
      uint32_t* deg = ctx.slot_t<uint32_t>("pr.deg", n + 1);
      uint32_t* off = ctx.slot_t<uint32_t>("pr.poff", n + 1);
      uint32_t* cur = ctx.slot_t<uint32_t>("pr.pcur", n + 1);
      uint32_t* src = ctx.slot_t<uint32_t>("pr.psrc", std::max<uint64_t>(n * letters, 1));
      mark = ctx.slot_t<uint32_t>("pr.mark", n);
      DFM_CUDA(cudaMemsetAsync(deg, 0, (n + 1) * 4, ctx.stream));
      DFM_CUDA(cudaMemsetAsync(mark, 0, n * 4, ctx.stream));
      const unsigned g2 = (unsigned)std::min<uint64_t>(ceil_div(n * letters, 256), ctx.num_sms * 16ull);
      pred_count_kernel<<<g2, 256, 0, ctx.stream>>>(rows, n, letters, deg);
      DFM_LAUNCH_CHECK();
      prims::lookback_scan(ctx, "pr.degscan", n + 1, DegIn{deg}, DegOut{off, cur}, nullptr);
      if (use_lmask) {  // the marks become three letter-mask arrays
        mark = ctx.slot_t<uint32_t>("pr.lmask", 3 * n);
        DFM_CUDA(cudaMemsetAsync(mark, 0, 3 * n * 4, ctx.stream));
      }
      pred_fill_kernel<<<g2, 256, 0, ctx.stream>>>(rows, n, letters, cur, src, use_lmask);
      DFM_LAUNCH_CHECK();
      pred_off = off;
      pred_src = src;
      dirty_from = pass + 1;
    };
    while (true) {
      if (dl.expired()) {
        out.status = DFM_STATUS_TIMEOUT;
        return out;
      }
      if (mark == nullptr && pass >= dirty_after() && dirty_enabled(n, letters)) build_dirty();
      DFM_CUDA(cudaMemsetAsync(chg, 0, chunk * 4, ctx.stream));
      FusedArgs fa{rows, n,     letters, lab[0], lab[1], cells,    cells1,   chg,
                   pass, chunk, sel,     pout,   pred_off, pred_src, mark,   dirty_from,
                   own_label_on()};
      chunk = std::min(kChunkMax, chunk * 2);
      void* args[] = {&fa};
      // once the letter masks exist: the kMask variant (its own occupancy and kOne test)
      const void* lk = (const void*)kern;
      unsigned lgrid = pgrid;
      if (mark != nullptr && use_lmask) {
        void (*mk_one)(FusedArgs) =
            policy == DFM_POLICY_MIN   ? fused_pr_kernel<DFM_POLICY_MIN, true, true>
            : policy == DFM_POLICY_MAX ? fused_pr_kernel<DFM_POLICY_MAX, true, true>
                                       : fused_pr_kernel<DFM_POLICY_ARBITRARY, true, true>;
        void (*mk)(FusedArgs) =
            (one && n <= fused_max_states(ctx, (const void*)mk_one)) ? mk_one
            : policy == DFM_POLICY_MIN ? fused_pr_kernel<DFM_POLICY_MIN, false, true>
            : policy == DFM_POLICY_MAX ? fused_pr_kernel<DFM_POLICY_MAX, false, true>
                                       : fused_pr_kernel<DFM_POLICY_ARBITRARY, false, true>;
        lk = (const void*)mk;
        if (mk != mk_one && queue_enabled())
          lk = policy == DFM_POLICY_MIN   ? (const void*)queue_pr_kernel<DFM_POLICY_MIN>
               : policy == DFM_POLICY_MAX ? (const void*)queue_pr_kernel<DFM_POLICY_MAX>
                                          : (const void*)queue_pr_kernel<DFM_POLICY_ARBITRARY>;
        lgrid = (unsigned)std::max<uint64_t>(
            1, std::min<uint64_t>(ceil_div(n, kPersistThreads),
                                  fused_max_states(ctx, lk) / kPersistThreads));
      }
      ProfScope prof(ctx, "elect", 0);
      DFM_CUDA(cudaLaunchCooperativeKernel(lk, lgrid, kPersistThreads, args, 0, ctx.stream));
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
  if (!tracing_ && n <= persist_max) {
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
