// sortPR for small automata in ONE persistent cooperative kernel (included by
// sortpr_hash.cu inside its anonymous namespace).
//
// Below ~1e6 states a pass of the multi-kernel engine is launch- and
// host-sync-bound (C1, random_dfa(1e5, 2): ~0.1 ms per pass for ~1 us of
// work).  Here every pass is two grid-barrier phases of one kernel, with the
// whole working set (ids, two hash tables, leader flags) in L2:
//   A  insert  : key = (block[q], block[delta_a(q)] ...) packed exactly; equal keys
//                meet in a CTA shared-memory table first, then one global slot per
//                key and CTA collects the group size, the minimum member q and
//                whether it holds the old leader; the other table is cleared for
//                the next pass
//   B  resolve : the minimum member of each group that lacks the old leader takes
//                a fresh id (one atomic per CTA), becomes the leader and publishes
//                the id in the slot; the other members wait for it; singleton
//                groups leave
// Same groups, ids-up-to-renaming, leaders and pass count as the host-driven
// loop (min_sort.hpp:72-126).  States are visited in place (no active-list
// compaction: a finished state carries flag 0 and is skipped), so the minimum
// member is the minimum q.  A pass whose packed key would exceed 62 bits ends
// the kernel; the host loop continues from the same state.
#pragma once

constexpr uint32_t kSmallMaxStates = 1u << 20;
constexpr int kSmallThreads = 1024;
constexpr int kSmallPer = 8;  // states per thread (n <= grid * 1024 * 8)

struct SmallArgs {
  const uint32_t* delta;
  uint32_t n, k;
  uint32_t* block;
  uint8_t* lead;
  uint8_t* flag;  // 1 = still in a block of >= 2 states
  Slot* tab0;
  Slot* tab1;
  unsigned long long* ctr;  // [0..2] fresh ids, [3..5] survivors; rotating by pass % 3
  uint32_t* state;          // [0] B [1] passes so far [2] active states [3] 1 = fixpoint, 2 = wide keys
  uint32_t max_passes;
  uint64_t seed;
  uint32_t per_cta;   // states per CTA (<= kSmallThreads * kSmallPer)
  uint32_t tab_mask;  // shared table slots - 1 (power of two >= 2 * per_cta, <= kSmallTab)
  // first launch: initial partition in the prologue (first_states/init of the host loop)
  const uint8_t* acc;
  uint32_t* first2;  // [2 * grid]: each CTA's first accepting / rejecting state
  bool init;
  // fixpoint: canonical labels in the epilogue (rank of each block's leader)
  uint32_t* canon;
  uint32_t* cob;      // [n] canonical label of each block id
  uint32_t* cta_cnt;  // [gridDim.x] leaders per CTA
  unsigned long long* tdbg;  // DFM_SMALL_TIMING=1: globaltimer at each phase boundary
};

__device__ __forceinline__ unsigned long long small_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// table capacity for m inserted keys: load <= 0.4, whole 8-slot lines
__host__ __device__ __forceinline__ uint32_t small_cap(uint32_t m) {
  return m * 5u / 2u > 1024u ? ((m * 5u / 2u + 7u) & ~7u) : 1024u;
}

constexpr uint32_t kSmallTab = 8192;  // shared-memory aggregation slots per CTA
constexpr uint32_t kGlobalSlot = 0x80000000u;
constexpr unsigned long long kPublished = 1ull << 63;  // slot key = published id (keys < 2^62)

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
constexpr size_t kSmallSmem = kSmallTab * (8 + 4 + 4 + 4 + 4);

// claim (or find) the global slot of a key.  One CAS at the home slot; if another
// key holds it, the home's aligned 8-slot group (one 128-byte line) is read in one
// round trip and its first empty slot in group order is claimed, then the next
// group: the slowest thread of a pass decides the grid barrier, so probe chains are
// bounded by lines, not slots.  Every inserter of a key walks the same fixed order
// and slots never empty within a pass, so equal keys meet in one slot.
__device__ __forceinline__ uint32_t small_claim(Slot* T, uint32_t cap, unsigned long long key,
                                                uint64_t seed, uint32_t rep, uint32_t info) {
  // a new key installs {key, rep, info} with one 128-bit CAS; a key already present
  // merges its (rep, info) with two atomics
  const unsigned long long stored = key + 1ull;
  const unsigned long long val = (unsigned long long)rep | ((unsigned long long)info << 32);
  auto try_slot = [&](uint32_t t, bool& done) {
    unsigned long long olo, ohi;
    cas128(&T[t], 0ull, 0ull, stored, val, olo, ohi);
    if (olo == 0ull && ohi == 0ull) {
      done = true;
    } else if (olo == stored) {
      atomicMax(&T[t].rep, rep);
      atomicAdd(&T[t].info, info);
      done = true;
    }
  };
  uint32_t t = (uint32_t)__umul64hi(mix64(key ^ seed), cap);
  bool done = false;
  try_slot(t, done);
  if (done) return t;
  uint32_t g0 = t & ~7u;
  while (true) {
    unsigned long long ks[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) ks[e] = __ldcg(&T[g0 + e].key);
    int empty = -1, found = -1;
#pragma unroll
    for (int e = 7; e >= 0; --e) {
      if (ks[e] == stored) found = e;
      if (ks[e] == 0ull) empty = e;
    }
    if (found >= 0) {
      atomicMax(&T[g0 + found].rep, rep);
      atomicAdd(&T[g0 + found].info, info);
      return g0 + found;
    }
    if (empty < 0) {  // full line: the next one
      g0 += 8;
      if (g0 >= cap) g0 = 0;
      continue;
    }
    try_slot(g0 + empty, done);
    if (done) return g0 + empty;
    // lost the slot to another key: re-read the same line
  }
}

__global__ void __launch_bounds__(kSmallThreads, 1) small_sortpr_kernel(SmallArgs a) {
  extern __shared__ unsigned long long s_key[];  // [kSmallTab] key + 1 (0 = empty)
  uint32_t* s_rep = reinterpret_cast<uint32_t*>(s_key + kSmallTab);
  uint32_t* s_info = s_rep + kSmallTab;
  uint32_t* s_gs = s_info + kSmallTab;  // global slot of each shared slot
  uint32_t* s_list = s_gs + kSmallTab;  // occupied shared slots
  cg::grid_group g = cg::this_grid();
  const uint32_t nth = gridDim.x * blockDim.x;
  const uint32_t first = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  // CTA c owns states [c * per_cta, (c + 1) * per_cta): every SM gets a share
  const uint32_t base_q = blockIdx.x * a.per_cta + threadIdx.x;
  __shared__ uint32_t s_warp[kSmallThreads / 32 + 1];
  __shared__ uint32_t s_warp2[kSmallThreads / 32];
  __shared__ uint32_t s_base;
  __shared__ uint32_t s_cnt;  // occupied shared slots (flush list length)
  auto owned = [&](int j) { return threadIdx.x + j * kSmallThreads < a.per_cta &&
                                   base_q + j * kSmallThreads < a.n; };
  uint32_t B, pass, m;
  // the thread's own states live in registers across passes (only their owner
  // writes them); the global copies serve the successor gathers and a relaunch
  uint32_t myb[kSmallPer];  // block id
  uint32_t mys[kSmallPer];  // bit0 in a block of >= 2 states, bit1 leader
  if (a.init) {
    // initial partition {accepting, rejecting} and its leaders (min_sort.hpp:80-88)
    uint32_t fa = kNoLeader, fr = kNoLeader;
#pragma unroll
    for (int j = 0; j < kSmallPer; ++j) {
      const uint32_t q = base_q + j * kSmallThreads;
      if (owned(j)) {
        if (a.acc[q]) fa = min(fa, q);
        else fr = min(fr, q);
      }
    }
    // per-CTA minima (no pre-initialised global cell needed), reduced after the barrier
    fa = __reduce_min_sync(0xffffffffu, fa);
    fr = __reduce_min_sync(0xffffffffu, fr);
    if (lane == 0) {
      s_warp[threadIdx.x >> 5] = fa;
      s_warp2[threadIdx.x >> 5] = fr;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t x = threadIdx.x < kSmallThreads / 32 ? s_warp[threadIdx.x] : kNoLeader;
      uint32_t y = threadIdx.x < kSmallThreads / 32 ? s_warp2[threadIdx.x] : kNoLeader;
      x = __reduce_min_sync(0xffffffffu, x);
      y = __reduce_min_sync(0xffffffffu, y);
      if (threadIdx.x == 0) {
        a.first2[2 * blockIdx.x] = x;
        a.first2[2 * blockIdx.x + 1] = y;
      }
    }
    {
      const uint32_t cap0 = small_cap(a.n);
      uint4* z = reinterpret_cast<uint4*>(a.tab0);
      for (uint32_t s = first; s < cap0; s += nth) z[s] = make_uint4(0, 0, 0, 0);
      if (first < 6) a.ctr[first] = 0;
    }
    g.sync();
    fa = kNoLeader;
    fr = kNoLeader;
    for (uint32_t c = lane; c < gridDim.x; c += 32) {
      fa = min(fa, __ldcg(&a.first2[2 * c]));
      fr = min(fr, __ldcg(&a.first2[2 * c + 1]));
    }
    fa = __reduce_min_sync(0xffffffffu, fa);
    fr = __reduce_min_sync(0xffffffffu, fr);
    const bool split = fa != kNoLeader && fr != kNoLeader;
#pragma unroll
    for (int j = 0; j < kSmallPer; ++j) {
      const uint32_t q = base_q + j * kSmallThreads;
      myb[j] = 0;
      mys[j] = 0;
      if (owned(j)) {
        myb[j] = (split && a.acc[q] == 0) ? 1u : 0u;
        const bool ld = q == fa || q == fr || (!split && q == 0);
        mys[j] = 1u | (ld ? 2u : 0u);
        a.block[q] = myb[j];
        a.lead[q] = ld ? 1 : 0;
        a.flag[q] = 1;
      }
    }
    B = split ? 2u : 1u;
    pass = 0;
    m = a.n;
    g.sync();
  } else {
    B = a.state[0];
    pass = a.state[1];
    m = a.state[2];
#pragma unroll
    for (int j = 0; j < kSmallPer; ++j) {
      const uint32_t q = base_q + j * kSmallThreads;
      myb[j] = 0;
      mys[j] = 0;
      if (owned(j)) {
        myb[j] = a.block[q];
        mys[j] = (a.flag[q] ? 1u : 0u) | (a.lead[q] ? 2u : 0u);
      }
    }
  }
  uint32_t status = 0;
  const bool timing = a.tdbg != nullptr && first == 0;
  auto clear_shared = [&]() {
    for (uint32_t i = threadIdx.x; i <= a.tab_mask; i += blockDim.x) {
      s_key[i] = 0;
      s_rep[i] = 0;
      s_info[i] = 0;
    }
    if (threadIdx.x == 0) s_cnt = 0;
  };
  clear_shared();
  for (uint32_t it = 0; it < a.max_passes; ++it) {
    if (timing) a.tdbg[8 * it] = small_now();
    const int w = B <= 1 ? 1 : 32 - __clz(B - 1);
    if ((uint64_t)(a.k + 1) * (uint64_t)w > 62) {
      status = 2;
      break;
    }
    Slot* T = (pass & 1) ? a.tab1 : a.tab0;
    Slot* Tn = (pass & 1) ? a.tab0 : a.tab1;
    const uint32_t cap = small_cap(m);
    unsigned long long* fresh = a.ctr + pass % 3;
    unsigned long long* surv = a.ctr + 3 + pass % 3;
    if (first == 0) {  // last read two passes ago
      a.ctr[(pass + 1) % 3] = 0;
      a.ctr[3 + (pass + 1) % 3] = 0;
    }
    {  // clear the other table for the next pass (its states are a subset of these)
      uint4* z = reinterpret_cast<uint4*>(Tn);
      for (uint32_t s = first; s < cap; s += nth) z[s] = make_uint4(0, 0, 0, 0);
    }
    // ---- A: insert, aggregated per CTA in a shared-memory table first (early passes
    // have a few huge groups: one global atomic per group per CTA, not per state)
    unsigned long long keys[kSmallPer];
#pragma unroll
    for (int j = 0; j < kSmallPer; ++j) {  // all gathers of the thread in flight together
      const uint32_t q = base_q + j * kSmallThreads;
      keys[j] = myb[j];
      if (mys[j] & 1u)
        for (uint32_t x = 0; x < a.k; ++x)
          keys[j] = (keys[j] << w) | __ldcg(a.block + __ldg(a.delta + (uint64_t)x * a.n + q));
    }
    __syncthreads();
    uint32_t slot[kSmallPer];  // shared index, or global slot | kGlobalSlot
    uint32_t stat[kSmallPer];  // bit0 active, bit1 rep, bit2 keeper, bit3 singleton
#pragma unroll
    for (int j = 0; j < kSmallPer; ++j) {
      const uint32_t q = base_q + j * kSmallThreads;
      stat[j] = 0;
      slot[j] = 0;
      const bool act = (mys[j] & 1u) != 0;
      const uint32_t vmask = __ballot_sync(0xffffffffu, act);
      if (vmask == 0) continue;
      if (act) {
        const unsigned long long key = keys[j];
        // lanes with equal keys: the lowest (= minimum q) inserts for all
        const uint32_t peers = __match_any_sync(vmask, key);
        const uint32_t leads = __ballot_sync(vmask, (mys[j] & 2u) != 0) & peers;
        const int low = __ffs(peers) - 1;
        uint32_t t = 0;
        if (lane == (uint32_t)low) {
          const unsigned long long stored = key + 1ull;
          const uint32_t add = (uint32_t)__popc(peers) | (leads ? 0x80000000u : 0u);
          uint32_t h = (uint32_t)mix64(key ^ ~a.seed) & a.tab_mask;
          bool local = false;
          for (int probe = 0; probe < 32; ++probe) {
            const unsigned long long cur = atomicCAS(&s_key[h], 0ull, stored);
            if (cur == 0ull || cur == stored) {
              local = true;
              break;
            }
            h = (h + 1) & a.tab_mask;
          }
          if (local) {
            atomicMax(&s_rep[h], ~q);
            atomicAdd(&s_info[h], add);
            t = h;
          } else {  // crowded shared table: straight to the global one
            t = small_claim(T, cap, key, a.seed, ~q, add) | kGlobalSlot;
          }
        }
        slot[j] = __shfl_sync(vmask, t, low);
        stat[j] = 1;
      }
    }
    __syncthreads();
    if (timing) a.tdbg[8 * it + 4] = small_now();
    {  // the CTA's distinct keys, compacted (any order), then one global claim per thread
      for (uint32_t i0 = threadIdx.x & ~31u; i0 <= a.tab_mask; i0 += blockDim.x) {
        const uint32_t i = i0 + lane;
        const bool used = s_key[i] != 0ull;
        const uint32_t bal = __ballot_sync(0xffffffffu, used);
        uint32_t pos = 0;
        if (lane == 0 && bal) pos = atomicAdd(&s_cnt, (uint32_t)__popc(bal));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (used) s_list[pos + __popc(bal & ((1u << lane) - 1u))] = i;
      }
      __syncthreads();
      const uint32_t tot = s_cnt;
      for (uint32_t x = threadIdx.x; x < tot; x += blockDim.x) {
        const uint32_t i = s_list[x];
        s_gs[i] = small_claim(T, cap, s_key[i] - 1ull, a.seed, s_rep[i], s_info[i]);
      }
    }
    __syncthreads();
    if (timing) a.tdbg[8 * it + 5] = small_now();
#pragma unroll
    for (int j = 0; j < kSmallPer; ++j)
      if (stat[j]) slot[j] = (slot[j] & kGlobalSlot) ? (slot[j] & ~kGlobalSlot) : s_gs[slot[j]];
    clear_shared();  // (the claims above read it before the last block barrier)
    g.sync();
    if (timing) a.tdbg[8 * it + 1] = small_now();
    // ---- B: resolve
    uint32_t want = 0, survivors = 0;
#pragma unroll
    for (int j = 0; j < kSmallPer; ++j) {
      const uint32_t q = base_q + j * kSmallThreads;
      if (stat[j]) {
        const uint2 sl = __ldcg(reinterpret_cast<const uint2*>(&T[slot[j]].rep));
        const bool is_rep = ~sl.x == q;
        const bool keeper = (sl.y >> 31) != 0;
        const bool single = (sl.y & 0x7FFFFFFFu) == 1u;
        stat[j] |= (is_rep ? 2u : 0u) | (keeper ? 4u : 0u) | (single ? 8u : 0u);
        want += (is_rep && !keeper) ? 1u : 0u;
        if (single) {
          a.flag[q] = 0;
          mys[j] &= ~1u;
        } else {
          ++survivors;
        }
      }
    }
    {  // fresh ids and the survivor count: one atomic per CTA (16-bit fields, <= 8192 each)
      uint32_t tot;
      const uint32_t off = prims::block_exclusive_sum<kSmallThreads>(want | survivors << 16,
                                                                     s_warp, &tot);
      if (threadIdx.x == 0) {
        s_base = (tot & 0xFFFFu) ? (uint32_t)atomicAdd(fresh, (unsigned long long)(tot & 0xFFFFu))
                                 : 0u;
        if (tot >> 16) atomicAdd(surv, (unsigned long long)(tot >> 16));
      }
      __syncthreads();
      uint32_t gid = B + s_base + (off & 0xFFFFu);
#pragma unroll
      for (int j = 0; j < kSmallPer; ++j) {
        if ((stat[j] & 7u) == 3u) {  // rep of a group without the old leader
          const uint32_t q = base_q + j * kSmallThreads;
          a.block[q] = gid;
          a.lead[q] = 1;
          myb[j] = gid;
          mys[j] |= 2u;
          if (!(stat[j] & 8u)) st_relaxed_u64(&T[slot[j]].key, kPublished | gid);  // for the members
          ++gid;
        }
      }
    }
    // members of groups that took a fresh id wait for their rep's publication (a rep
    // publishes unconditionally after the CTA scan above; all CTAs are co-resident)
#pragma unroll
    for (int j = 0; j < kSmallPer; ++j) {
      if ((stat[j] & 7u) == 1u) {  // active, not the rep, group without the old leader
        unsigned long long v = ld_relaxed_u64(&T[slot[j]].key);
        while (!(v & kPublished)) v = ld_relaxed_u64(&T[slot[j]].key);
        myb[j] = (uint32_t)v;
        a.block[base_q + j * kSmallThreads] = myb[j];
      }
    }
    g.sync();
    if (timing) a.tdbg[8 * it + 2] = small_now();
    const uint32_t nfresh = (uint32_t)__ldcg(fresh);
    ++pass;
    if (nfresh == 0) {  // fixpoint: min_sort.hpp:111-117
      status = 1;
      break;
    }
    B += nfresh;
    m = (uint32_t)__ldcg(surv);
  }
  if (status == 1) {
    // canonical labels: block -> rank of its leader (minimum state) among all leaders,
    // ranks in q order: CTA ranges are contiguous, chunks j ascend within a CTA
    if (B == a.n) {  // all singletons: the identity
#pragma unroll
      for (int j = 0; j < kSmallPer; ++j)
        if (owned(j)) a.canon[base_q + j * kSmallThreads] = base_q + j * kSmallThreads;
    } else {
      uint32_t rank[kSmallPer];
      uint32_t run = 0;
#pragma unroll
      for (int j = 0; j < kSmallPer; ++j) {
        const uint32_t v = (mys[j] >> 1) & 1u;
        uint32_t tot;
        const uint32_t e = prims::block_exclusive_sum<kSmallThreads>(v, s_warp, &tot);
        rank[j] = v ? run + e : kNoLeader;
        run += tot;
      }
      if (threadIdx.x == 0) a.cta_cnt[blockIdx.x] = run;
      g.sync();
      uint32_t before = 0;
      for (uint32_t c = threadIdx.x; c < blockIdx.x; c += blockDim.x) before += __ldcg(a.cta_cnt + c);
      uint32_t tot;
      prims::block_exclusive_sum<kSmallThreads>(before, s_warp, &tot);
#pragma unroll
      for (int j = 0; j < kSmallPer; ++j)
        if (rank[j] != kNoLeader)
          a.cob[myb[j]] = tot + rank[j];
      g.sync();
#pragma unroll
      for (int j = 0; j < kSmallPer; ++j) {
        const uint32_t q = base_q + j * kSmallThreads;
        if (owned(j)) a.canon[q] = __ldcg(a.cob + myb[j]);
      }
    }
  }
  if (first == 0) {
    a.state[0] = B;
    a.state[1] = pass;
    a.state[2] = m;
    a.state[3] = status;
  }
}
