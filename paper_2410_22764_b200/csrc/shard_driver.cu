// State-sharded sortPR driver in C++ over the
// context's communicator (comm.cuh: NCCL in production, in-process threads in the
// single-GPU tests), behind the C-ABI dfm_sort_pr_sharded[_dev] (include/dfm.h).
//
// Rank r owns the contiguous states [r*S, min(n, (r+1)*S)), S = ceil(n/world), and
// their rows (GLOBAL target ids).  Each pass of the reference loop
// (min_sort.hpp:93-118):
//   1. all-gather the owned block ids bit-packed at the narrowest width holding B
//      ids (1/2/4/8/16/32 bits) -> the full id vector on every rank  [NVLink]
//   2. per owned state its key: the exact packed (block, successor ids) while
//      (k+1)*bits(B-1) <= 63, else a 64-bit hash + the signature row, and the
//      rank dest(key) that groups it                                  [HBM, gathers]
//   3. stable partition of the owned states by dest (radix sort on the dest bits),
//      counts exchanged, one all-to-all of keys (+ rows)             [NVLink]
//   4. exact grouping of the received keys (shard_group: uniqueness filter + hash
//      table; equal hashes verified against the rows — a collision anywhere voids
//      the pass on every rank and it is redone under a new seed)
//   5. per-rank group counts all-gathered -> dense global ids (rank offsets), the
//      ids go back to the owners in the reverse all-to-all           [NVLink]
//   6. fixpoint when the global count did not grow (fresh == num_blocks); a pass
//      that leaves every block a singleton is followed by the counted fixpoint
//      pass without running it, as in the single-GPU engine.
// Grouping is by exact key equality, so the partition sequence and the pass count
// are the reference's for every world size.  Canonical labels: identity when all
// blocks are singletons, else every rank reduces the minimum member of each block
// (all-reduce min over B u32), marks those minima in an n-bit bitmap and ranks
// them with a prefix popcount (core.hpp:123-136: block = rank of its minimum).
// Host syncs per pass: the destination counts, the group counts (both a few
// bytes), nothing else.
#include <algorithm>
#include <cstring>
#include <vector>

#include "comm.cuh"
#include "prims.cuh"

struct dfm_ctx {};

namespace dfm {
namespace {

constexpr uint64_t kShardSeed0 = 0x5EED0001ull;

unsigned sgrid(const Ctx& ctx, uint64_t items) {
  return (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(items, 1), 256),
                                      (uint64_t)ctx.num_sms * 16);
}
int bitw(uint64_t x) { return x == 0 ? 0 : 64 - __builtin_clzll(x); }

__device__ __forceinline__ uint64_t dmix64(uint64_t z) {  // = shard.cu mix64
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

bool shard_blocked_enabled() {
  const char* e = getenv("DFM_SHARD_BLOCKED");
  return e == nullptr || e[0] != '0';
}

__global__ void count_acc_kernel(const uint8_t* __restrict__ acc, uint64_t n,
                                 unsigned long long* out) {
  uint32_t c = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    c += acc[i] != 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

__global__ void bad_target_kernel(const uint32_t* __restrict__ delta, uint64_t total,
                                  uint64_t n_total, unsigned long long* bad) {
  bool b = false;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
    b |= delta[i] >= n_total;
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1ull);
}

__global__ void init_block_kernel(const uint8_t* __restrict__ acc, uint64_t n, bool split,
                                  uint32_t* __restrict__ block) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    block[i] = split ? (acc[i] == 0 ? 1u : 0u) : 0u;  // min_sort.hpp:80-88
}

// this rank's ids packed at kBits per state (32/kBits per word; S is a multiple of 32)
template <int kBits>
__global__ void pack_ids_kernel(const uint32_t* __restrict__ block, uint64_t n, uint64_t S,
                                uint32_t* __restrict__ out) {
  constexpr uint32_t per = 32 / kBits;
  const uint64_t words = S / per;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
    uint32_t word = 0;
#pragma unroll
    for (uint32_t e = 0; e < per; ++e) {
      const uint64_t i = w * per + e;
      if (i < n) word |= (kBits == 32 ? block[i] : block[i] << (e * kBits));
    }
    out[w] = word;
  }
}

__global__ void dest_hist_kernel(const uint32_t* __restrict__ dest, uint64_t n, uint32_t world,
                                 unsigned long long* __restrict__ counts,
                                 unsigned long long* __restrict__ dest64) {
  __shared__ uint32_t s[64];
  if (threadIdx.x < 64) s[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t d = dest[i];
    dest64[i] = d;
    atomicAdd(&s[d], 1u);
  }
  __syncthreads();
  if (threadIdx.x < world && s[threadIdx.x])
    atomicAdd(&counts[threadIdx.x], (unsigned long long)s[threadIdx.x]);
}

__global__ void permute_kernel(const uint32_t* __restrict__ order, uint64_t n,
                               const unsigned long long* __restrict__ keys,
                               const uint32_t* __restrict__ sig, uint32_t words,
                               unsigned long long* __restrict__ keys_out,
                               uint32_t* __restrict__ sig_out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t o = order[i];
    keys_out[i] = keys[o];
    for (uint32_t x = 0; x < words; ++x) sig_out[i * words + x] = sig[(uint64_t)o * words + x];
  }
}

__global__ void add_kernel(uint32_t* __restrict__ v, uint64_t n, uint32_t off) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) v[i] += off;
}

__global__ void scatter_back_kernel(const uint32_t* __restrict__ order,
                                    const uint32_t* __restrict__ back, uint64_t n,
                                    uint32_t* __restrict__ block) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    block[order[i]] = back[i];
}

// keys from the blocked builder -> the shard kernels' conventions (packed keys + 1,
// hashed keys | 1: never 0, the empty-slot mark) and the grouping rank of each key
__global__ void key_fix_dest_kernel(unsigned long long* __restrict__ keys, uint64_t n, bool packed,
                                    uint32_t ranks, uint32_t* __restrict__ dest) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned long long key = keys[i];
    keys[i] = packed ? key + 1ull : (key | 1ull);
    if (ranks > 1) dest[i] = (uint32_t)__umul64hi(dmix64(key ^ 0xD1B54A32D192ED03ull), ranks);
  }
}

__global__ void iota_kernel(uint32_t* __restrict__ out, uint64_t n, uint64_t lo) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (uint32_t)(lo + i);
}

__global__ void block_min_kernel(const uint32_t* __restrict__ block, uint64_t n, uint64_t lo,
                                 uint32_t* __restrict__ minidx) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t b = block[i];
    const uint32_t peers = __match_any_sync(__activemask(), b);  // lanes ascend in q
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1) && minidx[b] > (uint32_t)(lo + i))
      atomicMin(&minidx[b], (uint32_t)(lo + i));
  }
}

__global__ void leader_bits_kernel(const uint32_t* __restrict__ minidx, uint64_t B,
                                   uint32_t* __restrict__ bits) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += stride) {
    const uint32_t m = minidx[b];
    atomicOr(&bits[m >> 5], 1u << (m & 31));
  }
}

struct PopIn {
  const uint32_t* bits;
  __device__ uint32_t operator()(uint64_t w) const { return __popc(bits[w]); }
};
struct PopOut {
  uint32_t* prefix;
  __device__ void operator()(uint64_t w, uint32_t excl, uint32_t) const { prefix[w] = excl; }
};

__global__ void canon_kernel(const uint32_t* __restrict__ block, uint64_t n,
                             const uint32_t* __restrict__ minidx, const uint32_t* __restrict__ bits,
                             const uint32_t* __restrict__ prefix, uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t m = minidx[block[i]];
    out[i] = prefix[m >> 5] + __popc(bits[m >> 5] & ((1u << (m & 31)) - 1u));
  }
}

struct Agree {  // per-rank scalars exchanged once per pass
  uint64_t groups, collision, expired;
};

}  // namespace

AlgoOut run_sort_pr_sharded(Ctx& ctx, uint64_t n_total, const DevDfa& loc, const Deadline& dl,
                            uint32_t* canon_dev, bool force_protocol, bool validate) {
  if (ctx.comm == nullptr) throw Error(DFM_ERR_INVALID, "not a sharded context");
  Comm& comm = *ctx.comm;
  const int world = comm.world, rank = comm.rank;
  const uint64_t S = shard_size(n_total, world);
  const uint64_t lo = std::min<uint64_t>(n_total, (uint64_t)rank * S);
  const uint64_t nl = std::min<uint64_t>(n_total, lo + S) - lo;
  const uint32_t k = loc.k;
  if (n_total < 1 || n_total > 0xFFFFFFFFull) throw Error(DFM_ERR_INVALID, "n_total out of range");
  if (loc.n != nl) throw Error(DFM_ERR_INVALID, "local rows do not match this rank's shard");
  AlgoOut out;
  out.peak_memory_estimate = n_total * (16 + 4ull * k);  // min_sort.hpp:121
  if (world == 1 && !force_protocol) {
    // one rank owns every state: the single-GPU engine is the sharded pass at world 1
    AlgoOut o = run_sort_pr_hash(ctx, loc, dl, nullptr);
    if (o.status == DFM_STATUS_OK) {
      if (o.canon_identity) {
        iota_kernel<<<sgrid(ctx, nl), 256, 0, ctx.stream>>>(canon_dev, nl, 0);
        DFM_LAUNCH_CHECK();
      } else {
        DFM_CUDA(cudaMemcpyAsync(canon_dev, o.canon_dev, nl * 4, cudaMemcpyDeviceToDevice,
                                 ctx.stream));
      }
    }
    o.canon_dev = canon_dev;
    o.canon_identity = false;
    return o;
  }
  cudaStream_t st = ctx.stream;
  uint64_t* sc = ctx.d_scalars + 56;  // [0] accepting count [1] out-of-range target seen
  // ---- init: two blocks iff both acceptance classes are non-empty (min_sort.hpp:80-88)
  DFM_CUDA(cudaMemsetAsync(sc, 0, 16, st));
  if (nl) {
    count_acc_kernel<<<sgrid(ctx, nl), 256, 0, st>>>(loc.acc, nl,
                                                       reinterpret_cast<unsigned long long*>(sc));
    DFM_LAUNCH_CHECK();
    // host input is checked like dfm_sort_pr's upload; a device-resident shard is
    // trusted like dfm_run_algorithm_dev's
    if (validate) {
      bad_target_kernel<<<sgrid(ctx, nl * k), 256, 0, st>>>(
          loc.delta, nl * k, n_total, reinterpret_cast<unsigned long long*>(sc + 1));
      DFM_LAUNCH_CHECK();
    }
  }
  DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 56, sc, 16, cudaMemcpyDeviceToHost, st));
  ctx.sync();
  std::vector<uint64_t> all(3 * (size_t)world);
  {
    const uint64_t mine[2] = {ctx.h_scalars[56], ctx.h_scalars[57]};
    comm.all_gather_host(mine, all.data(), 2, st);
  }
  uint64_t n_acc = 0;
  bool bad = false;
  for (int r = 0; r < world; ++r) {
    n_acc += all[2 * r];
    bad |= all[2 * r + 1] != 0;
  }
  if (bad) throw Error(DFM_ERR_INVALID, "transition target out of range");
  const bool split = n_acc > 0 && n_acc < n_total;
  uint32_t* block = ctx.slot_t<uint32_t>("sd.block", std::max<uint64_t>(nl, 1));
  if (nl) {
    init_block_kernel<<<sgrid(ctx, nl), 256, 0, st>>>(loc.acc, nl, split, block);
    DFM_LAUNCH_CHECK();
  }
  uint64_t B = split ? 2 : 1;
  uint64_t seed = kShardSeed0;
  // blocked signature builder over the owned rows (targets = all n_total states): used
  // only when EVERY rank could build it, so all ranks make keys the same way
  struct LayHolder {
    ShardLayout* p = nullptr;
    ~LayHolder() { shard_layout_free(p); }
  } lay;
  if (shard_blocked_enabled()) {
    ProfScope p(ctx, "layout", nl * k * 16ull);
    lay.p = shard_layout_build(ctx, loc, n_total);
  }
  {
    const uint64_t mine = lay.p != nullptr ? 1 : 0;
    comm.all_gather_host(&mine, all.data(), 1, st);
    bool every = true;
    for (int r = 0; r < world; ++r) every = every && all[r] != 0;
    if (!every) {
      shard_layout_free(lay.p);
      lay.p = nullptr;
    }
  }
  const int dbits = std::max(1, bitw((uint64_t)world - 1));
  auto* counts_dev = reinterpret_cast<unsigned long long*>(ctx.slot_t<uint64_t>("sd.counts", 64));
  std::vector<uint64_t> send_cnt(world), recv_cnt(world), so(world), sb(world), ro(world),
      rb(world), cnt_all((size_t)world * world);
  bool identity = false;
  while (true) {
    // ---- 1. all-gather of the owned ids at the narrowest width
    const int w = std::max(1, bitw(B - 1));
    const bool packed = (uint64_t)(k + 1) * w <= 63;
    // ids travel (and are gathered) at 1/2/4/8/16/32 bits: pass 1's vector is a bitmap
    const uint32_t ib = B <= 2 ? 1 : B <= 16 ? 4 : B <= 256 ? 8 : B <= 65536 ? 16 : 32;
    const uint64_t slice = S * ib / 8;  // bytes per rank
    void* send_ids = ctx.slot("sd.ids_send", slice);
    void* full = ctx.slot("sd.ids_full", (uint64_t)world * slice);
    {
      ProfScope p(ctx, "allgather", slice * (uint64_t)world);
      const unsigned g = sgrid(ctx, S * ib / 32);
      auto* sw = static_cast<uint32_t*>(send_ids);
      switch (ib) {
        case 1: pack_ids_kernel<1><<<g, 256, 0, st>>>(block, nl, S, sw); break;
        case 2: pack_ids_kernel<2><<<g, 256, 0, st>>>(block, nl, S, sw); break;
        case 4: pack_ids_kernel<4><<<g, 256, 0, st>>>(block, nl, S, sw); break;
        case 8: pack_ids_kernel<8><<<g, 256, 0, st>>>(block, nl, S, sw); break;
        case 16: pack_ids_kernel<16><<<g, 256, 0, st>>>(block, nl, S, sw); break;
        default: pack_ids_kernel<32><<<g, 256, 0, st>>>(block, nl, S, sw); break;
      }
      DFM_LAUNCH_CHECK();
      comm.all_gather(send_ids, full, slice, st);
    }
    // ---- 2. keys (+ rows) and destinations of the owned states
    const uint32_t words = packed ? 0 : k + 1;
    auto* keys = ctx.slot_t<unsigned long long>("sd.keys", std::max<uint64_t>(nl, 1));
    uint32_t* sig = words ? ctx.slot_t<uint32_t>("sd.sig", std::max<uint64_t>(nl * words, 1)) : nullptr;
    uint32_t* dest = ctx.slot_t<uint32_t>("sd.dest", std::max<uint64_t>(nl, 1));
    if (lay.p != nullptr && (uint64_t)n_total * ib / 8 > (32ull << 20) && nl > 0) {
      // the gathered vector is past the L2 plateau: shared-memory gathers per target range
      shard_layout_keys(ctx, lay.p, (int)ib, static_cast<const uint32_t*>(full), block, nl, w,
                        !packed, seed, keys, sig, k + 1);
      key_fix_dest_kernel<<<sgrid(ctx, nl), 256, 0, st>>>(keys, nl, packed, (uint32_t)world, dest);
      DFM_LAUNCH_CHECK();
    } else {
      shard_signature(ctx, loc.delta, nl, k, full, ib, lo, seed, (uint32_t)world,
                      packed ? (uint32_t)w : 0u, keys, sig, dest);
    }
    // ---- 3. route to the grouping ranks
    const unsigned long long* rkeys = keys;
    const uint32_t* rsig = sig;
    uint64_t nrecv = nl;
    uint32_t* order = nullptr;
    if (world > 1) {
      ProfScope p(ctx, "route", nl * (16ull + 8 + 4ull * words) * 2);
      auto* d64 = ctx.slot_t<uint64_t>("sd.d64", std::max<uint64_t>(nl, 1));
      auto* d64b = ctx.slot_t<uint64_t>("sd.d64b", std::max<uint64_t>(nl, 1));
      uint32_t* ord_a = ctx.slot_t<uint32_t>("sd.ord_a", std::max<uint64_t>(nl, 1));
      uint32_t* ord_b = ctx.slot_t<uint32_t>("sd.ord_b", std::max<uint64_t>(nl, 1));
      DFM_CUDA(cudaMemsetAsync(counts_dev, 0, 8ull * world, st));
      if (nl) {
        dest_hist_kernel<<<sgrid(ctx, nl), 256, 0, st>>>(dest, nl, (uint32_t)world, counts_dev,
                                                           reinterpret_cast<unsigned long long*>(d64));
        DFM_LAUNCH_CHECK();
      }
      const bool alt = nl ? prims::radix_sort_pairs(ctx, d64, ord_a, d64b, ord_b, nl, dbits, true)
                          : false;
      order = alt ? ord_b : ord_a;
      DFM_CUDA(cudaMemcpyAsync(send_cnt.data(), counts_dev, 8ull * world, cudaMemcpyDeviceToHost,
                               st));
      ctx.sync();
      comm.all_gather_host(send_cnt.data(), cnt_all.data(), world, st);
      nrecv = 0;
      for (int r = 0; r < world; ++r) {
        recv_cnt[r] = cnt_all[(size_t)r * world + rank];
        nrecv += recv_cnt[r];
      }
      auto* skeys = ctx.slot_t<unsigned long long>("sd.skeys", std::max<uint64_t>(nl, 1));
      uint32_t* ssig = words ? ctx.slot_t<uint32_t>("sd.ssig", std::max<uint64_t>(nl * words, 1)) : nullptr;
      if (nl) {
        permute_kernel<<<sgrid(ctx, nl), 256, 0, st>>>(order, nl, keys, sig, words, skeys, ssig);
        DFM_LAUNCH_CHECK();
      }
      auto* rk = ctx.slot_t<unsigned long long>("sd.rkeys", std::max<uint64_t>(nrecv, 1));
      uint32_t* rs = words ? ctx.slot_t<uint32_t>("sd.rsig", std::max<uint64_t>(nrecv * words, 1)) : nullptr;
      auto offsets = [&](const std::vector<uint64_t>& c, uint64_t unit, std::vector<uint64_t>& off,
                         std::vector<uint64_t>& bytes) {
        uint64_t o = 0;
        for (int r = 0; r < world; ++r) {
          off[r] = o * unit;
          bytes[r] = c[r] * unit;
          o += c[r];
        }
      };
      offsets(send_cnt, 8, so, sb);
      offsets(recv_cnt, 8, ro, rb);
      comm.all_to_all(skeys, so.data(), sb.data(), rk, ro.data(), rb.data(), st);
      if (words) {
        offsets(send_cnt, 4ull * words, so, sb);
        offsets(recv_cnt, 4ull * words, ro, rb);
        comm.all_to_all(ssig, so.data(), sb.data(), rs, ro.data(), rb.data(), st);
      }
      rkeys = rk;
      rsig = rs;
    }
    // ---- 4. exact grouping at this rank
    uint32_t* label = ctx.slot_t<uint32_t>("sd.label", std::max<uint64_t>(nrecv, 1));
    uint64_t groups = 0;
    int coll = 0;
    const uint64_t kbits = (uint64_t)(k + 1) * w;
    if (packed && kbits <= 30 && (1ull << kbits) <= std::max<uint64_t>(16 * nrecv, 1ull << 20))
      shard_group_direct(ctx, rkeys, nrecv, (uint32_t)kbits, label, &groups);
    else
      shard_group(ctx, rkeys, rsig, words, nrecv, label, &groups, &coll);
    Agree mine{groups, (uint64_t)coll, (uint64_t)dl.expired()};
    comm.all_gather_host(&mine.groups, all.data(), 3, st);
    bool any_coll = false, any_expired = false;
    uint64_t offset = 0, B_new = 0;
    for (int r = 0; r < world; ++r) {
      any_coll |= all[3 * r + 1] != 0;
      any_expired |= all[3 * r + 2] != 0;
      if (r < rank) offset += all[3 * r];
      B_new += all[3 * r];
    }
    if (any_expired) {
      out.status = DFM_STATUS_TIMEOUT;
      return out;
    }
    if (any_coll) {  // a hash collision on any rank voids the pass everywhere
      seed = seed * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
      continue;
    }
    // ---- 5. dense global ids back to the owners
    if (nrecv && offset) {
      add_kernel<<<sgrid(ctx, nrecv), 256, 0, st>>>(label, nrecv, (uint32_t)offset);
      DFM_LAUNCH_CHECK();
    }
    if (world == 1) {
      DFM_CUDA(cudaMemcpyAsync(block, label, nl * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      ProfScope p(ctx, "route", (nl + nrecv) * 8ull);
      uint32_t* back = ctx.slot_t<uint32_t>("sd.back", std::max<uint64_t>(nl, 1));
      uint64_t o = 0, o2 = 0;
      for (int r = 0; r < world; ++r) {
        so[r] = o * 4;
        sb[r] = recv_cnt[r] * 4;
        o += recv_cnt[r];
        ro[r] = o2 * 4;
        rb[r] = send_cnt[r] * 4;
        o2 += send_cnt[r];
      }
      comm.all_to_all(label, so.data(), sb.data(), back, ro.data(), rb.data(), st);
      if (nl) {
        scatter_back_kernel<<<sgrid(ctx, nl), 256, 0, st>>>(order, back, nl, block);
        DFM_LAUNCH_CHECK();
      }
    }
    ++out.iterations;
    if (B_new == B) break;  // fixpoint, min_sort.hpp:111-117
    B = B_new;
    if (B == n_total) {
      // every block a singleton: the next pass grows nothing and ends the loop —
      // counted, not run (as the single-GPU engine does)
      ++out.iterations;
      ++out.skipped_passes;
      identity = true;
      break;
    }
  }
  // ---- canonical labels (core.hpp:123-136)
  if (identity) {
    if (nl) {
      iota_kernel<<<sgrid(ctx, nl), 256, 0, st>>>(canon_dev, nl, lo);
      DFM_LAUNCH_CHECK();
    }
  } else {
    ProfScope p(ctx, "canon", nl * 16 + B * 12 + n_total / 4);
    uint32_t* minidx = ctx.slot_t<uint32_t>("sd.minidx", B);
    DFM_CUDA(cudaMemsetAsync(minidx, 0xFF, B * 4, st));
    if (nl) {
      block_min_kernel<<<sgrid(ctx, nl), 256, 0, st>>>(block, nl, lo, minidx);
      DFM_LAUNCH_CHECK();
    }
    comm.all_reduce_min_u32(minidx, B, st);
    const uint64_t words = ceil_div(n_total, 32);
    uint32_t* bits = ctx.slot_t<uint32_t>("sd.lbits", words);
    uint32_t* prefix = ctx.slot_t<uint32_t>("sd.lpref", words);
    DFM_CUDA(cudaMemsetAsync(bits, 0, words * 4, st));
    leader_bits_kernel<<<sgrid(ctx, B), 256, 0, st>>>(minidx, B, bits);
    DFM_LAUNCH_CHECK();
    prims::lookback_scan(ctx, "sd.lscan", words, PopIn{bits}, PopOut{prefix}, nullptr);
    if (nl) {
      canon_kernel<<<sgrid(ctx, nl), 256, 0, st>>>(block, nl, minidx, bits, prefix, canon_dev);
      DFM_LAUNCH_CHECK();
    }
  }
  out.num_blocks = (uint32_t)B;
  out.canon_dev = canon_dev;
  out.status = DFM_STATUS_OK;
  return out;
}

}  // namespace dfm

// ------------------------------------------------------------------ C-ABI
using namespace dfm;

namespace {
template <class F>
int guarded_sd(dfm_ctx* c, F&& f) {
  Ctx* ctx = reinterpret_cast<Ctx*>(c);
  if (ctx == nullptr) return DFM_ERR_INVALID;
  std::lock_guard<std::mutex> lk(ctx->mu);
  try {
    DFM_CUDA(cudaSetDevice(ctx->device));
    f(*ctx);
    ctx->harvest();
    return DFM_OK;
  } catch (const Error& e) {
    ctx->last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    ctx->last_error = e.what();
    return DFM_ERR_INVALID;
  }
}

void fill_stats(const AlgoOut& o, const Deadline& dl, dfm_stats* st) {
  if (!st) return;
  st->iterations = o.iterations;
  st->executed_passes = o.iterations - o.skipped_passes;
  st->closure_steps = 0;
  st->peak_memory_estimate = o.peak_memory_estimate;
  st->status = o.status;
  st->elapsed_ms = dl.elapsed();
}

bool force_protocol() {
  const char* e = getenv("DFM_SHARD_PROTOCOL");
  return e != nullptr && e[0] == '1';
}

// canonical labels of this rank (device) -> host: own slice, or the whole partition
// (all-gathered over the ranks) when gather_all
void labels_out(Ctx& ctx, const uint32_t* canon, uint64_t n_total, uint64_t nl, bool gather_all,
                uint32_t* host) {
  if (!gather_all || ctx.comm->world == 1) {
    DFM_CUDA(cudaMemcpyAsync(host, canon, nl * 4, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    return;
  }
  const uint64_t S = shard_size(n_total, ctx.comm->world);
  uint32_t* send = ctx.slot_t<uint32_t>("sd.out_send", S);
  uint32_t* full = ctx.slot_t<uint32_t>("sd.out_full", S * ctx.comm->world);
  DFM_CUDA(cudaMemcpyAsync(send, canon, nl * 4, cudaMemcpyDeviceToDevice, ctx.stream));
  ctx.comm->all_gather(send, full, S * 4, ctx.stream);
  DFM_CUDA(cudaMemcpyAsync(host, full, n_total * 4, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
}
}  // namespace

extern "C" {

int dfm_nccl_get_unique_id(uint8_t* id_out) {
  if (id_out == nullptr) return DFM_ERR_INVALID;
  try {
    nccl_unique_id(id_out);
    return DFM_OK;
  } catch (const Error& e) {
    return e.code;
  }
}

static int create_sharded(int device, int rank, int world, dfm_ctx** out,
                          Comm* (*make)(int, int, int, const void*), const void* arg) {
  if (out == nullptr || world < 1 || rank < 0 || rank >= world || world > 64)
    return DFM_ERR_INVALID;
  *out = nullptr;
  dfm_ctx* c = nullptr;
  const int rc = dfm_ctx_create(device, &c);
  if (rc != DFM_OK) return rc;
  try {
    DFM_CUDA(cudaSetDevice(device));
    reinterpret_cast<Ctx*>(c)->comm = make(device, rank, world, arg);
  } catch (const Error& e) {
    dfm_ctx_destroy(c);
    return e.code;
  }
  *out = c;
  return DFM_OK;
}

int dfm_ctx_create_sharded(int device, int rank, int world, const uint8_t* nccl_id,
                           dfm_ctx** out) {
  if (nccl_id == nullptr) return DFM_ERR_INVALID;
  return create_sharded(device, rank, world, out,
                        [](int d, int r, int w, const void* id) {
                          return make_nccl_comm(d, r, w, static_cast<const uint8_t*>(id));
                        },
                        nccl_id);
}

int dfm_ctx_create_sharded_local(int device, int rank, int world, const char* group,
                                 dfm_ctx** out) {
  if (group == nullptr) return DFM_ERR_INVALID;
  return create_sharded(device, rank, world, out,
                        [](int, int r, int w, const void* g) {
                          return make_local_comm(static_cast<const char*>(g), r, w);
                        },
                        group);
}

int dfm_ctx_shard_info(const dfm_ctx* c, int* rank, int* world, const char** transport) {
  const Ctx* ctx = reinterpret_cast<const Ctx*>(c);
  if (ctx == nullptr) return DFM_ERR_INVALID;
  if (rank) *rank = ctx->comm ? ctx->comm->rank : 0;
  if (world) *world = ctx->comm ? ctx->comm->world : 1;
  if (transport) *transport = ctx->comm ? ctx->comm->kind() : "none";
  return DFM_OK;
}

void dfm_shard_bounds(uint64_t n_total, int world, int rank, uint64_t* lo, uint64_t* hi) {
  const uint64_t S = shard_size(n_total, std::max(1, world));
  const uint64_t l = std::min<uint64_t>(n_total, (uint64_t)std::max(0, rank) * S);
  if (lo) *lo = l;
  if (hi) *hi = std::min<uint64_t>(n_total, l + S);
}

int dfm_sort_pr_sharded_dev(dfm_ctx* c, uint64_t n_total, uint32_t n_local, uint32_t k,
                            const void* delta_dev, const void* acc_dev, void* block_out_dev,
                            uint32_t* num_blocks_out, int64_t timeout_ms, dfm_stats* stats) {
  return guarded_sd(c, [&](Ctx& ctx) {
    if (ctx.comm == nullptr) throw Error(DFM_ERR_INVALID, "not a sharded context");
    const Deadline dl(timeout_ms);
    DevDfa loc;
    loc.n = n_local;
    loc.k = k;
    loc.delta = static_cast<uint32_t*>(const_cast<void*>(delta_dev));
    loc.acc = static_cast<uint8_t*>(const_cast<void*>(acc_dev));
    loc.owns = false;
    AlgoOut o = run_sort_pr_sharded(ctx, n_total, loc, dl,
                                    static_cast<uint32_t*>(block_out_dev), force_protocol(),
                                    /*validate=*/false);
    ctx.sync();
    if (num_blocks_out) *num_blocks_out = o.status == DFM_STATUS_OK ? o.num_blocks : 0;
    fill_stats(o, dl, stats);
  });
}

int dfm_sort_pr_sharded(dfm_ctx* c, uint64_t n_total, const dfm_dfa* local, int gather_all,
                        uint32_t* block_out, uint32_t* num_blocks_out, int64_t timeout_ms,
                        dfm_stats* stats) {
  return guarded_sd(c, [&](Ctx& ctx) {
    if (ctx.comm == nullptr) throw Error(DFM_ERR_INVALID, "not a sharded context");
    if (local == nullptr || local->accepting == nullptr || (local->alphabet_size && !local->delta))
      throw Error(DFM_ERR_INVALID, "null shard");
    const Deadline dl(timeout_ms);
    const uint64_t nl = local->num_states, k = local->alphabet_size;
    DevDfa loc;
    loc.n = (uint32_t)nl;
    loc.k = (uint32_t)k;
    loc.delta = ctx.slot_t<uint32_t>("sd.in_delta", std::max<uint64_t>(nl * k, 1));
    loc.acc = ctx.slot_t<uint8_t>("sd.in_acc", std::max<uint64_t>(nl, 1));
    loc.owns = false;
    std::vector<H2DPiece> pieces;
    for (uint64_t a = 0; a < k; ++a) {
      if (local->delta[a] == nullptr && nl) throw Error(DFM_ERR_INVALID, "null row");
      pieces.push_back({loc.delta + a * nl, local->delta[a], nl * 4});
    }
    pieces.push_back({loc.acc, local->accepting, nl});
    if (nl) h2d_batch(ctx, pieces);
    uint32_t* canon = ctx.slot_t<uint32_t>("sd.canon", std::max<uint64_t>(nl, 1));
    AlgoOut o = run_sort_pr_sharded(ctx, n_total, loc, dl, canon, force_protocol());
    if (o.status == DFM_STATUS_OK && block_out) labels_out(ctx, canon, n_total, nl, gather_all != 0, block_out);
    ctx.sync();
    if (num_blocks_out) *num_blocks_out = o.status == DFM_STATUS_OK ? o.num_blocks : 0;
    fill_stats(o, dl, stats);
  });
}

}  // extern "C"
