// Device primitives of the state-sharded sortPR.
// One process per GPU; the collectives (all-gather of block ids, the key
// exchange, count all-gathers) are issued by the host driver
// (paper_2410_22764_b200/sharded.py) through torch.distributed/NCCL.  Here:
//   shard_signature : per owned state, the full signature row (block[q], block[δa(q)])
//                     read from the all-gathered block vector, its 64-bit hash and
//                     the destination rank that groups that key
//   shard_group     : exact grouping of the (key, signature) pairs a rank received:
//                     dense local group ids; equal-hash members are verified
//                     against the group's first member (collision flag otherwise)
//   sort_pairs      : the onesweep radix sort (routing by destination rank)
//   random slice    : bit-exact random_dfa rows for an owned state range
#include <algorithm>
#include <cstring>

#include "prims.cuh"

namespace dfm {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) shard_sig_kernel(
    const uint32_t* __restrict__ delta, uint64_t n_local, uint32_t k,
    const uint32_t* __restrict__ block_full, uint64_t lo, uint64_t seed, uint32_t ranks,
    unsigned long long* __restrict__ keys, uint32_t* __restrict__ sig,
    uint32_t* __restrict__ dest) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_local; i += stride) {
    const uint32_t b = block_full[lo + i];
    uint32_t* row = sig + i * (uint64_t)(k + 1);
    row[0] = b;
    unsigned long long h = mix64(seed * kGolden + b);
    for (uint32_t a = 0; a < k; ++a) {
      const uint32_t s = block_full[delta[(uint64_t)a * n_local + i]];
      row[a + 1] = s;
      h = mix64(h + kGolden + s);
    }
    keys[i] = h | 1ull;  // never 0: 0 marks an empty table slot
    dest[i] = (uint32_t)__umul64hi(mix64(h ^ 0xD1B54A32D192ED03ull), ranks);
  }
}

struct GSlot {
  unsigned long long key;
  uint32_t rep;  // ~(first member) via atomicMax
  uint32_t gid;
};

__global__ void __launch_bounds__(256) group_insert_kernel(const unsigned long long* __restrict__ keys,
                                                           uint64_t count, GSlot* slots,
                                                           uint64_t cap, uint32_t* __restrict__ slot_of) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const unsigned long long key = keys[i];
    uint64_t t = __umul64hi(key, cap);
    while (true) {
      const unsigned long long cur = atomicCAS(&slots[t].key, 0ull, key);
      if (cur == 0ull || cur == key) break;
      if (++t == cap) t = 0;
    }
    slot_of[i] = (uint32_t)t;
    atomicMax(&slots[t].rep, ~(uint32_t)i);
  }
}

struct GroupIn {
  const GSlot* slots;
  const uint32_t* slot_of;
  const uint32_t* sig;
  uint32_t words;
  unsigned long long* collision;
  __device__ uint32_t operator()(uint64_t i) const {
    const uint32_t rep = ~slots[slot_of[i]].rep;
    if (rep == (uint32_t)i) return 1u;
    const uint32_t* a = sig + i * (uint64_t)words;
    const uint32_t* b = sig + (uint64_t)rep * words;
    for (uint32_t x = 0; x < words; ++x)
      if (a[x] != b[x]) {
        atomicOr(collision, 1ull);
        break;
      }
    return 0u;
  }
};
struct GroupOut {
  GSlot* slots;
  const uint32_t* slot_of;
  uint32_t* label;
  __device__ void operator()(uint64_t i, uint32_t excl, uint32_t v) const {
    if (v) {
      slots[slot_of[i]].gid = excl;
      label[i] = excl;
    }
  }
};
__global__ void group_members_kernel(uint64_t count, const GSlot* __restrict__ slots,
                                     const uint32_t* __restrict__ slot_of,
                                     uint32_t* __restrict__ label) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const GSlot& s = slots[slot_of[i]];
    if (~s.rep != (uint32_t)i) label[i] = s.gid;
  }
}

__global__ void random_slice_kernel(uint32_t* __restrict__ delta, uint8_t* __restrict__ acc,
                                    uint64_t n_total, uint32_t k, uint64_t lo, uint64_t count,
                                    uint64_t seed, double p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    for (uint32_t a = 0; a <= k; ++a) {
      // draw j of SplitMix64(seed): row a, state q -> j = a*n + q; acceptance -> k*n + q
      uint64_t z = seed + ((uint64_t)a * n_total + lo + i + 1) * kGolden;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      if (a < k) delta[(uint64_t)a * count + i] = (uint32_t)(z % n_total);
      else acc[i] = ((double)(z >> 11) * 0x1.0p-53) < p ? 1 : 0;
    }
  }
}

unsigned grid_for(const Ctx& ctx, uint64_t items) {
  return (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(items, 1), 256),
                                      (uint64_t)ctx.num_sms * 16);
}

}  // namespace
}  // namespace dfm

using namespace dfm;

namespace {
template <class F>
int guarded_shard(dfm_ctx* c, F&& f) {
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
}  // namespace

extern "C" {

int dfm_shard_signature(dfm_ctx* c, const void* delta_local, uint64_t n_local, uint32_t k,
                        const void* block_full, uint64_t lo, uint64_t seed, uint32_t ranks,
                        void* keys_out, void* sig_out, void* dest_out) {
  return guarded_shard(c, [&](Ctx& ctx) {
    if (ranks == 0) throw Error(DFM_ERR_INVALID, "ranks must be >= 1");
    if (n_local == 0) return;
    ProfScope p(ctx, "sig", n_local * (4ull * k + 4ull * k + 4 + 8 + 4ull * (k + 1) + 4));
    shard_sig_kernel<<<grid_for(ctx, n_local), 256, 0, ctx.stream>>>(
        static_cast<const uint32_t*>(delta_local), n_local, k,
        static_cast<const uint32_t*>(block_full), lo, seed, ranks,
        static_cast<unsigned long long*>(keys_out), static_cast<uint32_t*>(sig_out),
        static_cast<uint32_t*>(dest_out));
    DFM_LAUNCH_CHECK();
  });
}

int dfm_shard_group(dfm_ctx* c, const void* keys, const void* sig, uint32_t words, uint64_t count,
                    void* label_out, uint64_t* groups_out, int* collision_out) {
  return guarded_shard(c, [&](Ctx& ctx) {
    if (count >= (1ull << 32)) throw Error(DFM_ERR_INVALID, "too many items for one rank");
    uint64_t* sc = ctx.d_scalars + 48;  // [0] groups [1] collision
    DFM_CUDA(cudaMemsetAsync(sc, 0, 16, ctx.stream));
    if (count > 0) {
      const uint64_t cap = std::max<uint64_t>(1024, count + count / 2);
      auto* slots = static_cast<GSlot*>(ctx.slot("shard.table", cap * sizeof(GSlot)));
      uint32_t* slot_of = ctx.slot_t<uint32_t>("shard.slotof", count);
      DFM_CUDA(cudaMemsetAsync(slots, 0, cap * sizeof(GSlot), ctx.stream));
      ProfScope p(ctx, "group", count * (8ull + 16 + 4 + 4 + 4 + 4ull * words));
      group_insert_kernel<<<grid_for(ctx, count), 256, 0, ctx.stream>>>(
          static_cast<const unsigned long long*>(keys), count, slots, cap, slot_of);
      DFM_LAUNCH_CHECK();
      prims::lookback_scan(ctx, "sc.shard", count,
                           GroupIn{slots, slot_of, static_cast<const uint32_t*>(sig), words,
                                   reinterpret_cast<unsigned long long*>(sc + 1)},
                           GroupOut{slots, slot_of, static_cast<uint32_t*>(label_out)}, sc);
      group_members_kernel<<<grid_for(ctx, count), 256, 0, ctx.stream>>>(
          count, slots, slot_of, static_cast<uint32_t*>(label_out));
      DFM_LAUNCH_CHECK();
    }
    DFM_CUDA(cudaMemcpyAsync(ctx.h_scalars + 48, sc, 16, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    if (groups_out) *groups_out = ctx.h_scalars[48];
    if (collision_out) *collision_out = ctx.h_scalars[49] != 0;
  });
}

int dfm_sort_pairs(dfm_ctx* c, void* keys, void* values, uint64_t count, uint32_t bits) {
  return guarded_shard(c, [&](Ctx& ctx) {
    if (count == 0) return;
    auto* k2 = ctx.slot_t<uint64_t>("sp2.keys", count);
    auto* v2 = ctx.slot_t<uint32_t>("sp2.vals", count);
    const bool alt = prims::radix_sort_pairs(ctx, static_cast<uint64_t*>(keys),
                                             static_cast<uint32_t*>(values), k2, v2, count,
                                             (int)std::max(1u, bits), false);
    if (alt) {
      DFM_CUDA(cudaMemcpyAsync(keys, k2, count * 8, cudaMemcpyDeviceToDevice, ctx.stream));
      DFM_CUDA(cudaMemcpyAsync(values, v2, count * 4, cudaMemcpyDeviceToDevice, ctx.stream));
    }
    ctx.sync();
  });
}

int dfm_canonicalize_dev(dfm_ctx* c, const void* raw_dev, uint64_t n, void* out_dev,
                         uint32_t* num_blocks_out) {
  return guarded_shard(c, [&](Ctx& ctx) {
    const uint32_t nb = canonicalize_dev(ctx, static_cast<const uint32_t*>(raw_dev), n,
                                         static_cast<uint32_t*>(out_dev));
    if (num_blocks_out) *num_blocks_out = nb;
  });
}

int dfm_random_dfa_slice_dev(dfm_ctx* c, uint64_t n_total, uint32_t k, uint64_t seed,
                             double accept_prob, uint64_t lo, uint64_t count, void* delta_out,
                             void* accepting_out) {
  return guarded_shard(c, [&](Ctx& ctx) {
    if (n_total < 1 || n_total > 0xFFFFFFFFull || lo + count > n_total)
      throw Error(DFM_ERR_INVALID, "bad random_dfa slice");
    if (count == 0) return;
    random_slice_kernel<<<grid_for(ctx, count), 256, 0, ctx.stream>>>(
        static_cast<uint32_t*>(delta_out), static_cast<uint8_t*>(accepting_out), n_total, k, lo,
        count, seed, accept_prob);
    DFM_LAUNCH_CHECK();
    ctx.sync();
  });
}

}  // extern "C"
