// Context, scratch arena and profiling for libdfm.so.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "comm.cuh"
#include "dfm_internal.cuh"

#include <atomic>

namespace dfm {

static std::atomic<uint64_t> g_launches{0};
uint64_t note_launch() { return g_launches.fetch_add(1, std::memory_order_relaxed) + 1; }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

int per_device_memo(const void* key, int device, int (*f)(const void* key)) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> memo;
  std::lock_guard<std::mutex> lk(mu);
  const auto it = memo.find({key, device});
  if (it != memo.end()) return it->second;
  const int v = f(key);
  memo[{key, device}] = v;
  return v;
}

Ctx::Ctx(int dev) : device(dev) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    throw Error(DFM_ERR_NO_DEVICE, "no CUDA device visible: libdfm has no CPU fallback");
  if (dev < 0 || dev >= count) throw Error(DFM_ERR_INVALID, "device index out of range");
  DFM_CUDA(cudaSetDevice(dev));
  cudaDeviceProp prop{};
  DFM_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10 || prop.minor != 0)
    throw Error(DFM_ERR_NO_DEVICE, std::string("libdfm is built for sm_100a; device is sm_") +
                                       std::to_string(prop.major) + std::to_string(prop.minor));
  num_sms = prop.multiProcessorCount;
  DFM_CUDA(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
  stream = own_stream;
  // keep freed stream-ordered allocations cached in the pool across calls
  cudaMemPool_t pool;
  DFM_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t threshold = UINT64_MAX;
  DFM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  DFM_CUDA(cudaMalloc(&d_scalars, 64 * sizeof(uint64_t)));
  DFM_CUDA(cudaMallocHost(&h_scalars, 64 * sizeof(uint64_t)));
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  delete comm;
  for (auto& kv : slots)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  for (auto& p : pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : free_events) cudaEventDestroy(e);
  if (pinned) cudaFreeHost(pinned);
  if (d_scalars) cudaFree(d_scalars);
  if (h_scalars) cudaFreeHost(h_scalars);
  if (copy_stream) {
    cudaStreamSynchronize(copy_stream);
    cudaStreamDestroy(copy_stream);
  }
  for (auto e : chunk_events) cudaEventDestroy(e);
  if (own_stream) cudaStreamDestroy(own_stream);
}

cudaStream_t Ctx::copy() {
  if (!copy_stream) DFM_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
  return copy_stream;
}

const cudaEvent_t* Ctx::chunk_event_pool(uint32_t count) {
  while (chunk_events.size() < count) {
    cudaEvent_t e;
    DFM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    chunk_events.push_back(e);
  }
  return chunk_events.data();
}

void* Ctx::slot(const std::string& name, size_t bytes) {
  if (bytes == 0) bytes = 16;
  Buf& b = slots[name];
  if (b.bytes >= bytes) return b.ptr;
  if (b.ptr) {
    DFM_CUDA(cudaFreeAsync(b.ptr, stream));
    held_bytes -= b.bytes;
    b.ptr = nullptr;
    b.bytes = 0;
  }
  // round up so slowly growing requests do not reallocate every call
  const size_t want = std::max(bytes, (size_t)256) + bytes / 8;
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, want, stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    // retry exactly-sized after draining the pool
    cudaStreamSynchronize(stream);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, device);
    cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(&p, bytes, stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(DFM_ERR_NO_MEMORY, "device allocation of " + std::to_string(bytes) +
                                         " bytes failed for slot '" + name + "'");
    }
    b.bytes = bytes;
  } else {
    b.bytes = want;
  }
  b.ptr = p;
  held_bytes += b.bytes;
  return p;
}

void Ctx::release_slot(const std::string& name) {
  auto it = slots.find(name);
  if (it == slots.end()) return;
  if (it->second.ptr) {
    DFM_CUDA(cudaFreeAsync(it->second.ptr, stream));
    held_bytes -= it->second.bytes;
  }
  slots.erase(it);
}

void* Ctx::host_pinned(size_t bytes) {
  if (pinned_bytes >= bytes) return pinned;
  if (pinned) {
    sync();
    DFM_CUDA(cudaFreeHost(pinned));
    pinned = nullptr;
    pinned_bytes = 0;
  }
  DFM_CUDA(cudaMallocHost(&pinned, bytes));
  pinned_bytes = bytes;
  return pinned;
}

cudaEvent_t Ctx::take_event() {
  if (!free_events.empty()) {
    cudaEvent_t e = free_events.back();
    free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  DFM_CUDA(cudaEventCreate(&e));
  return e;
}

void Ctx::harvest() {
  if (pending.empty()) return;
  sync();
  for (auto& p : pending) {
    float ms = 0.f;
    DFM_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    Acc& a = prof[p.name];
    if (a.launches == 0) {
      if (!prof_names.empty()) prof_names += ",";
      prof_names += p.name;
    }
    a.launches += 1;
    a.ms += ms;
    a.bytes += p.bytes;
    free_events.push_back(p.a);
    free_events.push_back(p.b);
  }
  pending.clear();
}

ProfScope::ProfScope(Ctx& c, const char* n, uint64_t algo_bytes)
    : ctx(c), name(n), bytes(algo_bytes) {
  if (!ctx.profiling) return;
  ev0 = ctx.take_event();
  ev1 = ctx.take_event();
  DFM_CUDA(cudaEventRecord(ev0, ctx.stream));
}

void ProfScope::stop() {
  if (!ctx.profiling || ev0 == nullptr || stopped) return;
  cudaEventRecord(ev1, ctx.stream);
  stopped = true;
}

ProfScope::~ProfScope() {
  if (!ctx.profiling || ev0 == nullptr) return;
  if (!stopped) cudaEventRecord(ev1, ctx.stream);
  ctx.pending.push_back({name, ev0, ev1, bytes});
  if (ctx.pending.size() > 4096) {
    try {
      ctx.harvest();
    } catch (...) {
    }
  }
}

}  // namespace dfm
