// Transports of the sharded sortPR (comm.cuh): NCCL through dlopen, and an
// in-process threads transport for the single-GPU test boxes.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "comm.cuh"
#include "dfm_internal.cuh"

namespace dfm {
namespace {

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    // RTLD_NOLOAD first: reuse an NCCL the process already has (torch's)
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      if (!f && err.empty()) err = std::string("libnccl lacks ") + name;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.AllGather, "ncclAllGather");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
  });
  if (!err.empty()) throw Error(DFM_ERR_CUDA, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(DFM_ERR_CUDA, std::string(what) + " failed: " + nccl().GetErrorString(r));
}

class NcclComm final : public Comm {
 public:
  NcclComm(int device, int r, int w, const uint8_t id[128]) {
    rank = r;
    world = w;
    DFM_CUDA(cudaSetDevice(device));
    ncclUniqueId uid;
    static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl().CommInitRank(&comm_, w, uid, r), "ncclCommInitRank");
    DFM_CUDA(cudaMalloc(&scratch_, kScratch));
  }
  ~NcclComm() override {
    if (scratch_) cudaFree(scratch_);
    if (comm_) nccl().CommDestroy(comm_);
  }
  const char* kind() const override { return "nccl"; }
  void all_gather(const void* send, void* recv, uint64_t bytes, cudaStream_t s) override {
    nccl_check(nccl().AllGather(send, recv, bytes, ncclUint8, comm_, s), "ncclAllGather");
  }
  void all_to_all(const void* send, const uint64_t* so, const uint64_t* sb, void* recv,
                  const uint64_t* ro, const uint64_t* rb, cudaStream_t s) override {
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int r = 0; r < world; ++r) {
      if (sb[r])
        nccl_check(nccl().Send(static_cast<const char*>(send) + so[r], sb[r], ncclUint8, r, comm_, s),
                   "ncclSend");
      if (rb[r])
        nccl_check(nccl().Recv(static_cast<char*>(recv) + ro[r], rb[r], ncclUint8, r, comm_, s),
                   "ncclRecv");
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  }
  void all_reduce_min_u32(uint32_t* buf, uint64_t count, cudaStream_t s) override {
    nccl_check(nccl().AllReduce(buf, buf, count, ncclUint32, ncclMin, comm_, s), "ncclAllReduce");
  }
  void all_gather_host(const uint64_t* mine, uint64_t* all, int count, cudaStream_t s) override {
    const uint64_t b = 8ull * count;
    if (b * (world + 1) > kScratch) throw Error(DFM_ERR_INVALID, "all_gather_host: too many values");
    char* dev = static_cast<char*>(scratch_);
    DFM_CUDA(cudaMemcpyAsync(dev, mine, b, cudaMemcpyHostToDevice, s));
    all_gather(dev, dev + b, b, s);
    DFM_CUDA(cudaMemcpyAsync(all, dev + b, b * world, cudaMemcpyDeviceToHost, s));
    DFM_CUDA(cudaStreamSynchronize(s));
  }

 private:
  static constexpr uint64_t kScratch = 64ull << 10;  // (world + 1) * count u64 values
  ncclComm_t comm_ = nullptr;
  void* scratch_ = nullptr;
};

// ------------------------------------------------------------------ local threads
struct LocalGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;
  std::vector<const uint64_t*> off, bytes;
  explicit LocalGroup(int w) : world(w), ptr(w), off(w), bytes(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

std::mutex g_groups_mu;
std::map<std::string, std::weak_ptr<LocalGroup>> g_groups;

__global__ void min_into_kernel(uint32_t* __restrict__ acc, const uint32_t* __restrict__ other,
                                uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
    acc[i] = min(acc[i], other[i]);
}

class LocalComm final : public Comm {
 public:
  LocalComm(const std::string& name, int r, int w) {
    rank = r;
    world = w;
    std::lock_guard<std::mutex> lk(g_groups_mu);
    auto& slot = g_groups[name];
    g_ = slot.lock();
    if (!g_) {
      g_ = std::make_shared<LocalGroup>(w);
      slot = g_;
    }
    if (g_->world != w) throw Error(DFM_ERR_INVALID, "local group world size mismatch");
  }
  const char* kind() const override { return "local"; }
  void all_gather(const void* send, void* recv, uint64_t bytes, cudaStream_t s) override {
    DFM_CUDA(cudaStreamSynchronize(s));  // our send buffer is complete
    g_->ptr[rank] = send;
    g_->barrier();
    for (int r = 0; r < world; ++r)
      if (bytes)
        DFM_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + (uint64_t)r * bytes, g_->ptr[r], bytes,
                                 cudaMemcpyDeviceToDevice, s));
    DFM_CUDA(cudaStreamSynchronize(s));
    g_->barrier();  // peers may reuse their send buffers
  }
  void all_to_all(const void* send, const uint64_t* so, const uint64_t* sb, void* recv,
                  const uint64_t* ro, const uint64_t* rb, cudaStream_t s) override {
    DFM_CUDA(cudaStreamSynchronize(s));
    g_->ptr[rank] = send;
    g_->off[rank] = so;
    g_->bytes[rank] = sb;
    g_->barrier();
    for (int p = 0; p < world; ++p) {
      const uint64_t b = g_->bytes[p][rank];
      if (b != rb[p]) throw Error(DFM_ERR_INVALID, "all_to_all: byte counts disagree");
      if (b)
        DFM_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + ro[p],
                                 static_cast<const char*>(g_->ptr[p]) + g_->off[p][rank], b,
                                 cudaMemcpyDeviceToDevice, s));
    }
    DFM_CUDA(cudaStreamSynchronize(s));
    g_->barrier();
  }
  void all_reduce_min_u32(uint32_t* buf, uint64_t count, cudaStream_t s) override {
    uint32_t* tmp = nullptr;
    DFM_CUDA(cudaMallocAsync(&tmp, std::max<uint64_t>(count, 1) * 4, s));
    DFM_CUDA(cudaMemcpyAsync(tmp, buf, count * 4, cudaMemcpyDeviceToDevice, s));
    DFM_CUDA(cudaStreamSynchronize(s));
    g_->ptr[rank] = buf;
    g_->barrier();
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(std::max<uint64_t>(count, 1), 256), 4096);
    for (int p = 0; p < world; ++p)
      if (p != rank && count) {
        min_into_kernel<<<grid, 256, 0, s>>>(tmp, static_cast<const uint32_t*>(g_->ptr[p]), count);
        DFM_LAUNCH_CHECK();
      }
    DFM_CUDA(cudaStreamSynchronize(s));
    g_->barrier();  // every rank has read every buffer
    DFM_CUDA(cudaMemcpyAsync(buf, tmp, count * 4, cudaMemcpyDeviceToDevice, s));
    DFM_CUDA(cudaFreeAsync(tmp, s));
    DFM_CUDA(cudaStreamSynchronize(s));
  }
  void all_gather_host(const uint64_t* mine, uint64_t* all, int count, cudaStream_t) override {
    g_->ptr[rank] = mine;
    g_->barrier();
    for (int r = 0; r < world; ++r)
      std::memcpy(all + (uint64_t)r * count, g_->ptr[r], 8ull * count);
    g_->barrier();
  }

 private:
  std::shared_ptr<LocalGroup> g_;
};

}  // namespace

Comm* make_nccl_comm(int device, int rank, int world, const uint8_t id[128]) {
  return new NcclComm(device, rank, world, id);
}

void nccl_unique_id(uint8_t id[128]) {
  ncclUniqueId uid;
  nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(id, &uid, 128);
}

Comm* make_local_comm(const std::string& group, int rank, int world) {
  return new LocalComm(group, rank, world);
}

}  // namespace dfm
