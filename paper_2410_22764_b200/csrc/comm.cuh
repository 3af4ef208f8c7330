// Collectives of the state-sharded sortPR, owned by
// a dfm_ctx created with dfm_ctx_create_sharded[_local].  Two transports behind one
// interface:
//   * NCCL (the product, one process per GPU over NVLink/NVSwitch): libnccl is
//     dlopen'ed on first use, so the process's NCCL (torch's, when torch is
//     loaded first) is the one used and libdfm.so has no link-time NCCL dependency;
//   * local (tests): `world` ranks as host threads of ONE process sharing one
//     device — contexts exchange device buffers with D2D copies between a pair of
//     host barriers.  It runs the whole C++ protocol at world 2/3/4 on the single
//     GPU the test boxes have (NCCL refuses two ranks on one device).
// Every call is collective: all ranks call it in the same order.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>

namespace dfm {

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // recv = the ranks' `bytes`-byte send buffers, rank-major (world * bytes)
  virtual void all_gather(const void* send, void* recv, uint64_t bytes, cudaStream_t s) = 0;
  // send[send_off[r] .. +send_bytes[r]) goes to rank r, where it lands at
  // recv[recv_off[src] ..]; byte counts must match pairwise
  virtual void all_to_all(const void* send, const uint64_t* send_off, const uint64_t* send_bytes,
                          void* recv, const uint64_t* recv_off, const uint64_t* recv_bytes,
                          cudaStream_t s) = 0;
  // elementwise minimum over the ranks of a device u32 array, in place
  virtual void all_reduce_min_u32(uint32_t* buf, uint64_t count, cudaStream_t s) = 0;
  // host vectors of `count` u64 from every rank -> all[rank * count + i] (synchronous)
  virtual void all_gather_host(const uint64_t* mine, uint64_t* all, int count, cudaStream_t s) = 0;
  virtual const char* kind() const = 0;
};

// NCCL communicator of `world` ranks from a 128-byte ncclUniqueId (rank 0's
// nccl_unique_id(), distributed by the host)
Comm* make_nccl_comm(int device, int rank, int world, const uint8_t id[128]);
void nccl_unique_id(uint8_t id[128]);
// threads-of-one-process transport, ranks meet in the named group
Comm* make_local_comm(const std::string& group, int rank, int world);

}  // namespace dfm
