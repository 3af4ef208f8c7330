// Bulk input path: a binary DFA file beside the reference's
// text format (ingest.hpp:286-369, single-threaded parse; a 1e9 x 4 text file is
// ~40 GB), loaded straight into HBM through double-buffered pinned staging so
// the file reads overlap the H2D copies.
//
// Layout (little endian):  "DFMBIN01" | u32 n | u32 k | u32 initial | u32 0 |
//                          acc[n] u8 | zero pad to 4 bytes | delta[k][n] u32
// i.e. the reference's Dfa (core.hpp:24-33) in its own SoA row order.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "dfm_internal.cuh"

namespace dfm {
namespace {

constexpr char kMagic[8] = {'D', 'F', 'M', 'B', 'I', 'N', '0', '1'};
constexpr size_t kHeader = 24;
constexpr size_t kChunk = 64ull << 20;  // pinned staging buffer size

uint64_t acc_bytes_padded(uint64_t n) { return (n + 3) & ~3ull; }

// pread the whole range with a few threads (page-cache bound files read faster)
void pread_all(int fd, void* dst, size_t bytes, uint64_t off) {
  const unsigned T = std::max(1u, std::min(8u, (unsigned)(bytes >> 24)));
  std::vector<std::thread> th;
  std::vector<int> bad(T, 0);
  auto work = [&](unsigned t) {
    const size_t lo = bytes * t / T, hi = bytes * (t + 1) / T;
    size_t done = lo;
    while (done < hi) {
      const ssize_t r = pread(fd, static_cast<char*>(dst) + done, hi - done, (off_t)(off + done));
      if (r <= 0) {
        bad[t] = 1;
        return;
      }
      done += (size_t)r;
    }
  };
  for (unsigned t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  for (int b : bad)
    if (b) throw Error(DFM_ERR_INVALID, "short read from DFA file");
}

void pwrite_all(int fd, const void* src, size_t bytes, uint64_t off) {
  size_t done = 0;
  while (done < bytes) {
    const ssize_t r =
        pwrite(fd, static_cast<const char*>(src) + done, bytes - done, (off_t)(off + done));
    if (r <= 0) throw Error(DFM_ERR_INVALID, "write to DFA file failed");
    done += (size_t)r;
  }
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

}  // namespace

void write_dfa_bin(const char* path, uint32_t n, uint32_t k, uint32_t initial,
                   const uint32_t* const* rows, const uint8_t* acc) {
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (f.fd < 0) throw Error(DFM_ERR_INVALID, std::string("cannot open ") + path);
  char hdr[kHeader] = {};
  std::memcpy(hdr, kMagic, 8);
  const uint32_t h[4] = {n, k, initial, 0};
  std::memcpy(hdr + 8, h, 16);
  pwrite_all(f.fd, hdr, kHeader, 0);
  pwrite_all(f.fd, acc, n, kHeader);
  const uint32_t zero = 0;
  if (acc_bytes_padded(n) > n) pwrite_all(f.fd, &zero, acc_bytes_padded(n) - n, kHeader + n);
  uint64_t off = kHeader + acc_bytes_padded(n);
  for (uint32_t a = 0; a < k; ++a, off += 4ull * n) pwrite_all(f.fd, rows[a], 4ull * n, off);
}

DevDfa load_dfa_bin(Ctx& ctx, const char* path) {
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) throw Error(DFM_ERR_INVALID, std::string("cannot open ") + path);
  char hdr[kHeader];
  pread_all(f.fd, hdr, kHeader, 0);
  if (std::memcmp(hdr, kMagic, 8) != 0) throw Error(DFM_ERR_INVALID, "not a DFMBIN01 file");
  uint32_t h[4];
  std::memcpy(h, hdr + 8, 16);
  const uint64_t n = h[0], k = h[1];
  if (n < 1) throw Error(DFM_ERR_INVALID, "automaton needs at least one state");
  if (h[2] >= n) throw Error(DFM_ERR_INVALID, "initial state out of range");
  struct stat st;
  fstat(f.fd, &st);
  const uint64_t need = kHeader + acc_bytes_padded(n) + 4ull * n * k;
  if ((uint64_t)st.st_size < need) throw Error(DFM_ERR_INVALID, "DFA file is truncated");
  DevDfa dd;
  dd.n = (uint32_t)n;
  dd.k = (uint32_t)k;
  dd.initial = h[2];
  dd.owns = true;
  DFM_CUDA(cudaMalloc(&dd.delta, std::max<uint64_t>(n * k, 1) * 4));
  DFM_CUDA(cudaMalloc(&dd.acc, n));
  try {
    // two pinned staging buffers: read chunk i+1 while chunk i is in flight
    char* stage = static_cast<char*>(ctx.host_pinned(2 * kChunk));
    struct Events {  // destroyed on every exit, including a throw mid-staging
      cudaEvent_t e[2] = {nullptr, nullptr};
      ~Events() {
        for (cudaEvent_t x : e)
          if (x) cudaEventDestroy(x);
      }
    } ev;
    cudaEvent_t* done = ev.e;
    DFM_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    DFM_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    // the file payload after the header maps onto [acc (padded) | delta] in device order
    const uint64_t acc_pad = acc_bytes_padded(n);
    const uint64_t total = acc_pad + 4ull * n * k;
    int buf = 0;
    bool used[2] = {false, false};
    for (uint64_t off = 0; off < total; off += kChunk, buf ^= 1) {
      const uint64_t len = std::min<uint64_t>(kChunk, total - off);
      if (used[buf]) DFM_CUDA(cudaEventSynchronize(done[buf]));
      char* s = stage + (uint64_t)buf * kChunk;
      pread_all(f.fd, s, len, kHeader + off);
      // split the chunk across the acc region and the delta region
      uint64_t o = off, p = 0;
      while (p < len) {
        if (o < acc_pad) {
          const uint64_t take = std::min<uint64_t>(len - p, acc_pad - o);
          const uint64_t real = o < n ? std::min<uint64_t>(take, n - o) : 0;
          if (real)
            DFM_CUDA(cudaMemcpyAsync(dd.acc + o, s + p, real, cudaMemcpyHostToDevice, ctx.stream));
          o += take;
          p += take;
        } else {
          const uint64_t take = len - p;
          DFM_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(dd.delta) + (o - acc_pad), s + p, take,
                                   cudaMemcpyHostToDevice, ctx.stream));
          o += take;
          p += take;
        }
      }
      DFM_CUDA(cudaEventRecord(done[buf], ctx.stream));
      used[buf] = true;
    }
    ctx.sync();
  } catch (...) {
    cudaFree(dd.delta);
    cudaFree(dd.acc);
    throw;
  }
  return dd;
}

void save_dfa_bin(Ctx& ctx, const DevDfa& dd, const char* path) {
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (f.fd < 0) throw Error(DFM_ERR_INVALID, std::string("cannot open ") + path);
  const uint64_t n = dd.n, k = dd.k;
  char hdr[kHeader] = {};
  std::memcpy(hdr, kMagic, 8);
  const uint32_t h[4] = {dd.n, dd.k, dd.initial, 0};
  std::memcpy(hdr + 8, h, 16);
  pwrite_all(f.fd, hdr, kHeader, 0);
  char* stage = static_cast<char*>(ctx.host_pinned(2 * kChunk));
  // acc (padded), then the rows, chunk by chunk through the pinned buffer
  const uint64_t acc_pad = acc_bytes_padded(n);
  std::vector<char> pad(acc_pad - n, 0);
  uint64_t file_off = kHeader;
  for (uint64_t o = 0; o < n; o += kChunk) {
    const uint64_t len = std::min<uint64_t>(kChunk, n - o);
    DFM_CUDA(cudaMemcpyAsync(stage, dd.acc + o, len, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    pwrite_all(f.fd, stage, len, file_off);
    file_off += len;
  }
  if (!pad.empty()) pwrite_all(f.fd, pad.data(), pad.size(), file_off);
  file_off = kHeader + acc_pad;
  const uint64_t dbytes = 4ull * n * k;
  for (uint64_t o = 0; o < dbytes; o += kChunk) {
    const uint64_t len = std::min<uint64_t>(kChunk, dbytes - o);
    DFM_CUDA(cudaMemcpyAsync(stage, reinterpret_cast<const char*>(dd.delta) + o, len,
                             cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    pwrite_all(f.fd, stage, len, file_off + o);
  }
}

}  // namespace dfm
