// tcgen05 int8 squaring engine for the Cho–Huynh closure (see trans_tc.cu).
#pragma once

#include <cstdint>

#include "dfm_internal.cuh"

namespace dfm {

struct TransTcState {
  uint64_t V = 0;     // pair nodes
  uint64_t Vp = 0;    // padded to the GEMM tile
  int8_t* reach = nullptr;   // Vp x Vp 0/1 bytes, row-major (A K-major, B MN-major)
  int8_t* next = nullptr;
  // 128x128-tile occupancy of reach / next (bit mt*T + kt, T = Vp/128): the squaring
  // skips the K blocks whose A or B tile is all zero
  uint32_t* nz = nullptr;
  uint32_t* nz_next = nullptr;
};

namespace trans_tc {
bool usable(uint64_t V, int engine);  // engine: DFM_TRANS_AUTO / _BIT / _TENSOR
TransTcState init(Ctx& ctx, const DevDfa& d, uint64_t V);
// one pass: next = reach | (reach*reach > 0); apart_next |= rows reaching apart;
// then swaps reach<->next inside the state
void square_and_propagate(Ctx& ctx, TransTcState& st, const unsigned long long* apart,
                          unsigned long long* apart_next);
}  // namespace trans_tc

}  // namespace dfm
