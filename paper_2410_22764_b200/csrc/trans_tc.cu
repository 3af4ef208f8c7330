// tcgen05 int8 GEMM squaring for the Cho–Huynh closure.  (engine selection
// lives in usable())
#include "trans_tc.cuh"

namespace dfm {
namespace trans_tc {

bool usable(uint64_t) { return false; }

TransTcState init(Ctx&, const DevDfa&, uint64_t) {
  throw Error(DFM_ERR_INVALID, "tcgen05 closure engine not built");
}

void square_and_propagate(Ctx&, TransTcState&, const unsigned long long*, unsigned long long*) {
  throw Error(DFM_ERR_INVALID, "tcgen05 closure engine not built");
}

}  // namespace trans_tc
}  // namespace dfm
