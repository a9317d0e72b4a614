// mpk_dp_ce.cu -- instantiations of the lean ring walk over DP (diagonal-private
// dictionary) blocks: complex128 vectors, exact row sums.
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_dp_fn_c_e(int np) {
  return np == 4 ? reinterpret_cast<const void*>(mpk_lean_kernel<true, true, true, true, 4, false, true>)
                 : reinterpret_cast<const void*>(mpk_lean_kernel<true, true, true, true, 2, false, true>);
}
}  // namespace lmpk
