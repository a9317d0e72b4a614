// mpk_dp_cf.cu -- instantiations of the lean ring walk over DP (diagonal-private
// dictionary) blocks: complex128 vectors, FMA row sums.
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_dp_fn_c_f(int np) {
  return np == 4 ? reinterpret_cast<const void*>(mpk_lean_kernel<true, false, true, true, 4, false, true>)
                 : reinterpret_cast<const void*>(mpk_lean_kernel<true, false, true, true, 2, false, true>);
}
}  // namespace lmpk
