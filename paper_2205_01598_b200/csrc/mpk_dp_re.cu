// mpk_dp_re.cu -- instantiations of the lean ring walk over DP (diagonal-private
// dictionary) blocks: real vectors, exact row sums.
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_dp_fn_r_e(bool gen, int np) {
#define LMPK_DP_FN(G) (np == 4 ? reinterpret_cast<const void*>(mpk_lean_kernel<false, true, true, G, 4, false, true>) \
                               : reinterpret_cast<const void*>(mpk_lean_kernel<false, true, true, G, 2, false, true>))
  return gen ? LMPK_DP_FN(true) : LMPK_DP_FN(false);
#undef LMPK_DP_FN
}
}  // namespace lmpk
