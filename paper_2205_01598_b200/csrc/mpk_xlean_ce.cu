// mpk_xlean_ce.cu -- instantiations of the staged lean walk (complex128 vectors, exact row sums).
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_xlean_fn_c_e(bool vd, bool xp, int ctas) {
#define LMPK_XLEAN_FN(V, X)                                                                                  \
  (ctas == 2 ? reinterpret_cast<const void*>(mpk_xlean_kernel<true, true, V, true, X, kXleanConsumers2, 2>) \
             : reinterpret_cast<const void*>(mpk_xlean_kernel<true, true, V, true, X>))
  if (vd && xp) return LMPK_XLEAN_FN(true, true);
  return vd ? LMPK_XLEAN_FN(true, false) : LMPK_XLEAN_FN(false, false);
#undef LMPK_XLEAN_FN
}
}  // namespace lmpk
