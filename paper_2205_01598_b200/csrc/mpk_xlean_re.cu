// mpk_xlean_re.cu -- instantiations of the staged lean walk (real vectors, exact row sums).
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_xlean_fn_r_e(bool vd, bool gen, bool xp, int ctas) {
#define LMPK_XLEAN_FN(V, G, X)                                                                               \
  (ctas == 2 ? reinterpret_cast<const void*>(mpk_xlean_kernel<false, true, V, G, X, kXleanConsumers2, 2>) \
             : reinterpret_cast<const void*>(mpk_xlean_kernel<false, true, V, G, X>))
  if (vd && xp) return gen ? LMPK_XLEAN_FN(true, true, true) : LMPK_XLEAN_FN(true, false, true);
  if (vd) return gen ? LMPK_XLEAN_FN(true, true, false) : LMPK_XLEAN_FN(true, false, false);
  return gen ? LMPK_XLEAN_FN(false, true, false) : LMPK_XLEAN_FN(false, false, false);
#undef LMPK_XLEAN_FN
}
}  // namespace lmpk
