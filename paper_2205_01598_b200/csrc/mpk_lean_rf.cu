// mpk_lean_rf.cu -- instantiations of the lean ring walk (real vectors, FMA row sums;
// one translation unit per variant family so they compile in parallel).
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_lean_fn_r_f(bool vd, bool gen, int np, bool xp) {
#define LMPK_LEAN_FN(V, G, X) (np == 4 ? reinterpret_cast<const void*>(mpk_lean_kernel<false, false, V, G, 4, X>) \
                                       : reinterpret_cast<const void*>(mpk_lean_kernel<false, false, V, G, 2, X>))
  if (vd && xp) return gen ? LMPK_LEAN_FN(true, true, true) : LMPK_LEAN_FN(true, false, true);
  if (vd) return gen ? LMPK_LEAN_FN(true, true, false) : LMPK_LEAN_FN(true, false, false);
  return gen ? LMPK_LEAN_FN(false, true, false) : LMPK_LEAN_FN(false, false, false);
#undef LMPK_LEAN_FN
}
}  // namespace lmpk
