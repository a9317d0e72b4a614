// mpk_lean_cf.cu -- instantiations of the lean ring walk (complex128 vectors, FMA row sums;
// one translation unit per variant family so they compile in parallel).
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_lean_fn_c_f(bool vd, int np, bool xp) {
#define LMPK_LEAN_FN(V, X) (np == 4 ? reinterpret_cast<const void*>(mpk_lean_kernel<true, false, V, true, 4, X>) \
                                    : reinterpret_cast<const void*>(mpk_lean_kernel<true, false, V, true, 2, X>))
  if (vd && xp) return LMPK_LEAN_FN(true, true);
  return vd ? LMPK_LEAN_FN(true, false) : LMPK_LEAN_FN(false, false);
#undef LMPK_LEAN_FN
}
}  // namespace lmpk
