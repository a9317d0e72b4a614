// mpk_lean_ce.cu -- instantiations of the lean ring walk (complex128 vectors, exact row sums;
// one translation unit per variant family so they compile in parallel).
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_lean_fn_c_e(bool vd, int np, bool xp) {
#define LMPK_LEAN_FN(V, X) (np == 4 ? reinterpret_cast<const void*>(mpk_lean_kernel<true, true, V, true, 4, X>) \
                                    : reinterpret_cast<const void*>(mpk_lean_kernel<true, true, V, true, 2, X>))
  if (vd && xp) return LMPK_LEAN_FN(true, true);
  return vd ? LMPK_LEAN_FN(true, false) : LMPK_LEAN_FN(false, false);
#undef LMPK_LEAN_FN
}
}  // namespace lmpk
