// mpk_lean_rf.cu -- instantiations of the lean ring walk (real vectors, FMA row sums;
// one translation unit per variant family so they compile in parallel).
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_lean_fn_r_f(bool vd, bool gen, int np) {
#define LMPK_LEAN_FN(V, G) (np == 4 ? reinterpret_cast<const void*>(mpk_lean_kernel<false, false, V, G, 4>) \
                                    : reinterpret_cast<const void*>(mpk_lean_kernel<false, false, V, G, 2>))
  if (vd) return gen ? LMPK_LEAN_FN(true, true) : LMPK_LEAN_FN(true, false);
  return gen ? LMPK_LEAN_FN(false, true) : LMPK_LEAN_FN(false, false);
#undef LMPK_LEAN_FN
}
}  // namespace lmpk
