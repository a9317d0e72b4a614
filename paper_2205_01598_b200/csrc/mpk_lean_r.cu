// mpk_lean_r.cu -- instantiations of the lean ring walk, real vectors.
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_lean_fn_r(bool exact, bool vd, bool gen) {
#define LMPK_LEAN_FN(E, V, G) reinterpret_cast<const void*>(mpk_lean_kernel<false, E, V, G>)
  if (exact) {
    if (vd) return gen ? LMPK_LEAN_FN(true, true, true) : LMPK_LEAN_FN(true, true, false);
    return gen ? LMPK_LEAN_FN(true, false, true) : LMPK_LEAN_FN(true, false, false);
  }
  if (vd) return gen ? LMPK_LEAN_FN(false, true, true) : LMPK_LEAN_FN(false, true, false);
  return gen ? LMPK_LEAN_FN(false, false, true) : LMPK_LEAN_FN(false, false, false);
#undef LMPK_LEAN_FN
}
}  // namespace lmpk
