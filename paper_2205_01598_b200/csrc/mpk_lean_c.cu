// mpk_lean_c.cu -- instantiations of the lean ring walk, complex128 vectors
// (real matrix; the general epilogue covers plain, Chebyshev and accumulation).
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_lean_fn_c(bool exact, bool vd) {
#define LMPK_LEAN_FN(E, V) reinterpret_cast<const void*>(mpk_lean_kernel<true, E, V, true>)
  if (exact) return vd ? LMPK_LEAN_FN(true, true) : LMPK_LEAN_FN(true, false);
  return vd ? LMPK_LEAN_FN(false, true) : LMPK_LEAN_FN(false, false);
#undef LMPK_LEAN_FN
}
}  // namespace lmpk
