// mpk_lean_ce.cu -- instantiations of the lean ring walk (complex128 vectors, exact row sums;
// one translation unit per variant family so they compile in parallel).
#include "lean_kernel.cuh"

namespace lmpk {
const void* mpk_lean_fn_c_e(bool vd, int np) {
#define LMPK_LEAN_FN(V) (np == 4 ? reinterpret_cast<const void*>(mpk_lean_kernel<true, true, V, true, 4>) \
                                 : reinterpret_cast<const void*>(mpk_lean_kernel<true, true, V, true, 2>))
  return vd ? LMPK_LEAN_FN(true) : LMPK_LEAN_FN(false);
#undef LMPK_LEAN_FN
}
}  // namespace lmpk
