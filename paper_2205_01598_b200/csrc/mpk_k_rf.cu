// mpk_k_rf.cu -- one instantiation of the group walk kernel (complex=false, exact=false).
#include "mpk_kernel.cuh"

namespace lmpk {
const void* mpk_ring_fn_rf(bool has_long) {
  return has_long ? reinterpret_cast<const void*>(mpk_ring_kernel<false, false, kRingConsumers, true>)
                  : reinterpret_cast<const void*>(mpk_ring_kernel<false, false, kRingConsumers, false>);
}
const void* mpk_ring_fn_rf_uniform(int u) {
  if (u == 3) return reinterpret_cast<const void*>(mpk_ring_kernel<false, false, kRingConsumers, false, 3>);
  return u == 1 ? reinterpret_cast<const void*>(mpk_ring_kernel<false, false, kRingConsumers, false, 1>)
                : reinterpret_cast<const void*>(mpk_ring_kernel<false, false, kRingConsumers, false, 2>);
}
const void* mpk_group_fn_rf() { return reinterpret_cast<const void*>(mpk_group_kernel<false, false, kConsumers>); }
}  // namespace lmpk
