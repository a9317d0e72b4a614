// mpk_k_ce.cu -- one instantiation of the group walk kernel (complex=true, exact=true).
#include "mpk_kernel.cuh"

namespace lmpk {
const void* mpk_ring_fn_ce(bool has_long) {
  return has_long ? reinterpret_cast<const void*>(mpk_ring_kernel<true, true, kRingConsumers, true>)
                  : reinterpret_cast<const void*>(mpk_ring_kernel<true, true, kRingConsumers, false>);
}
const void* mpk_ring_fn_ce_uniform(int u) {
  return u == 1 ? reinterpret_cast<const void*>(mpk_ring_kernel<true, true, kRingConsumers, false, 1>)
                : reinterpret_cast<const void*>(mpk_ring_kernel<true, true, kRingConsumers, false, 2>);
}
const void* mpk_group_fn_ce() { return reinterpret_cast<const void*>(mpk_group_kernel<true, true, kConsumers>); }
}  // namespace lmpk
