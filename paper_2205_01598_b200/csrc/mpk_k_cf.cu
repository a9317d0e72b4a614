// mpk_k_cf.cu -- one instantiation of the group walk kernel (complex=true, exact=false).
#include "mpk_kernel.cuh"

namespace lmpk {
const void* mpk_ring_fn_cf(bool has_long) {
  return has_long ? reinterpret_cast<const void*>(mpk_ring_kernel<true, false, kRingConsumers, true>)
                  : reinterpret_cast<const void*>(mpk_ring_kernel<true, false, kRingConsumers, false>);
}
const void* mpk_ring_fn_cf_uniform(int u) {
  return u == 1 ? reinterpret_cast<const void*>(mpk_ring_kernel<true, false, kRingConsumers, false, 1>)
                : reinterpret_cast<const void*>(mpk_ring_kernel<true, false, kRingConsumers, false, 2>);
}
const void* mpk_group_fn_cf() { return reinterpret_cast<const void*>(mpk_group_kernel<true, false, kConsumers>); }
}  // namespace lmpk
