// mpk_k_re.cu -- one instantiation of the group walk kernel (complex=false, exact=true).
#include "mpk_kernel.cuh"

namespace lmpk {
const void* mpk_ring_fn_re(bool has_long) {
  return has_long ? reinterpret_cast<const void*>(mpk_ring_kernel<false, true, kRingConsumers, true>)
                  : reinterpret_cast<const void*>(mpk_ring_kernel<false, true, kRingConsumers, false>);
}
const void* mpk_ring_fn_re_uniform(int u) {
  if (u == 3) return reinterpret_cast<const void*>(mpk_ring_kernel<false, true, kRingConsumers, false, 3>);
  return u == 1 ? reinterpret_cast<const void*>(mpk_ring_kernel<false, true, kRingConsumers, false, 1>)
                : reinterpret_cast<const void*>(mpk_ring_kernel<false, true, kRingConsumers, false, 2>);
}
const void* mpk_group_fn_re() { return reinterpret_cast<const void*>(mpk_group_kernel<false, true, kConsumers>); }
}  // namespace lmpk
