// k_cluster_f16.cu -- the cluster-per-frame kernel with half-precision messages, see dispatch.cuh
#include "dispatch.cuh"

namespace nbk {
void* persist_f16_ptr(int m, int big) { return persist_kernel_ptr_t<false, true>(m, big); }
}  // namespace nbk
