// k_cluster.cu -- the cluster-per-frame kernel, LLR input (the hot path), see dispatch.cuh
#include "dispatch.cuh"

namespace nbk {
void* persist_plain_ptr(int m, int big) { return persist_kernel_ptr_t<false, false>(m, big); }
}  // namespace nbk
