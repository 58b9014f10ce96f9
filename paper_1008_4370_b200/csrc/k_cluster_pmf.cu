// k_cluster_pmf.cu -- the cluster-per-frame kernel, symbol-pmf input, see dispatch.cuh
#include "dispatch.cuh"

namespace nbk {
void* persist_pmf_ptr(int m, int big) { return persist_kernel_ptr_t<true, false>(m, big); }
}  // namespace nbk
