// k_cluster_soft.cu -- soft-output instantiations of the cluster kernel (fp64 decision), LLR input
// and symbol outputs; see dispatch.cuh
#include "dispatch.cuh"

namespace nbk {
void* persist_soft_ptr(int m, int big, int var) {
  switch (var) {
    case 0: return persist_soft_ptr_t<0>(m, big);
    case 3: return persist_soft_ptr_t<3>(m, big);
  }
  return persist_soft2_ptr(m, big, var);
}
}  // namespace nbk
