// k_cluster_soft2.cu -- soft-output instantiations of the cluster kernel (fp64 decision), symbol-pmf
// input and half-precision messages; see dispatch.cuh
#include "dispatch.cuh"

namespace nbk {
void* persist_soft2_ptr(int m, int big, int var) {
  switch (var) {
    case 1: return persist_soft_ptr_t<1>(m, big);
    case 2: return persist_soft_ptr_t<2>(m, big);
  }
  return nullptr;
}
}  // namespace nbk
