// k_pass_soft.cu -- soft-output instantiations of the slot-pass kernel (fp64 decision), see dispatch.cuh
#include "dispatch.cuh"

namespace nbk {
void* pass_kernel_soft_ptr(int m, int big, int direct) {
  if (direct == 2) return pass_kernel_ptr_t<true, true, true>(m, big);
  return direct ? pass_kernel_ptr_t<true, false, true>(m, big) : pass_kernel_ptr_t<false, false, true>(m, big);
}
}  // namespace nbk
