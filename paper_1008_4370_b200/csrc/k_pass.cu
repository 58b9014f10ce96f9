// k_pass.cu -- the slot-pass kernel family (nb_pass_kernel), see dispatch.cuh
#include "dispatch.cuh"

namespace nbk {
// direct = 1: the paper's q^2-term convolution; 0: separable butterflies;
// 2: the direct convolution with the channel spectrum of a general pmf (nbldpc_decode_pmf)
void* pass_kernel_ptr(int m, int big, int direct) {
  if (direct == 2) return pass_kernel_ptr_t<true, true>(m, big);
  return direct ? pass_kernel_ptr_t<true, false>(m, big) : pass_kernel_ptr_t<false, false>(m, big);
}
}  // namespace nbk
