// k_other.cu -- the Log-SP comparison kernel and the general-column-weight kernel families
#include "kernels.h"
#include "lf_general.cuh"
#include "logsp.cuh"

namespace nbk {
template <int MB>
void* ls_fn() { return reinterpret_cast<void*>(&nb::ls_frame_kernel<MB>); }
void* ls_kernel_ptr(int m) {
  switch (m) {
    case 1: return ls_fn<1>();
    case 2: return ls_fn<2>();
    case 3: return ls_fn<3>();
    case 4: return ls_fn<4>();
    case 5: return ls_fn<5>();
    case 6: return ls_fn<6>();
    case 7: return ls_fn<7>();
    case 8: return ls_fn<8>();
  }
  return nullptr;
}

template <int MB>
void* gen_fn(int soft) {
  return soft ? reinterpret_cast<void*>(&nb::lfg_frame_kernel<MB, true>)
              : reinterpret_cast<void*>(&nb::lfg_frame_kernel<MB, false>);
}
void* gen_kernel_ptr(int m, int soft) {
  switch (m) {
    case 1: return gen_fn<1>(soft);
    case 2: return gen_fn<2>(soft);
    case 3: return gen_fn<3>(soft);
    case 4: return gen_fn<4>(soft);
    case 5: return gen_fn<5>(soft);
    case 6: return gen_fn<6>(soft);
    case 7: return gen_fn<7>(soft);
    case 8: return gen_fn<8>(soft);
  }
  return nullptr;
}

}  // namespace nbk
