// dispatch.cuh -- kernel-pointer dispatch templates of the C-ABI library (host code).  Each
// k_*.cu translation unit instantiates one family of kernels through these templates, so that nvcc
// compiles the families in parallel (build.py); nbldpc.cu reaches them through kernels.h.
#pragma once
#include "lf_cluster.cuh"
#include "kernels.h"

namespace nbk {

constexpr int kBigBlock = 512;  // block-size variant for k_max * TT > 256 (as in nbldpc.cu)

template <int MB, int MAXB, bool DIRECT, bool PMF, bool SOFT>
void* pass_fn() { return reinterpret_cast<void*>(&nb::nb_pass_kernel<MB, MAXB, DIRECT, PMF, SOFT>); }

template <bool DIRECT, bool PMF, bool SOFT = false>
void* pass_kernel_ptr_t(int m, int big) {
  switch (m * 2 + (big ? 1 : 0)) {
    case 2: return pass_fn<1, 256, DIRECT, PMF, SOFT>();
    case 3: return pass_fn<1, kBigBlock, DIRECT, PMF, SOFT>();
    case 4: return pass_fn<2, 256, DIRECT, PMF, SOFT>();
    case 5: return pass_fn<2, kBigBlock, DIRECT, PMF, SOFT>();
    case 6: return pass_fn<3, 256, DIRECT, PMF, SOFT>();
    case 7: return pass_fn<3, kBigBlock, DIRECT, PMF, SOFT>();
    case 8: return pass_fn<4, 256, DIRECT, PMF, SOFT>();
    case 9: return pass_fn<4, kBigBlock, DIRECT, PMF, SOFT>();
    case 10: return pass_fn<5, 256, DIRECT, PMF, SOFT>();
    case 11: return pass_fn<5, kBigBlock, DIRECT, PMF, SOFT>();
    case 12: return pass_fn<6, 256, DIRECT, PMF, SOFT>();
    case 13: return pass_fn<6, kBigBlock, DIRECT, PMF, SOFT>();
    case 14: return pass_fn<7, 256, DIRECT, PMF, SOFT>();
    case 15: return pass_fn<7, kBigBlock, DIRECT, PMF, SOFT>();
    case 16: return pass_fn<8, 256, DIRECT, PMF, SOFT>();
    case 17: return pass_fn<8, kBigBlock, DIRECT, PMF, SOFT>();
  }
  return nullptr;
}

template <int MB, int NTHR, bool PMF, bool F16>
void* cluster_fn() {
  if constexpr (F16 && (PMF || MB < 3)) {  // half messages: LLR input, q >= 8 (16-byte row units)
    return nullptr;
  } else {
    return reinterpret_cast<void*>(&nb::lf_cluster_kernel<MB, NTHR, PMF, F16>);
  }
}
template <bool PMF, bool F16>
void* persist_kernel_ptr_t(int m, int big) {
  switch (m * 2 + (big ? 1 : 0)) {
    case 2: return cluster_fn<1, 256, PMF, F16>();
    case 3: return cluster_fn<1, 512, PMF, F16>();
    case 4: return cluster_fn<2, 256, PMF, F16>();
    case 5: return cluster_fn<2, 512, PMF, F16>();
    case 6: return cluster_fn<3, 256, PMF, F16>();
    case 7: return cluster_fn<3, 512, PMF, F16>();
    case 8: return cluster_fn<4, 256, PMF, F16>();
    case 9: return cluster_fn<4, 512, PMF, F16>();
    case 10: return cluster_fn<5, 256, PMF, F16>();
    case 11: return cluster_fn<5, 512, PMF, F16>();
    case 12: return cluster_fn<6, 256, PMF, F16>();
    case 13: return cluster_fn<6, 512, PMF, F16>();
    case 14: return cluster_fn<7, 256, PMF, F16>();
    case 15: return cluster_fn<7, 512, PMF, F16>();
    case 16: return cluster_fn<8, 256, PMF, F16>();
    case 17: return cluster_fn<8, 512, PMF, F16>();
  }
  return nullptr;
}

template <int MB, int KP>
void* cluster_kp_fn() {
  constexpr int TT = MB <= 4 ? 1 : (1 << MB) / 16;
  if constexpr (KP * TT > 512) {
    return nullptr;
  } else {
    return reinterpret_cast<void*>(&nb::lf_cluster_kernel<MB, (KP * TT > 256 ? 512 : 256), false, false, KP>);
  }
}
template <int MB>
void* cluster_kp_m(int kpad) {
  switch (kpad) {
    case 4: return cluster_kp_fn<MB, 4>();
    case 8: return cluster_kp_fn<MB, 8>();
    case 16: return cluster_kp_fn<MB, 16>();
    case 32: return cluster_kp_fn<MB, 32>();
  }
  return nullptr;
}

template <int MB, int NTHR>
void* cluster_sym_fn() { return reinterpret_cast<void*>(&nb::lf_cluster_kernel<MB, NTHR, false, false, 0, true>); }

// soft-output instantiations (SOFT = true): variant 0 plain LLR, 1 symbol pmf, 2 half messages, 3 symbol outputs
template <int MB, int NTHR, int VAR>
void* cluster_soft_fn() {
  if constexpr (VAR == 2 && MB < 3) {
    return nullptr;
  } else {
    return reinterpret_cast<void*>(&nb::lf_cluster_kernel<MB, NTHR, VAR == 1, VAR == 2, 0, VAR == 3, true>);
  }
}
template <int VAR>
void* persist_soft_ptr_t(int m, int big) {
  switch (m * 2 + (big ? 1 : 0)) {
    case 2: return cluster_soft_fn<1, 256, VAR>();
    case 3: return cluster_soft_fn<1, 512, VAR>();
    case 4: return cluster_soft_fn<2, 256, VAR>();
    case 5: return cluster_soft_fn<2, 512, VAR>();
    case 6: return cluster_soft_fn<3, 256, VAR>();
    case 7: return cluster_soft_fn<3, 512, VAR>();
    case 8: return cluster_soft_fn<4, 256, VAR>();
    case 9: return cluster_soft_fn<4, 512, VAR>();
    case 10: return cluster_soft_fn<5, 256, VAR>();
    case 11: return cluster_soft_fn<5, 512, VAR>();
    case 12: return cluster_soft_fn<6, 256, VAR>();
    case 13: return cluster_soft_fn<6, 512, VAR>();
    case 14: return cluster_soft_fn<7, 256, VAR>();
    case 15: return cluster_soft_fn<7, 512, VAR>();
    case 16: return cluster_soft_fn<8, 256, VAR>();
    case 17: return cluster_soft_fn<8, 512, VAR>();
  }
  return nullptr;
}

}  // namespace nbk
