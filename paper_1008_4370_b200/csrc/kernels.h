// kernels.h -- host-side entry points to the kernel families (one translation unit each, so that
// the library builds in parallel).  Each returns the kernel for the given field degree and variant,
// or nullptr when that variant does not exist.
#pragma once

namespace nbk {
void* pass_kernel_ptr(int m, int big, int direct);  // k_pass.cu: nb_pass_kernel (0 separable, 1 direct, 2 pmf)
void* pass_kernel_soft_ptr(int m, int big, int direct);  // k_pass_soft.cu: its soft-output instantiations
void* persist_plain_ptr(int m, int big);            // k_cluster.cu: lf_cluster_kernel, LLR input
void* persist_pmf_ptr(int m, int big);              // k_cluster_pmf.cu: the symbol-pmf variant
void* persist_f16_ptr(int m, int big);              // k_cluster_f16.cu: half-precision messages (m >= 3)
void* persist_kp_ptr(int m, int kpad);              // k_cluster_kp.cu: compile-time chunk geometry
void* persist_sym_ptr(int m, int big);              // k_cluster_sym.cu: symbol-level outputs
void* persist_soft_ptr(int m, int big, int var);    // k_cluster_soft.cu: soft outputs (0 plain, 1 pmf, 2 f16, 3 sym)
void* persist_soft2_ptr(int m, int big, int var);   // k_cluster_soft2.cu: its pmf / f16 part
void* ls_kernel_ptr(int m);                         // k_other.cu: the conventional Log-SP kernel
void* gen_kernel_ptr(int m, int soft);              // k_other.cu: the general-column-weight kernel (soft: fp64 decision)
}  // namespace nbk
