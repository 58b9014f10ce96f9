// k_cluster_sym.cu -- the cluster-per-frame kernel with symbol-level outputs, see dispatch.cuh
#include "dispatch.cuh"

namespace nbk {
void* persist_sym_ptr(int m, int big) {
  switch (m * 2 + (big ? 1 : 0)) {
    case 2: return cluster_sym_fn<1, 256>();
    case 3: return cluster_sym_fn<1, 512>();
    case 4: return cluster_sym_fn<2, 256>();
    case 5: return cluster_sym_fn<2, 512>();
    case 6: return cluster_sym_fn<3, 256>();
    case 7: return cluster_sym_fn<3, 512>();
    case 8: return cluster_sym_fn<4, 256>();
    case 9: return cluster_sym_fn<4, 512>();
    case 10: return cluster_sym_fn<5, 256>();
    case 11: return cluster_sym_fn<5, 512>();
    case 12: return cluster_sym_fn<6, 256>();
    case 13: return cluster_sym_fn<6, 512>();
    case 14: return cluster_sym_fn<7, 256>();
    case 15: return cluster_sym_fn<7, 512>();
    case 16: return cluster_sym_fn<8, 256>();
    case 17: return cluster_sym_fn<8, 512>();
  }
  return nullptr;
}

}  // namespace nbk
