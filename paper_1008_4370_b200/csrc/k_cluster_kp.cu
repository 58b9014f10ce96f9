// k_cluster_kp.cu -- the cluster-per-frame kernel with compile-time chunk geometry, see dispatch.cuh
#include "dispatch.cuh"

namespace nbk {
void* persist_kp_ptr(int m, int kpad) {
  switch (m) {
    case 1: return cluster_kp_m<1>(kpad);
    case 2: return cluster_kp_m<2>(kpad);
    case 3: return cluster_kp_m<3>(kpad);
    case 4: return cluster_kp_m<4>(kpad);
    case 5: return cluster_kp_m<5>(kpad);
    case 6: return cluster_kp_m<6>(kpad);
    case 7: return cluster_kp_m<7>(kpad);
    case 8: return cluster_kp_m<8>(kpad);
  }
  return nullptr;
}

}  // namespace nbk
