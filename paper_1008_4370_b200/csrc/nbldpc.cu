// nbldpc.cu -- host side of the C-ABI declared in include/nbldpc.h.
//
// Builds the immutable code tables (GF(2^m) exp/log, the k_max-padded edge
// table with the Fourier-domain permutation bases of PAPER.md Appendix A), owns
// the per-handle workspace (frame slots resident in L2/HBM), and drives the
// pass kernel either through a CUDA graph whose WHILE conditional node loops on
// the device until every frame has stopped, or through a host launch loop.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/nbldpc.h"
#define NB_CONTROL_KERNELS  // the setup / control kernels live in this translation unit
#include "decoder.cuh"
#include "logsp.cuh"
#include "lf_general.cuh"
#include "kernels.h"
#include "lf_cluster.cuh"

using nb::CallDev;
using nb::CodeDev;
using nb::EdgeDev;
using nb::PassParams;
using nb::WorkDev;

namespace {

constexpr int kPassesPerGraphIter = 8;               // pass kernels per WHILE-body iteration
constexpr size_t kDefaultSlotBudget = 64ull << 20;  // bytes of slot state kept L2-resident
constexpr int kBigBlock = 512;                       // block-size variant for k_max * TT > 256
constexpr int kMaxColWeight = 16;                    // column weights 1..16 (the general kernel)
constexpr int kMaxChunks = 16;                       // nbldpc_decode_host: host-to-device copy chunks

struct Workspace {
  int S = 0, Y = 1;
  void* base = nullptr;
  size_t bytes = 0;
  WorkDev dev{};
  int32_t* host_flag = nullptr;  // pinned, host loop
  cudaGraphExec_t graph = nullptr;
  int graph_direct = 0;           // VN algorithm the graph was built with
  float* llr_stage = nullptr;  // device staging for nbldpc_decode_host
  size_t llr_stage_bytes = 0;
  uint8_t* out_stage = nullptr;
  size_t out_stage_bytes = 0;
  cudaStream_t copy_stream = nullptr;  // nbldpc_decode_host: the host-to-device copies
  cudaEvent_t ev_start = nullptr, ev_first = nullptr;
  int32_t* chunk_flags = nullptr;       // [kMaxChunks]
  float* p0buf = nullptr;  // nbldpc_decode_pmf: [S][N][q] channel spectra
  size_t p0buf_bytes = 0;
  void* ls_base = nullptr;  // conventional Log-SP: W [2][S][E][q], L0 [S][N][q], xhat [S][N], counter
  size_t ls_bytes = 0;
  cudaEvent_t ev_done = nullptr;  // recorded on the stream of every decode that used this workspace
  // launch accounting of the most recent decode
  cudaStream_t last_stream = nullptr;
  int last_graph = 0;
  long long last_host_launches = 0;
};

}  // namespace

struct nbldpc_code_s {
  int device = 0;
  int m = 0, q = 0, M = 0, N = 0, E = 0, k_max = 0, kpad = 4, con_stride = 16;
  bool row_regular = true;
  uint32_t poly = 0;
  EdgeDev* edges_d = nullptr;
  uint8_t* gf_exp_d = nullptr;
  uint8_t* gf_log_d = nullptr;
  uint64_t* pinv_tab_d = nullptr;
  // variable -> edges (internal slots), for the general-column-weight kernel
  int j_max = 2, nnz = 0;
  bool colw2 = true;  // every column has weight 2: the cluster / pass kernels apply
  int32_t* v_ptr_d = nullptr;
  int32_t* v_edges_d = nullptr;
  std::mutex mu;
  Workspace ws;
  // launch geometry of the pass kernel (NBLDPC_VN_DIRECT)
  int TT = 1, TPC = 1, CPC = 1, groups = 1, block = 32, big = 0, blocks_per_sm = 1, sms = 148;  // TPC padded
  size_t smem = 0;
  // launch geometry of the cluster kernel (NBLDPC_VN_SEPARABLE): TPC a power of two, clusters of
  // p_cs CTAs per frame, p_ncl clusters resident
  int p_tpc = 1, p_cpc = 1, p_groups = 1, p_block = 32, p_big = 0, p_cs = 1, p_ncl = 1, p_recs = 0;
  int p_kp = 0;  // > 0: the plain LLR launch uses the compile-time-geometry instantiation (KP = kpad)
  size_t p_smem = 0;
  size_t p_smem_pmf = 0;  // the pmf variant: + its staged pmf rows for one-thread teams (PSTAGE)
  // false: the cluster kernel cannot run this code (its per-CTA edge records do not fit in shared memory
  // even with 16-CTA clusters, or no cluster fits on the GPU): NBLDPC_VN_SEPARABLE decodes run the
  // general-column-weight kernel instead (same results up to rounding)
  bool cluster_ok = true;
};

namespace {

thread_local char g_last_error[256] = "";

nbldpc_status_t cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return NBLDPC_OK;
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return NBLDPC_ERR_OUT_OF_MEMORY;
  return NBLDPC_ERR_CUDA;
}

#define NB_TRY(expr)                               \
  do {                                             \
    cudaError_t e_ = (expr);                       \
    if (e_ != cudaSuccess) return cuda_status(e_); \
  } while (0)

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int team_threads(int m) { return m <= 4 ? 1 : (1 << m) / 16; }

int team_floats(int m) {
  const int q = 1 << m;
  const int tt = team_threads(m);
  const int pad = (tt > 1 && tt < 8) ? 4 * tt : 0;
  return 5 * (q + pad) + 16;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t slot_bytes_of(const nbldpc_code_s* c) {
  const size_t q = c->q;
  size_t b = 0;
  b += 2 * (size_t)c->E * q * sizeof(float);  // W ping-pong
  b += (size_t)c->N * 8 * sizeof(float);      // tanh (rows of 8)
  b += (size_t)c->N;                          // xhat
  b += (size_t)c->N * c->m * sizeof(float);   // soft
  b += (size_t)c->con_stride;                 // syndrome contributions
  b += 5 * sizeof(int32_t);
  return b;
}

void free_workspace(Workspace& w) {
  // the handle's last decode may still run (stream-ordered buffers are not freed synchronously): wait for it
  if (w.ev_done) cudaEventSynchronize(w.ev_done);
  if (w.graph) cudaGraphExecDestroy(w.graph);
  if (w.base) cudaFree(w.base);
  if (w.host_flag) cudaFreeHost(w.host_flag);
  if (w.llr_stage) cudaFree(w.llr_stage);
  if (w.out_stage) cudaFree(w.out_stage);
  if (w.p0buf) cudaFree(w.p0buf);
  if (w.ls_base) cudaFree(w.ls_base);
  if (w.copy_stream) cudaStreamDestroy(w.copy_stream);
  if (w.ev_start) cudaEventDestroy(w.ev_start);
  if (w.ev_first) cudaEventDestroy(w.ev_first);
  if (w.chunk_flags) cudaFree(w.chunk_flags);
  if (w.ev_done) cudaEventDestroy(w.ev_done);
  w = Workspace{};
}

// the slot-pass kernel for a VN variant (0 separable, 1 direct, 2 pmf), soft = 1: its soft-output instantiation
void* pass_kernel_ptr(int m, int big, int direct, int soft = 0) {
  return soft ? nbk::pass_kernel_soft_ptr(m, big, direct) : nbk::pass_kernel_ptr(m, big, direct);
}
using nbk::persist_kp_ptr;

// pmf = 1: the nbldpc_decode_pmf variant; f16 = 1: half-precision messages (NBLDPC_MSG_F16);
// sym = 1: the symbol-output variant (LLR input)
void* persist_kernel_ptr(int m, int big, int pmf = 0, int f16 = 0, int sym = 0, int soft = 0) {
  if (soft) return (sym && (pmf || f16)) ? nullptr : nbk::persist_soft_ptr(m, big, sym ? 3 : f16 ? 2 : pmf ? 1 : 0);
  if (sym) return (pmf || f16) ? nullptr : nbk::persist_sym_ptr(m, big);
  if (f16) return pmf ? nullptr : nbk::persist_f16_ptr(m, big);
  return pmf ? nbk::persist_pmf_ptr(m, big) : nbk::persist_plain_ptr(m, big);
}
// shared-memory words per edge team of the cluster kernel (nb::CCfg<m>::TEAM)
int persist_team_words(int m) {
  switch (m) {
    case 1: return nb::CCfg<1>::TEAMW;
    case 2: return nb::CCfg<2>::TEAMW;
    case 3: return nb::CCfg<3>::TEAMW;
    case 4: return nb::CCfg<4>::TEAMW;
    case 5: return nb::CCfg<5>::TEAMW;
    case 6: return nb::CCfg<6>::TEAMW;
    case 7: return nb::CCfg<7>::TEAMW;
    case 8: return nb::CCfg<8>::TEAMW;
  }
  return 0;
}

cudaError_t launch_cluster(const nbldpc_code_s* c, const nb::ClusterParams& P, int ncl, cudaStream_t st, int pmf = 0,
                           int f16 = 0, int sym = 0, int soft = 0) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ncl * c->p_cs));
  cfg.blockDim = dim3((unsigned)c->p_block);
  cfg.dynamicSmemBytes = pmf ? c->p_smem_pmf : c->p_smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)c->p_cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<nb::ClusterParams*>(&P)};
  void* fn = (c->p_kp && !pmf && !f16 && !sym && !soft) ? persist_kp_ptr(c->m, c->p_kp)
                                                        : persist_kernel_ptr(c->m, c->p_big, pmf, f16, sym, soft);
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a property of the kernel (one instantiation per
// (m, block variant)) shared by every code on the device: only ever raise it.
std::mutex g_attr_mu;
size_t g_attr_smem[64][108] = {};

cudaError_t ensure_smem_attr(const nbldpc_code_s* c) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  for (int direct = 0; direct < 6; ++direct) {  // 3 VN variants x {plain, soft}
    const int d = c->device & 63, k = (c->m * 2 + c->big) * 6 + direct;
    if (g_attr_smem[d][k] >= c->smem) continue;
    cudaError_t e = cudaFuncSetAttribute(pass_kernel_ptr(c->m, c->big, direct % 3, direct / 3),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem);
    if (e != cudaSuccess) return e;
    g_attr_smem[d][k] = c->smem;
  }
  static size_t p_attr[64][18 * 9 + 32] = {};
  for (int var = 0; c->cluster_ok && var < 9; ++var) {
    // plain, pmf, f16, compile-time geometry, symbol outputs; then the soft-output plain, pmf, f16, sym
    const int soft = var >= 5;
    const int pmf = var == 1 || var == 6, f16 = var == 2 || var == 7, sym = var == 4 || var == 8;
    void* fn = var == 3 ? (c->p_kp ? persist_kp_ptr(c->m, c->p_kp) : nullptr)
                        : persist_kernel_ptr(c->m, c->p_big, pmf, f16, sym, soft);
    if (!fn) continue;
    if (c->p_cs > 8) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    // one cache slot per kernel: (m, big, variant), or (m, kpad) for the compile-time-geometry one
    int k = (c->m * 2 + c->p_big) * 9 + var;
    if (var == 3) k = 18 * 9 + (c->m - 1) * 4 + (c->p_kp == 4 ? 0 : c->p_kp == 8 ? 1 : c->p_kp == 16 ? 2 : 3);
    const int d = c->device & 63;
    const size_t need = pmf ? c->p_smem_pmf : c->p_smem;
    if (p_attr[d][k] < need) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
      if (e != cudaSuccess) return e;
      p_attr[d][k] = need;
    }
  }
  return cudaSuccess;
}

// Slot lanes Y: CTA (g, y) processes slots y, y+Y, ... .  Minimise the makespan
// ceil(G*Y / resident CTAs) * ceil(S / Y) (waves x slots per CTA).
int choose_lanes(const nbldpc_code_s* c, int S) {
  const long target = (long)c->blocks_per_sm * c->sms;
  int best = 1;
  long best_cost = -1;
  for (int Y = 1; Y <= S; ++Y) {
    const long per = (S + Y - 1) / Y;
    if (per > nb::kMaxSlotsPerCta) continue;
    const long waves = ((long)c->groups * Y + target - 1) / target;
    const long cost = waves * per;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = Y;
    }
  }
  return best;
}

// Carves the slot state of S resident frames out of `b` (NULL: sizing only); returns the bytes used.
// Layout: W [2][S][E][q] | Tt [S][N][8] | xhat | soft | con (syndrome contributions, zeroed) | per-slot
// counters | glob[16] | CallDev.  Everything from `con` on must be zero before the first decode.
size_t layout_workspace(const nbldpc_code_s* c, int S, char* b, WorkDev* dev, size_t* zero_from = nullptr) {
  const size_t q = c->q;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t oW = take(2 * (size_t)S * c->E * q * sizeof(float));
  const size_t oT = take((size_t)S * c->N * 8 * sizeof(float));
  const size_t oX = take((size_t)S * c->N);
  const size_t oS = take((size_t)S * c->N * c->m * sizeof(float));
  const size_t oP = take((size_t)S * c->con_stride);
  const size_t oF = take((size_t)S * sizeof(int32_t));
  const size_t oI = take((size_t)S * sizeof(int32_t));
  const size_t oV = take((size_t)S * sizeof(int32_t));
  const size_t oC = take((size_t)S * sizeof(int32_t));
  const size_t oE = take((size_t)S * sizeof(int32_t));
  const size_t oG = take(16 * sizeof(int32_t));
  const size_t oK = take(sizeof(CallDev));
  if (zero_from) *zero_from = oP;
  if (b && dev) {
    *dev = WorkDev{};
    dev->S = S;
    dev->W = reinterpret_cast<float*>(b + oW);
    dev->Tt = reinterpret_cast<float*>(b + oT);
    dev->xhat = reinterpret_cast<uint8_t*>(b + oX);
    dev->soft = reinterpret_cast<float*>(b + oS);
    dev->con = reinterpret_cast<uint8_t*>(b + oP);
    dev->con_stride = c->con_stride;
    dev->slot_frame = reinterpret_cast<int32_t*>(b + oF);
    dev->slot_iter = reinterpret_cast<int32_t*>(b + oI);
    dev->slot_events = reinterpret_cast<int32_t*>(b + oV);
    dev->slot_counter = reinterpret_cast<int32_t*>(b + oC);
    dev->slot_epoch = reinterpret_cast<int32_t*>(b + oE);
    dev->glob = reinterpret_cast<int32_t*>(b + oG);
    dev->call = reinterpret_cast<CallDev*>(b + oK);
  }
  return off;
}

// Grows a handle buffer to >= need bytes, stream-ordered on `st` (no host or device-wide sync): the
// old buffer is released with cudaFreeAsync after the handle's previous decode (event ev_done, which
// may have run on another stream) and everything earlier on `st`; the new one comes from
// cudaMallocAsync on `st`.
template <class T>
nbldpc_status_t grow_buffer(Workspace& w, T** buf, size_t* have, size_t need, cudaStream_t st) {
  if (*buf && *have >= need) return NBLDPC_OK;
  if (*buf) {
    if (w.ev_done) NB_TRY(cudaStreamWaitEvent(st, w.ev_done, 0));
    NB_TRY(cudaFreeAsync(*buf, st));
    *buf = nullptr;
    *have = 0;
  }
  void* p = nullptr;
  NB_TRY(cudaMallocAsync(&p, need, st));
  *buf = static_cast<T*>(p);
  *have = need;
  return NBLDPC_OK;
}

// the decode just enqueued on `st` used the handle's workspace: later reallocations wait for it
nbldpc_status_t mark_done(Workspace& w, cudaStream_t st) {
  if (!w.ev_done) NB_TRY(cudaEventCreateWithFlags(&w.ev_done, cudaEventDisableTiming));
  NB_TRY(cudaEventRecord(w.ev_done, st));
  return NBLDPC_OK;
}

// The handle's slot state for S resident frames, re-carved (and grown, stream-ordered) when S changes.
nbldpc_status_t ensure_workspace(nbldpc_code_s* c, int S, cudaStream_t st) {
  Workspace& w = c->ws;
  if (w.base && w.S == S) return NBLDPC_OK;
  if (w.graph) {  // captured the old slot layout; an in-flight launch completes before it is freed
    cudaGraphExecDestroy(w.graph);
    w.graph = nullptr;
  }
  size_t zero_from = 0;
  const size_t off = layout_workspace(c, S, nullptr, nullptr, &zero_from);
  void* base = w.base;
  nbldpc_status_t rs = grow_buffer(w, &base, &w.bytes, off, st);
  w.base = base;
  if (rs != NBLDPC_OK) {
    w.S = 0;
    return rs;
  }
  char* b = static_cast<char*>(base);
  if (w.ev_done) NB_TRY(cudaStreamWaitEvent(st, w.ev_done, 0));  // a previous decode may still use it
  NB_TRY(cudaMemsetAsync(b + zero_from, 0, off - zero_from, st));  // padding edge slots of `con` stay zero
  w.S = S;
  w.Y = choose_lanes(c, S);
  layout_workspace(c, S, b, &w.dev);
  if (!w.host_flag) NB_TRY(cudaMallocHost(&w.host_flag, 64));
  return NBLDPC_OK;
}

PassParams make_params(const nbldpc_code_s* c, int step_mode, float* u_out) {  // NOLINT
  PassParams P{};
  P.code.m = c->m;
  P.code.M = c->M;
  P.code.N = c->N;
  P.code.E = c->E;
  P.code.k_max = c->k_max;
  P.code.kpad = c->kpad;
  P.code.edges = c->edges_d;
  P.code.gf_exp = c->gf_exp_d;
  P.code.gf_log = c->gf_log_d;
  P.code.pinv_tab = c->pinv_tab_d;
  P.ws = c->ws.dev;
  P.groups = c->groups;
  P.slot_lanes = c->ws.Y;
  P.checks_per_cta = c->CPC;
  P.tpc = c->TPC;
  P.step_mode = step_mode;
  P.u_out = u_out;
  return P;
}

nb::ClusterParams make_cparams(const nbldpc_code_s* c, int step_mode, int step_iter, float* u_out,
                               const WorkDev* dev = nullptr);

template <int MB>
cudaError_t launch_layout_t(const nb::CodeDev& cd, const float* src, float* dst, int frames, int to_kernel, int lin,
                            cudaStream_t st) {
  nb::nb_msg_layout_kernel<MB><<<512, 256, 0, st>>>(src, dst, frames, cd, to_kernel, lin);
  return cudaGetLastError();
}
// lin = 1: the cluster kernel stores linear messages (its plain / KP / pmf / symbol instantiations for
// m >= 7, see LIN in lf_cluster.cuh); lin = 0: the packed log format (all others)
cudaError_t launch_layout(const nbldpc_code_s* c, const float* src, float* dst, int frames, int to_kernel, int lin,
                          cudaStream_t st) {
  const nb::CodeDev cd = make_cparams(c, 0, 0, nullptr).code;
  switch (c->m) {
    case 1: return launch_layout_t<1>(cd, src, dst, frames, to_kernel, lin, st);
    case 2: return launch_layout_t<2>(cd, src, dst, frames, to_kernel, lin, st);
    case 3: return launch_layout_t<3>(cd, src, dst, frames, to_kernel, lin, st);
    case 4: return launch_layout_t<4>(cd, src, dst, frames, to_kernel, lin, st);
    case 5: return launch_layout_t<5>(cd, src, dst, frames, to_kernel, lin, st);
    case 6: return launch_layout_t<6>(cd, src, dst, frames, to_kernel, lin, st);
    case 7: return launch_layout_t<7>(cd, src, dst, frames, to_kernel, lin, st);
    default: return launch_layout_t<8>(cd, src, dst, frames, to_kernel, lin, st);
  }
}

nb::ClusterParams make_cparams(const nbldpc_code_s* c, int step_mode, int step_iter, float* u_out,
                               const WorkDev* dev) {
  nb::ClusterParams P{};
  P.code.m = c->m;
  P.code.M = c->M;
  P.code.N = c->N;
  P.code.E = c->E;
  P.code.k_max = c->k_max;
  P.code.kpad = c->kpad;
  P.code.edges = c->edges_d;
  P.code.gf_exp = c->gf_exp_d;
  P.code.gf_log = c->gf_log_d;
  P.code.pinv_tab = c->pinv_tab_d;
  P.ws = dev ? *dev : c->ws.dev;
  P.chunks = c->p_groups;
  P.checks_per_cta = c->p_cpc;
  P.tpc = c->p_tpc;
  P.step_mode = step_mode;
  P.step_iter = step_iter;
  P.rec_per_cta = c->p_recs;
  P.u_out = u_out;
  return P;
}

dim3 pass_grid(const nbldpc_code_s* c) { return dim3((unsigned)(c->groups * c->ws.Y)); }

cudaError_t launch_pass(const nbldpc_code_s* c, const PassParams& P, int direct, cudaStream_t st, int soft = 0) {
  void* args[] = {const_cast<PassParams*>(&P)};
  return cudaLaunchKernel(pass_kernel_ptr(c->m, c->big, direct, soft), pass_grid(c), dim3(c->block), args, c->smem, st);
}

nbldpc_status_t build_graph(nbldpc_code_s* c, int direct, int soft = 0) {
  Workspace& w = c->ws;
  if (w.graph && w.graph_direct == direct + 3 * soft) return NBLDPC_OK;
  if (w.graph) {
    cudaGraphExecDestroy(w.graph);
    w.graph = nullptr;
  }
  cudaGraph_t g = nullptr;
  NB_TRY(cudaGraphCreate(&g, 0));
  auto fail = [&](cudaError_t e) {
    cudaGraphDestroy(g);
    return cuda_status(e);
  };
  cudaGraphConditionalHandle h;
  if (cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault)) return fail(e);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cn;
  if (cudaError_t e = cudaGraphAddNode(&cn, g, nullptr, 0, &cp)) return fail(e);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  PassParams P = make_params(c, 0, nullptr);  // node parameters are copied at creation
  cudaGraphNode_t prev = nullptr;
  for (int i = 0; i < kPassesPerGraphIter; ++i) {
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    kp.kernel.func = pass_kernel_ptr(c->m, c->big, direct, soft);
    kp.kernel.gridDim = pass_grid(c);
    kp.kernel.blockDim = dim3(c->block);
    kp.kernel.sharedMemBytes = (unsigned)c->smem;
    void* args[] = {&P};
    kp.kernel.kernelParams = args;
    cudaGraphNode_t kn;
    if (cudaError_t e = cudaGraphAddNode(&kn, body, prev ? &prev : nullptr, prev ? 1 : 0, &kp)) return fail(e);
    prev = kn;
  }
  {
    cudaGraphNodeParams kp = {};
    kp.type = cudaGraphNodeTypeKernel;
    kp.kernel.func = reinterpret_cast<void*>(&nb::nb_control_kernel);
    kp.kernel.gridDim = dim3(1);
    kp.kernel.blockDim = dim3(32);
    int32_t* glob = w.dev.glob;
    void* args[] = {&glob, &h};
    kp.kernel.kernelParams = args;
    cudaGraphNode_t kn;
    if (cudaError_t e = cudaGraphAddNode(&kn, body, &prev, 1, &kp)) return fail(e);
  }
  cudaError_t e = cudaGraphInstantiate(&w.graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    w.graph = nullptr;
    return cuda_status(e);
  }
  w.graph_direct = direct + 3 * soft;
  return NBLDPC_OK;
}

int default_slots(const nbldpc_code_s* c, int frames) {
  const size_t sb = slot_bytes_of(c);
  long S = (long)(kDefaultSlotBudget / sb);
  if (S < 1) S = 1;
  if (S > frames) S = frames;
  return (int)S;
}

// ---- conventional Log-SP (NBLDPC_ALG_LOG_SP): one CTA per frame, persistent
using nbk::ls_kernel_ptr;

nbldpc_status_t decode_logsp(nbldpc_code_s* c, const float* llr, const float* pmf, int frames, int max_iters,
                             uint8_t* hard, uint8_t* ok, int32_t* iters, int early, cudaStream_t st) {
  NB_TRY(cudaSetDevice(c->device));
  const int q = c->q, tt = q < 16 ? 1 : q / 16;
  // teams of tt threads, each with (k_max + 1) vectors of q floats in shared memory; at most 256
  // threads and ~200 KB per CTA
  const size_t per_team = (size_t)(c->k_max + 1) * q * sizeof(float);
  const size_t tables = (size_t)3 * q * sizeof(int);
  int teams = std::min(256 / tt, (int)((200u * 1024u - tables) / per_team));
  if (teams < 1) return NBLDPC_ERR_UNSUPPORTED;
  const int threads = ((teams * tt + 31) / 32) * 32;
  const size_t smem = teams * per_team + tables;
  void* fn = ls_kernel_ptr(c->m);
  NB_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  NB_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  if (per_sm < 1) return NBLDPC_ERR_UNSUPPORTED;
  const int S = std::min(frames, per_sm * c->sms);
  Workspace& w = c->ws;
  const size_t bW = align_up(2 * (size_t)S * c->E * q * sizeof(float), 256);
  const size_t bL = align_up((size_t)S * c->N * q * sizeof(float), 256);
  const size_t bX = align_up((size_t)S * c->N, 256);
  const size_t need = bW + bL + bX + 256;
  {
    nbldpc_status_t rs = grow_buffer(w, &w.ls_base, &w.ls_bytes, need, st);
    if (rs != NBLDPC_OK) return rs;
  }
  char* b = static_cast<char*>(w.ls_base);
  nb::LsParams P{};
  P.code = make_params(c, 0, nullptr).code;
  P.W = reinterpret_cast<float*>(b);
  P.L0s = reinterpret_cast<float*>(b + bW);
  P.xh = reinterpret_cast<uint8_t*>(b + bW + bL);
  P.glob = reinterpret_cast<int32_t*>(b + bW + bL + bX);
  P.llr = llr;
  P.pmf = pmf;
  P.hard = hard;
  P.ok = ok;
  P.iters = iters;
  P.frames = frames;
  P.max_iters = max_iters;
  P.early_stop = early;
  P.teams = teams;
  P.kmax = c->k_max;
  NB_TRY(cudaMemsetAsync(P.glob, 0, sizeof(int32_t), st));
  void* args[] = {&P};
  NB_TRY(cudaLaunchKernel(fn, dim3((unsigned)S), dim3((unsigned)threads), args, smem, st));
  w.last_stream = st;
  w.last_graph = 0;
  w.last_host_launches = 1;
  return mark_done(w, st);
}

// ---- any column weight (NBLDPC_VN_GENERAL, lf_general.cuh): one CTA per frame, persistent
using nbk::gen_kernel_ptr;

nbldpc_status_t decode_general(nbldpc_code_s* c, const float* llr, const float* pmf, int frames, int max_iters,
                               uint8_t* hard, uint8_t* ok, int32_t* iters, int early, float* soft, int32_t* events,
                               float* post, uint8_t* xmap, cudaStream_t st) {
  NB_TRY(cudaSetDevice(c->device));
  const int q = c->q, tt = q < 16 ? 1 : q / 16;
  const int vs = std::max(2, c->j_max);  // as the kernel's VS: >= 2 vectors (TOT and a staged U row)
  const int ts = vs * q + ((tt - (vs * q) % 32) & 31);  // the kernel's padded team stride (floats)
  const size_t per_team = (size_t)ts * sizeof(float);
  const size_t tables = (size_t)3 * q * sizeof(int);
  const int teams = std::min(256 / tt, (int)((100u * 1024u - tables) / per_team));
  if (teams < 1) return NBLDPC_ERR_UNSUPPORTED;
  const int threads = ((teams * tt + 31) / 32) * 32;
  const size_t smem = teams * per_team + tables;
  void* fn = gen_kernel_ptr(c->m, soft != nullptr);
  NB_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  NB_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
  if (per_sm < 1) return NBLDPC_ERR_UNSUPPORTED;
  const int S = std::min(frames, per_sm * c->sms);
  Workspace& w = c->ws;
  const size_t bM = align_up((size_t)S * c->E * q * sizeof(float), 256);
  const size_t bX = align_up((size_t)S * c->N, 256);
  const size_t need = 2 * bM + bX + 256;
  {  // shares the Log-SP workspace (one decode per handle at a time)
    nbldpc_status_t rs = grow_buffer(w, &w.ls_base, &w.ls_bytes, need, st);
    if (rs != NBLDPC_OK) return rs;
  }
  char* b = static_cast<char*>(w.ls_base);
  nb::GenParams P{};
  P.code = make_params(c, 0, nullptr).code;
  P.v_ptr = c->v_ptr_d;
  P.v_edges = c->v_edges_d;
  P.U = reinterpret_cast<float*>(b);
  P.W = reinterpret_cast<float*>(b + bM);
  P.xh = reinterpret_cast<uint8_t*>(b + 2 * bM);
  P.glob = reinterpret_cast<int32_t*>(b + 2 * bM + bX);
  P.llr = llr;
  P.pmf = pmf;
  P.hard = hard;
  P.ok = ok;
  P.iters = iters;
  P.soft_out = soft;
  P.events_out = events;
  P.post_out = post;
  P.map_out = xmap;
  P.frames = frames;
  P.max_iters = max_iters;
  P.early_stop = early;
  P.teams = teams;
  P.jmax = c->j_max;
  NB_TRY(cudaMemsetAsync(P.glob, 0, sizeof(int32_t), st));
  void* args[] = {&P};
  NB_TRY(cudaLaunchKernel(fn, dim3((unsigned)S), dim3((unsigned)threads), args, smem, st));
  w.last_stream = st;
  w.last_graph = 0;
  w.last_host_launches = 1;
  return mark_done(w, st);
}

// Copies caller options into a zeroed struct: callers built against the round-1 header (without the
// workspace fields) pass a smaller struct_size, and fields past it read as zero.
constexpr size_t kOptsV1Size = offsetof(nbldpc_decode_opts_t, workspace);
bool normalise_opts(const nbldpc_decode_opts_t* in, nbldpc_decode_opts_t* out) {
  std::memset(out, 0, sizeof(*out));
  out->struct_size = sizeof(*out);
  if (!in) return true;
  if (in->struct_size < kOptsV1Size) return false;
  std::memcpy(out, in, std::min(in->struct_size, sizeof(*out)));
  out->struct_size = sizeof(*out);
  return true;
}

// pmf != NULL: nbldpc_decode_pmf (llr unused; the direct kernel with the general channel spectrum)
// chunk_flags: nbldpc_decode_host's arrival flags (cluster path only; see there)
// opts->workspace != NULL: the caller's workspace (cluster kernel only); the handle's state is not
// touched, so the caller need not hold the handle lock (see nbldpc_decode_ex)
nbldpc_status_t decode_impl(nbldpc_code_s* c, const float* llr, int frames, int max_iters, uint8_t* hard,
                            uint8_t* ok, int32_t* iters, cudaStream_t st, const nbldpc_decode_opts_t* opts,
                            const float* pmf = nullptr, const int32_t* chunk_flags = nullptr, int chunk_frames = 0) {
  int mode = 0, early = 1, slots = 0, use_graph = 0, direct = 0;
  float* soft = nullptr;
  int32_t* events = nullptr;
  float* post = nullptr;
  uint8_t* xmap = nullptr;
  int f16 = 0;
  nbldpc_decode_opts_t onorm;
  if (!normalise_opts(opts, &onorm)) return NBLDPC_ERR_INVALID_ARGUMENT;
  void* user_ws = onorm.workspace;
  const size_t user_ws_bytes = onorm.workspace_bytes;
  if (opts) {
    opts = &onorm;
    mode = opts->syndrome_mode;
    early = opts->no_early_stop ? 0 : 1;
    soft = opts->soft_out;
    events = opts->events_out;
    slots = opts->slots;
    use_graph = opts->use_graph;
    direct = opts->vn_algorithm;
    post = opts->symbol_post_out;
    xmap = opts->symbol_map_out;
    if (opts->message_format != NBLDPC_MSG_F32 && opts->message_format != NBLDPC_MSG_F16) return NBLDPC_ERR_INVALID_ARGUMENT;
    f16 = opts->message_format == NBLDPC_MSG_F16;
    if (f16 && (opts->algorithm != NBLDPC_ALG_LOG_FOURIER || opts->vn_algorithm != NBLDPC_VN_SEPARABLE || pmf || post ||
                xmap || !c->colw2))
      return NBLDPC_ERR_INVALID_ARGUMENT;  // half messages: the cluster kernel with LLR input
    if (f16 && c->m < 3) return NBLDPC_ERR_UNSUPPORTED;
    if (opts->algorithm == NBLDPC_ALG_LOG_SP) {
      // the comparison algorithm: symbol-MAP decisions and the exact syndrome only
      if (mode != 0 || soft || events || post || xmap) return NBLDPC_ERR_INVALID_ARGUMENT;
      if (!c->colw2) return NBLDPC_ERR_UNSUPPORTED;  // its variable node is the degree-2 one
      return decode_logsp(c, llr, pmf, frames, max_iters, hard, ok, iters, early, st);
    }
    if (opts->algorithm != NBLDPC_ALG_LOG_FOURIER) return NBLDPC_ERR_INVALID_ARGUMENT;
  }
  if ((post && (!is_device_ptr(post) || ((uintptr_t)post & 15))) || (xmap && !is_device_ptr(xmap)))
    return NBLDPC_ERR_INVALID_ARGUMENT;
  if (mode != 0 && mode != 1) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (direct < 0 || direct > 2) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (f16 && !c->cluster_ok) return NBLDPC_ERR_UNSUPPORTED;  // half messages live in the cluster kernel only
  if (!c->cluster_ok && direct == 0 && !(pmf && (post || xmap))) direct = 2;  // cluster kernel cannot hold this code
  if (!c->colw2 || direct == 2) {  // column weights != 2, or asked for: the general kernel
    if (mode != 0) return NBLDPC_ERR_INVALID_ARGUMENT;
    if ((soft && !is_device_ptr(soft)) || (events && !is_device_ptr(events))) return NBLDPC_ERR_INVALID_ARGUMENT;
    return decode_general(c, llr, pmf, frames, max_iters, hard, ok, iters, early, soft, events, post, xmap, st);
  }
  if ((post || xmap) && direct == 0 && pmf) direct = 1;  // pmf + symbol outputs: the pass kernel
  if (pmf && direct == 0 && c->p_smem_pmf > 227 * 1024) direct = 1;  // staged pmf rows do not fit: the pass kernel
  if (pmf && direct) direct = 2;                   // the pass kernel's pmf variant
  if (slots < 0) return NBLDPC_ERR_INVALID_ARGUMENT;
  if ((soft && !is_device_ptr(soft)) || (events && !is_device_ptr(events))) return NBLDPC_ERR_INVALID_ARGUMENT;
  int S = slots > 0 ? std::min(slots, frames) : default_slots(c, frames);
  if (!direct) S = std::min(slots > 0 ? slots : c->p_ncl, std::min(c->p_ncl, frames));  // slots = clusters
  NB_TRY(cudaSetDevice(c->device));
  Workspace& w = c->ws;
  nbldpc_status_t rs = NBLDPC_OK;
  WorkDev udev{};
  if (user_ws) {
    // the caller's workspace (nbldpc_decode_opts_t::workspace): cluster kernel, LLR input only
    if (direct || pmf || chunk_flags) return NBLDPC_ERR_UNSUPPORTED;
    size_t zero_from = 0;
    const size_t need = layout_workspace(c, S, nullptr, nullptr, &zero_from);
    if (user_ws_bytes < need || ((uintptr_t)user_ws & 255) || !is_device_ptr(user_ws))
      return NBLDPC_ERR_INVALID_ARGUMENT;
    layout_workspace(c, S, static_cast<char*>(user_ws), &udev);
    NB_TRY(cudaMemsetAsync(static_cast<char*>(user_ws) + zero_from, 0, need - zero_from, st));
  } else {
    rs = ensure_workspace(c, S, st);
    if (rs != NBLDPC_OK) return rs;
  }
  const WorkDev& dv = user_ws ? udev : w.dev;
  CallDev call{};
  if (pmf) {
    const size_t need = (size_t)S * c->N * c->q * sizeof(float);
    rs = grow_buffer(w, &w.p0buf, &w.p0buf_bytes, need, st);  // stream-ordered (a previous pmf decode may read it)
    if (rs != NBLDPC_OK) return rs;
    call.pmf = pmf;
    call.p0buf = w.p0buf;
  }
  call.post_out = post;
  call.map_out = xmap;
  if (!direct) {
    call.chunk_flags = chunk_flags;
    call.chunk_frames = chunk_frames;
  }
  call.llr = llr;
  call.hard = hard;
  call.ok = ok;
  call.iters = iters;
  call.soft_out = soft;
  call.events_out = events;
  call.frames = frames;
  call.max_iters = max_iters;
  call.mode = mode;
  call.early_stop = early;
  call.want_soft = soft != nullptr;
  if (direct) {
    nb::nb_setup_kernel<<<(S + 255) / 256, 256, 0, st>>>(w.dev, call);
  } else {
    nb::nb_cluster_setup_kernel<<<(S + 255) / 256, 256, 0, st>>>(dv, call);
  }
  NB_TRY(cudaGetLastError());
  if (user_ws) {
    nb::ClusterParams PP = make_cparams(c, 0, 0, nullptr, &udev);
    NB_TRY(launch_cluster(c, PP, S, st, 0, f16, (post || xmap) ? 1 : 0, soft != nullptr));
    return NBLDPC_OK;
  }
  w.last_stream = st;
  w.last_graph = use_graph >= 0;
  w.last_host_launches = 1;
  if (!direct) {
    nb::ClusterParams PP = make_cparams(c, 0, 0, nullptr);
    NB_TRY(launch_cluster(c, PP, S, st, pmf != nullptr, f16, (post || xmap) ? 1 : 0, soft != nullptr));
    w.last_graph = 0;
    w.last_host_launches = 2;
    return mark_done(w, st);
  }
  if (use_graph >= 0) {
    rs = build_graph(c, direct, soft != nullptr);
    if (rs != NBLDPC_OK) return rs;
    NB_TRY(cudaGraphLaunch(w.graph, st));
    return mark_done(w, st);
  }
  // host-driven loop: launch passes, poll the active-slot counter every few passes
  PassParams P = make_params(c, 0, nullptr);
  for (;;) {
    for (int i = 0; i < kPassesPerGraphIter; ++i) {
      NB_TRY(launch_pass(c, P, direct, st, soft != nullptr));
      w.last_host_launches++;
    }
    NB_TRY(cudaMemcpyAsync(w.host_flag, w.dev.glob + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    NB_TRY(cudaStreamSynchronize(st));
    if (*w.host_flag == 0) break;
  }
  return mark_done(w, st);
}

// Which edge of a degree-2 variable evaluates its tentative decision ("is_a") is free: both give
// M_v = P^0 (*) W_a (*) W_b.  The cluster kernel runs an edge team per TT threads in barrier groups of
// max(32, kpad TT) threads (a warp, or one check when a check is wider than a warp); a group with no
// deciding edge skips the decision, while a group with any waits for it at its next barrier.  So
// choose the deciding groups as a small vertex cover of the graph whose nodes are groups and whose
// edges are variables (greedy: repeatedly the group covering most uncovered variables), and let each
// variable decide in a covering group.  (Measured cover: 82% of the checks of C4, 73% of C3, against
// 57% of the warps at warp granularity -- every check of those had some deciding warp.)
// q = 256 (tt = 16, two edge slots per warp): the cluster kernel computes a deciding team's decision with
// the whole warp (WARPDEC), so the best assignment gives every warp exactly one deciding slot.  The graph
// whose nodes are warps and whose edges are variables has degree <= 2 (a path or a cycle per component);
// walking each component and handing every variable to the warp the walk arrives at gives every warp at
// most one (on a cycle exactly one) deciding slot.
void orient_decision_owners(std::vector<EdgeDev>& edges, int E) {
  const int nw = (E + 1) / 2;
  std::vector<int> deg(nw, 0);
  for (int e = 0; e < E; ++e)
    if (edges[e].var >= 0) deg[e / 2]++;
  std::vector<char> done(E, 0);  // indexed by either slot of a variable (both set when assigned)
  auto walk = [&](int w) {
    for (;;) {
      int e = -1;
      for (int k = 2 * w; k < std::min(E, 2 * w + 2); ++k)
        if (edges[k].var >= 0 && !done[k]) { e = k; break; }
      if (e < 0) return;
      const int o = edges[e].partner;  // the variable's other slot; its warp decides
      done[e] = done[o] = 1;
      edges[e].is_a = 0;
      edges[o].is_a = 1;
      w = o / 2;
    }
  };
  for (int w = 0; w < nw; ++w)
    if (deg[w] == 1) walk(w);  // paths from one end first
  for (int w = 0; w < nw; ++w) walk(w);  // then the cycles
}

// q = 256 (tt = 16, two edge slots 2w, 2w + 1 per warp): the cluster kernel splits each variable's decision
// over its two edges (SPLITDEC in lf_cluster.cuh), with different code for the kind_a half and the other half,
// so a warp whose two slots are of the same kind runs one of them.  Walking the warp graph (degree <= 2)
// and alternating the kinds along it makes every warp uniform except one per odd cycle.
void orient_uniform_kinds(std::vector<EdgeDev>& edges, int E) {
  std::vector<char> done(E, 0);
  auto walk = [&](int s, int kind) {
    while (s < E && edges[s].var >= 0 && !done[s]) {
      const int p = edges[s].partner;
      edges[s].kind_a = (uint8_t)kind;
      edges[p].kind_a = (uint8_t)(1 - kind);
      done[s] = done[p] = 1;
      s = p ^ 1;         // the other slot of the partner's warp takes the partner's kind
      kind = 1 - kind;
    }
  };
  for (int w = 0; 2 * w < E; ++w) {  // path ends first: warps with one used slot
    const bool u0 = edges[2 * w].var >= 0, u1 = 2 * w + 1 < E && edges[2 * w + 1].var >= 0;
    if (u0 != u1) walk(u0 ? 2 * w : 2 * w + 1, 1);
  }
  for (int s = 0; s < E; ++s) walk(s, 1);  // then the cycles
}

void assign_decision_owners(std::vector<EdgeDev>& edges, int E, int tt, int kpad) {
#ifdef NB_WARPDEC
  if (tt == 16) {  // goes with the kernel's WARPDEC (off by default, see lf_cluster.cuh)
    orient_decision_owners(edges, E);
    return;
  }
#endif
  const int per = std::max(32 / tt, kpad);  // edge slots per barrier group
  const int nw = (E + per - 1) / per;
  std::vector<int> deg(nw, 0);
  for (int e = 0; e < E; ++e)
    if (edges[e].var >= 0 && edges[e].is_a) {
      deg[e / per]++;
      deg[edges[e].partner / per]++;
    }
  std::vector<char> covered_var(E, 0), in_cover(nw, 0);  // indexed by the variable's first edge slot
  std::vector<std::vector<int>> bucket(2 * per + 1);
  for (int w = 0; w < nw; ++w) bucket[std::min(deg[w], 2 * per)].push_back(w);
  int top = 2 * per;
  while (true) {
    while (top > 0 && bucket[top].empty()) --top;
    if (top == 0) break;
    const int w = bucket[top].back();
    bucket[top].pop_back();
    if (in_cover[w] || std::min(deg[w], 2 * per) != top) continue;  // stale entry
    in_cover[w] = 1;
    for (int e = w * per; e < std::min(E, (w + 1) * per); ++e) {
      if (edges[e].var < 0) continue;
      const int a = edges[e].is_a ? e : edges[e].partner;  // the variable's key slot
      if (covered_var[a]) continue;
      covered_var[a] = 1;
      const int o = (e == a ? edges[a].partner : a) / per;  // the other warp loses this variable
      if (!in_cover[o] && deg[o] > 0) {
        deg[o]--;
        bucket[std::min(deg[o], 2 * per)].push_back(o);
      }
    }
    deg[w] = 0;
  }
  for (int e = 0; e < E; ++e) {
    if (edges[e].var < 0 || !edges[e].is_a) continue;
    const int b = edges[e].partner;
    if (!in_cover[e / per] && in_cover[b / per]) {  // hand the decision to the covering warp
      edges[e].is_a = 0;
      edges[b].is_a = 1;
    }
  }
}

bool gf_tables(int m, uint32_t poly, std::vector<int>& ex, std::vector<int>& lg) {
  const int q = 1 << m;
  if ((poly >> m) != 1u) return false;
  ex.assign(2 * (q - 1) + 1, 0);
  lg.assign(q, -1);
  int a = 1;
  for (int i = 0; i < q - 1; ++i) {
    if (lg[a] != -1) return false;
    ex[i] = a;
    lg[a] = i;
    a <<= 1;
    if (a & q) a ^= (int)poly;
  }
  if (a != 1) return false;
  for (int i = q - 1; i < 2 * (q - 1); ++i) ex[i] = ex[i - (q - 1)];
  return true;
}

}  // namespace

extern "C" {

const char* nbldpc_last_cuda_error(void) { return g_last_error; }

const char* nbldpc_status_string(nbldpc_status_t s) {
  switch (s) {
    case NBLDPC_OK: return "ok";
    case NBLDPC_ERR_INVALID_ARGUMENT: return "invalid argument";
    case NBLDPC_ERR_NOT_PRIMITIVE: return "polynomial is not primitive of degree m";
    case NBLDPC_ERR_UNSUPPORTED: return "unsupported code or option combination (column weights 1..16, row degrees >= 2)";
    case NBLDPC_ERR_CUDA: return "CUDA error";
    case NBLDPC_ERR_OUT_OF_MEMORY: return "out of memory";
  }
  return "unknown status";
}

nbldpc_status_t nbldpc_code_create(int m, uint32_t prim_poly, int M, int N, int nnz, const int32_t* rows,
                                   const int32_t* cols, const uint16_t* coeffs, nbldpc_code_t* out) {
  if (!out || !rows || !cols || !coeffs) return NBLDPC_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (m < 1 || m > 8 || M <= 0 || N <= 0 || nnz <= 0) return NBLDPC_ERR_INVALID_ARGUMENT;
  const int q = 1 << m;
  for (int i = 0; i < nnz; ++i) {
    if (rows[i] < 0 || rows[i] >= M || cols[i] < 0 || cols[i] >= N) return NBLDPC_ERR_INVALID_ARGUMENT;
    if (coeffs[i] < 1 || coeffs[i] >= q) return NBLDPC_ERR_INVALID_ARGUMENT;
  }
  std::vector<int> ex, lg;
  if (!gf_tables(m, prim_poly, ex, lg)) return NBLDPC_ERR_NOT_PRIMITIVE;
  auto gmul = [&](int a, int b) { return (a && b) ? ex[lg[a] + lg[b]] : 0; };
  auto ginv = [&](int a) { return ex[(q - 1 - lg[a]) % (q - 1)]; };

  // canonical order: sorted by (row, col)
  std::vector<int> order(nnz);
  for (int i = 0; i < nnz; ++i) order[i] = i;
  std::sort(order.begin(), order.end(),
            [&](int a, int b) { return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b]; });
  for (int i = 1; i < nnz; ++i)
    if (rows[order[i]] == rows[order[i - 1]] && cols[order[i]] == cols[order[i - 1]]) return NBLDPC_ERR_UNSUPPORTED;
  std::vector<int> colw(N, 0), roww(M, 0);
  for (int i = 0; i < nnz; ++i) {
    colw[cols[i]]++;
    roww[rows[i]]++;
  }
  // column weights 1..16 (weight 2: the Log-Fourier cluster kernel; others: lf_general.cuh)
  int j_max = 0;
  bool colw2 = true;
  for (int v = 0; v < N; ++v) {
    if (colw[v] < 1 || colw[v] > kMaxColWeight) return NBLDPC_ERR_UNSUPPORTED;
    j_max = std::max(j_max, colw[v]);
    colw2 = colw2 && colw[v] == 2;
  }
  int k_max = 0, k_min = 1 << 30;
  for (int r = 0; r < M; ++r) {
    if (roww[r] < 2) return NBLDPC_ERR_UNSUPPORTED;
    k_max = std::max(k_max, roww[r]);
    k_min = std::min(k_min, roww[r]);
  }
  const int tt = team_threads(m);
  if (k_max * tt > kBigBlock) return NBLDPC_ERR_UNSUPPORTED;
  if ((long long)M * 64 >= (1ll << 22)) return NBLDPC_ERR_UNSUPPORTED;  // edge slots must fit 22 bits

  // internal edge slots: e = c * kpad + j (j-th nonzero of row c in canonical order), kpad the
  // next power of two >= max(4, k_max); the padding slots have var = -1
  int kpad = 4;
  while (kpad < k_max) kpad <<= 1;
  const int E = M * kpad;
  std::vector<EdgeDev> edges(E);
  for (auto& ed : edges) {
    std::memset(&ed, 0, sizeof(ed));
    ed.var = -1;
  }
  std::vector<int> first(N, -1), fill(M, 0);
  for (int n = 0; n < nnz; ++n) {
    const int i = order[n];
    const int r = rows[i];
    const int e = r * kpad + fill[r]++;
    EdgeDev& ed = edges[e];
    ed.var = cols[i];
    ed.h = (uint8_t)coeffs[i];
    ed.hinv = (uint8_t)ginv(coeffs[i]);
    ed.logh = (uint8_t)lg[ed.h];
    // pi_h(e_i): bit j = bit i of h * alpha^j  (M_h^T e_i)
    for (int bi = 0; bi < m; ++bi) {
      int img = 0, imginv = 0;
      for (int bj = 0; bj < m; ++bj) {
        img |= ((gmul(ed.h, 1 << bj) >> bi) & 1) << bj;
        imginv |= ((gmul(ed.hinv, 1 << bj) >> bi) & 1) << bj;
      }
      ed.pib[bi] = (uint8_t)img;
      ed.pinvb[bi] = (uint8_t)imginv;
    }
    const int v = cols[i];
    if (!colw2) {  // no partner edge: the general kernel walks the variable's edge list
      ed.partner = e;
      ed.is_a = first[v] < 0 ? 1 : 0;
      if (first[v] < 0) first[v] = e;
    } else if (first[v] < 0) {
      first[v] = e;
      ed.is_a = 1;
    } else {
      EdgeDev& ea = edges[first[v]];
      ed.partner = first[v];
      ed.plogh = ea.logh;
      ea.partner = e;
      ea.plogh = ed.logh;
    }
  }
  if (colw2 && !getenv("NBLDPC_FIRST_EDGE_DECIDES")) assign_decision_owners(edges, E, tt, kpad);
  // q = 256: the split decision's kinds (kind_a), beside the deciding edges (is_a) of the whole decision
  if (colw2 && tt == 16) orient_uniform_kinds(edges, E);
  std::vector<uint8_t> gexp(2 * (q - 1) + 1), glog(q, 0);
  for (size_t i = 0; i < gexp.size(); ++i) gexp[i] = (uint8_t)ex[i];
  for (int x = 1; x < q; ++x) glog[x] = (uint8_t)lg[x];

  nbldpc_code_s* c = new (std::nothrow) nbldpc_code_s();
  if (!c) return NBLDPC_ERR_OUT_OF_MEMORY;
  cudaGetDevice(&c->device);
  c->m = m;
  c->q = q;
  c->M = M;
  c->N = N;
  c->E = E;
  c->k_max = k_max;
  c->kpad = kpad;
  c->con_stride = (int)align_up((size_t)E, 16);
  c->row_regular = k_min == k_max && kpad == k_max;
  c->poly = prim_poly;
  c->j_max = j_max;
  c->colw2 = colw2;
  c->nnz = nnz;
  auto bail = [&](cudaError_t e) {
    cudaGetLastError();
    nbldpc_destroy(c);
    return cuda_status(e);
  };
  if (cudaError_t e = cudaMalloc(&c->edges_d, sizeof(EdgeDev) * E)) return bail(e);
  if (cudaError_t e = cudaMalloc(&c->gf_exp_d, gexp.size())) return bail(e);
  if (cudaError_t e = cudaMalloc(&c->gf_log_d, q)) return bail(e);
  if (cudaError_t e = cudaMemcpy(c->edges_d, edges.data(), sizeof(EdgeDev) * E, cudaMemcpyHostToDevice)) return bail(e);
  if (cudaError_t e = cudaMemcpy(c->gf_exp_d, gexp.data(), gexp.size(), cudaMemcpyHostToDevice)) return bail(e);
  if (cudaError_t e = cudaMemcpy(c->gf_log_d, glog.data(), q, cudaMemcpyHostToDevice)) return bail(e);
  {
    // variable -> its edges in canonical order (internal slots)
    std::vector<int32_t> vptr(N + 1, 0), vedges(nnz);
    for (int v = 0; v < N; ++v) vptr[v + 1] = vptr[v] + colw[v];
    std::vector<int32_t> pos(vptr.begin(), vptr.end() - 1);
    for (int e = 0; e < E; ++e)
      if (edges[e].var >= 0) vedges[pos[edges[e].var]++] = e;
    if (cudaError_t e = cudaMalloc(&c->v_ptr_d, sizeof(int32_t) * (N + 1))) return bail(e);
    if (cudaError_t e = cudaMalloc(&c->v_edges_d, sizeof(int32_t) * nnz)) return bail(e);
    if (cudaError_t e = cudaMemcpy(c->v_ptr_d, vptr.data(), sizeof(int32_t) * (N + 1), cudaMemcpyHostToDevice)) return bail(e);
    if (cudaError_t e = cudaMemcpy(c->v_edges_d, vedges.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice)) return bail(e);
  }
  {
    // pi_h^-1(alpha^i) = pi_{h^-1}(alpha^i): bit j = bit i of h^-1 * alpha^j
    std::vector<uint64_t> pt(q, 0);
    for (int h = 1; h < q; ++h) {
      const int hi = ginv(h);
      uint64_t v = 0;
      for (int bi = 0; bi < m; ++bi) {
        int img = 0;
        for (int bj = 0; bj < m; ++bj) img |= ((gmul(hi, 1 << bj) >> bi) & 1) << bj;
        v |= (uint64_t)img << (8 * bi);
      }
      pt[h] = v;
    }
    if (cudaError_t e = cudaMalloc(&c->pinv_tab_d, sizeof(uint64_t) * q)) return bail(e);
    if (cudaError_t e = cudaMemcpy(c->pinv_tab_d, pt.data(), sizeof(uint64_t) * q, cudaMemcpyHostToDevice)) return bail(e);
  }
  // launch geometry: teams of TT threads per edge, k_max teams per check, <= 256 threads per CTA
  c->TT = tt;
  {
    // threads per check, padded so that a check never straddles a warp (<= 32: a power of two)
    // or fills whole warps (> 32: a multiple of 32, synchronised by a named barrier)
    int tpc = k_max * tt;
    if (tpc <= 32) {
      int p2 = 1;
      while (p2 < tpc) p2 <<= 1;
      tpc = p2;
    } else {
      tpc = (int)align_up((size_t)tpc, 32);
    }
    c->TPC = tpc;
  }
  if (c->TPC > kBigBlock) {
    nbldpc_destroy(c);
    return NBLDPC_ERR_UNSUPPORTED;
  }
  c->big = c->TPC > 256 ? 1 : 0;
  c->CPC = std::min(std::max(1, 256 / c->TPC), M);
  c->groups = (M + c->CPC - 1) / c->CPC;
  c->block = (int)align_up((size_t)c->CPC * c->TPC, 32);
  c->smem = ((size_t)(c->block / tt) * team_floats(m) + (size_t)c->CPC * q) * sizeof(float);
  {
    // persistent kernel: threads per check = next power of two >= k_max * TT
    // one team per edge slot of a check (KT = kpad teams), so that a group's message rows are the
    // contiguous edge slots of its checks
    int tpc = kpad * tt;
    if (tpc > kBigBlock) {
      nbldpc_destroy(c);
      return NBLDPC_ERR_UNSUPPORTED;
    }
    c->p_tpc = tpc;
    c->p_big = tpc > 256 ? 1 : 0;
    c->p_cpc = std::min(std::max(1, 256 / tpc), M);
    c->p_groups = (M + c->p_cpc - 1) / c->p_cpc;
    c->p_block = (int)align_up((size_t)c->p_cpc * tpc, 32);
    // cluster size: the largest divisor of the chunk count that is <= 8 (portable clusters)
    // small clusters measured fastest (fewer CTAs per barrier, more chunks per CTA per iteration):
    // 2 CTAs per frame when the chunk count is even
    // (measured: C2/C3/C4 fastest at 2, the one-thread-per-edge q <= 16 path at 4)
    int cs = c->p_groups % 2 == 0 ? 2 : 1;
    if (tt == 1 && c->p_groups % 4 == 0) cs = 4;
    if (const char* env = getenv("NBLDPC_CLUSTER_SIZE")) {  // tuning override (a divisor of the chunk count)
      const int v = atoi(env);
      if (v >= 1 && v <= 16 && c->p_groups % v == 0) cs = v;
    }
    // full CTAs (NTHR threads of checks of kpad teams): the geometry is a compile-time constant
    if (c->p_block == (tpc > 256 ? 512 : 256) && c->p_cpc * tpc == c->p_block && !getenv("NBLDPC_NO_KP") &&
        persist_kp_ptr(m, kpad) != nullptr)
      c->p_kp = kpad;
    const int kt = tpc / tt;
    // each CTA keeps the 8-byte edge records of its ceil(G / cs) chunks in shared memory, so long codes
    // need larger clusters: raise cs (2, 4, 8, then the non-portable 16) until the CTA fits in 227 KB
    // (the kernel balances chunk counts that cs does not divide); beyond that the code runs the
    // general kernel (cluster_ok = false)
    auto smem_for = [&](int csz) {
      const size_t recs = (size_t)((c->p_groups + csz - 1) / csz) * c->p_cpc * kt;
      return ((size_t)(c->p_block / tt) * persist_team_words(m) + (size_t)c->p_cpc * q) * sizeof(float) +
             (size_t)q * sizeof(uint64_t) + recs * sizeof(nb::EdgeRec) + align_up(3 * (size_t)q, 16) +
             // q = 256 (tt = 16): the split decision's staged W_e rows (WE in lf_cluster.cuh), [NS][teams][q]
             (tt == 16 ? 16 + (size_t)nb::CCfg<8>::NS * (size_t)(c->p_block / tt) * (q + 16) * sizeof(float) : 0);
    };
    while (smem_for(cs) > 227 * 1024 && cs < 16 && cs < c->p_groups) cs *= 2;
    c->p_cs = cs;
    c->p_recs = ((c->p_groups + cs - 1) / cs) * c->p_cpc * kt;
    c->p_smem = smem_for(cs);
    c->p_smem_pmf = c->p_smem;
    if (tt == 1 && q >= 4)  // PSTAGE in lf_cluster.cuh: [NS][teams][q] floats, 16-byte aligned after the GF tables
      c->p_smem_pmf += 16 + (size_t)nb::CCfg<1>::NS * (size_t)(c->p_block / tt) * q * sizeof(float);
    if (c->p_smem > 227 * 1024) c->cluster_ok = false;
  }
  if (cudaError_t e = ensure_smem_attr(c)) return bail(e);
  if (c->cluster_ok) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(c->p_cs * 64));
    cfg.blockDim = dim3((unsigned)c->p_block);
    cfg.dynamicSmemBytes = c->p_smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)c->p_cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    void* fn = c->p_kp ? persist_kp_ptr(m, c->p_kp) : persist_kernel_ptr(m, c->p_big);
    if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      c->cluster_ok = false;  // no cluster of this shape fits: the general kernel decodes this code
    } else {
      c->p_ncl = ncl;
    }
  }
  int bps = 0;
  if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, pass_kernel_ptr(m, c->big, 0), c->block, c->smem))
    return bail(e);
  if (bps < 1) {
    nbldpc_destroy(c);
    return NBLDPC_ERR_UNSUPPORTED;
  }
  c->blocks_per_sm = bps;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device);
  *out = c;
  return NBLDPC_OK;
}

void nbldpc_destroy(nbldpc_code_t c) {
  if (!c) return;
  free_workspace(c->ws);
  cudaFree(c->edges_d);
  cudaFree(c->gf_exp_d);
  cudaFree(c->gf_log_d);
  cudaFree(c->pinv_tab_d);
  cudaFree(c->v_ptr_d);
  cudaFree(c->v_edges_d);
  delete c;
}

nbldpc_status_t nbldpc_code_info(nbldpc_code_t c, int* m, int* M, int* N, int* E, int* k_max) {
  if (!c) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (m) *m = c->m;
  if (M) *M = c->M;
  if (N) *N = c->N;
  if (E) *E = c->nnz;
  if (k_max) *k_max = c->k_max;
  return NBLDPC_OK;
}

size_t nbldpc_slot_bytes(nbldpc_code_t c) { return c ? slot_bytes_of(c) : 0; }

size_t nbldpc_workspace_bytes(nbldpc_code_t c, int frames) {
  if (!c || frames < 1) return 0;
  // the default path: the cluster kernel keeps one slot per resident cluster (decode_impl);
  // codes with a column weight != 2 run the general kernel (two message sets + estimates per slot)
  if (!c->colw2 || !c->cluster_ok) return 0;  // allocated per call by decode_general, sized by occupancy
  return layout_workspace(c, std::min(c->p_ncl, frames), nullptr, nullptr);
}

nbldpc_status_t nbldpc_last_decode_launches(nbldpc_code_t c, long long* launches) {
  if (!c || !launches) return NBLDPC_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(c->mu);
  Workspace& w = c->ws;
  if (!w.base) {
    *launches = 0;
    return NBLDPC_OK;
  }
  if (!w.last_graph) {  // host loop or persistent kernel
    *launches = w.last_host_launches;
    return NBLDPC_OK;
  }
  NB_TRY(cudaStreamSynchronize(w.last_stream));
  int32_t it = 0;
  NB_TRY(cudaMemcpy(&it, w.dev.glob + 2, sizeof(int32_t), cudaMemcpyDeviceToHost));
  *launches = 1 + (long long)it * (kPassesPerGraphIter + 1);
  return NBLDPC_OK;
}

nbldpc_status_t nbldpc_decode_ex(nbldpc_code_t c, const float* llr, int frames, int max_iters, uint8_t* hard,
                                 uint8_t* ok, int32_t* iters, void* stream, const nbldpc_decode_opts_t* opts) {
  if (!c || frames < 1 || max_iters < 1) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (!is_device_ptr(llr) || !is_device_ptr(hard) || !is_device_ptr(ok) || !is_device_ptr(iters))
    return NBLDPC_ERR_INVALID_ARGUMENT;
  nbldpc_decode_opts_t o;
  if (!normalise_opts(opts, &o)) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (o.workspace)  // the caller's workspace: nothing of the handle is written, no lock (concurrent streams)
    return decode_impl(c, llr, frames, max_iters, hard, ok, iters, static_cast<cudaStream_t>(stream), &o);
  std::lock_guard<std::mutex> lk(c->mu);
  return decode_impl(c, llr, frames, max_iters, hard, ok, iters, static_cast<cudaStream_t>(stream), &o);
}

nbldpc_status_t nbldpc_decode_pmf(nbldpc_code_t c, const float* pmf, int frames, int max_iters, uint8_t* hard,
                                  uint8_t* ok, int32_t* iters, void* stream, const nbldpc_decode_opts_t* opts) {
  if (!c || frames < 1 || max_iters < 1) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (!is_device_ptr(pmf) || !is_device_ptr(hard) || !is_device_ptr(ok) || !is_device_ptr(iters))
    return NBLDPC_ERR_INVALID_ARGUMENT;
  if (((uintptr_t)pmf & 15) != 0) return NBLDPC_ERR_INVALID_ARGUMENT;  // rows are read as float4
  std::lock_guard<std::mutex> lk(c->mu);
  return decode_impl(c, nullptr, frames, max_iters, hard, ok, iters, static_cast<cudaStream_t>(stream), opts, pmf);
}

nbldpc_status_t nbldpc_decode(nbldpc_code_t c, const float* llr, int frames, int max_iters, uint8_t* hard,
                              uint8_t* ok, int32_t* iters, void* stream) {
  return nbldpc_decode_ex(c, llr, frames, max_iters, hard, ok, iters, stream, nullptr);
}

}  // extern "C"

namespace {
// nbldpc_decode_host / nbldpc_decode_pmf_host: in_host is float32 [frames][N*m] LLRs or, with is_pmf,
// [frames][N][q] symbol pmfs
nbldpc_status_t decode_host_impl(nbldpc_code_t c, const float* llr_host, int is_pmf, int frames, int max_iters,
                                 uint8_t* hard_host, uint8_t* ok_host, int32_t* iters_host, void* stream,
                                 const nbldpc_decode_opts_t* opts) {
  if (!c || frames < 1 || max_iters < 1 || !llr_host || !hard_host || !ok_host || !iters_host)
    return NBLDPC_ERR_INVALID_ARGUMENT;
  if (is_device_ptr(llr_host) || is_device_ptr(hard_host)) return NBLDPC_ERR_INVALID_ARGUMENT;
  nbldpc_decode_opts_t onorm;
  if (!normalise_opts(opts, &onorm)) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (onorm.workspace) return NBLDPC_ERR_UNSUPPORTED;  // the host entry points stage through the handle
  opts = &onorm;
  std::lock_guard<std::mutex> lk(c->mu);
  NB_TRY(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Workspace& w = c->ws;
  const size_t row = (size_t)c->N * (is_pmf ? c->q : c->m);  // floats per frame
  const size_t llr_bytes = (size_t)frames * row * sizeof(float);
  const size_t out_bytes = align_up((size_t)frames * c->N, 256) + align_up(frames, 256) + (size_t)frames * 4;
  {  // stream-ordered growth of the device staging buffers
    nbldpc_status_t rs = grow_buffer(w, &w.llr_stage, &w.llr_stage_bytes, llr_bytes, st);
    if (rs == NBLDPC_OK) rs = grow_buffer(w, &w.out_stage, &w.out_stage_bytes, out_bytes, st);
    if (rs != NBLDPC_OK) return rs;
  }
  uint8_t* hard_d = w.out_stage;
  uint8_t* ok_d = hard_d + align_up((size_t)frames * c->N, 256);
  int32_t* it_d = reinterpret_cast<int32_t*>(ok_d + align_up(frames, 256));
  nbldpc_decode_opts_t o{};
  o.struct_size = sizeof(o);
  if (opts) {
    o = *opts;
    o.struct_size = sizeof(o);
    o.soft_out = nullptr;
    o.events_out = nullptr;
  }
  // The cluster path overlaps the host-to-device copy with the decode: the LLRs go over in chunks on
  // a copy stream, each followed by a stream write of its arrival flag (no SM needed, so it cannot
  // wait behind the persistent kernel), and the kernel starts after the first chunk; a cluster that
  // takes a frame of a later chunk waits for that chunk's flag (ld.acquire.gpu).
  using write_value_fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static write_value_fn write_value = nullptr;
  static std::once_flag write_value_once;  // handles on other threads probe concurrently
  std::call_once(write_value_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      write_value = reinterpret_cast<write_value_fn>(fn);
    cudaGetLastError();
  });
  const bool cluster_path = c->colw2 && o.algorithm == NBLDPC_ALG_LOG_FOURIER && o.vn_algorithm == NBLDPC_VN_SEPARABLE &&
                            !o.symbol_post_out && !o.symbol_map_out;
  const int chunk = std::max(c->p_ncl, (frames + kMaxChunks - 1) / kMaxChunks);
  const int nchunk = (frames + chunk - 1) / chunk;
  if (cluster_path && write_value && nchunk >= 2 && !getenv("NBLDPC_NO_OVERLAP")) {
    if (!w.copy_stream) NB_TRY(cudaStreamCreateWithFlags(&w.copy_stream, cudaStreamNonBlocking));
    if (!w.ev_start) NB_TRY(cudaEventCreateWithFlags(&w.ev_start, cudaEventDisableTiming));
    if (!w.ev_first) NB_TRY(cudaEventCreateWithFlags(&w.ev_first, cudaEventDisableTiming));
    if (!w.chunk_flags) NB_TRY(cudaMalloc(&w.chunk_flags, kMaxChunks * sizeof(int32_t)));
    NB_TRY(cudaEventRecord(w.ev_start, st));  // the previous work on st (readers of llr_stage) is done first
    NB_TRY(cudaStreamWaitEvent(w.copy_stream, w.ev_start, 0));
    NB_TRY(cudaMemsetAsync(w.chunk_flags, 0, kMaxChunks * sizeof(int32_t), w.copy_stream));
    for (int k = 0; k < nchunk; ++k) {
      const int f0 = k * chunk, nf = std::min(chunk, frames - f0);
      NB_TRY(cudaMemcpyAsync(w.llr_stage + (size_t)f0 * row, llr_host + (size_t)f0 * row, (size_t)nf * row * sizeof(float),
                             cudaMemcpyHostToDevice, w.copy_stream));
      if (write_value(reinterpret_cast<CUstream>(w.copy_stream), reinterpret_cast<CUdeviceptr>(w.chunk_flags + k), 1,
                      CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        return NBLDPC_ERR_CUDA;
      if (k == 0) NB_TRY(cudaEventRecord(w.ev_first, w.copy_stream));
    }
    NB_TRY(cudaStreamWaitEvent(st, w.ev_first, 0));
    nbldpc_status_t rs = decode_impl(c, is_pmf ? nullptr : w.llr_stage, frames, max_iters, hard_d, ok_d, it_d, st, &o,
                                     is_pmf ? w.llr_stage : nullptr, w.chunk_flags, chunk);
    if (rs != NBLDPC_OK) {
      cudaStreamSynchronize(w.copy_stream);
      return rs;
    }
  } else {
    NB_TRY(cudaMemcpyAsync(w.llr_stage, llr_host, llr_bytes, cudaMemcpyHostToDevice, st));
    nbldpc_status_t rs = decode_impl(c, is_pmf ? nullptr : w.llr_stage, frames, max_iters, hard_d, ok_d, it_d, st, &o,
                                     is_pmf ? w.llr_stage : nullptr);
    if (rs != NBLDPC_OK) return rs;
  }
  NB_TRY(cudaMemcpyAsync(hard_host, hard_d, (size_t)frames * c->N, cudaMemcpyDeviceToHost, st));
  NB_TRY(cudaMemcpyAsync(ok_host, ok_d, frames, cudaMemcpyDeviceToHost, st));
  NB_TRY(cudaMemcpyAsync(iters_host, it_d, (size_t)frames * 4, cudaMemcpyDeviceToHost, st));
  NB_TRY(cudaStreamSynchronize(st));
  return NBLDPC_OK;
}
}  // namespace

extern "C" {

nbldpc_status_t nbldpc_decode_host(nbldpc_code_t c, const float* llr_host, int frames, int max_iters,
                                   uint8_t* hard_host, uint8_t* ok_host, int32_t* iters_host, void* stream,
                                   const nbldpc_decode_opts_t* opts) {
  return decode_host_impl(c, llr_host, 0, frames, max_iters, hard_host, ok_host, iters_host, stream, opts);
}

nbldpc_status_t nbldpc_decode_pmf_host(nbldpc_code_t c, const float* pmf_host, int frames, int max_iters,
                                       uint8_t* hard_host, uint8_t* ok_host, int32_t* iters_host, void* stream,
                                       const nbldpc_decode_opts_t* opts) {
  return decode_host_impl(c, pmf_host, 1, frames, max_iters, hard_host, ok_host, iters_host, stream, opts);
}

}  // extern "C"

namespace {
// pmf != NULL: nbldpc_step_pmf (the cluster kernel's symbol-pmf variant; llr unused)
nbldpc_status_t step_impl(nbldpc_code_t c, const float* llr, const float* pmf, int frames, int iter, const float* w_in,
                          float* w_out, float* u_out, uint8_t* hard, float* soft, int vn_algorithm, void* stream) {
  if (!c || frames < 1 || iter < 0 || !is_device_ptr(pmf ? pmf : llr) || !is_device_ptr(w_out))
    return NBLDPC_ERR_INVALID_ARGUMENT;
  if (pmf && vn_algorithm != 0) return NBLDPC_ERR_UNSUPPORTED;  // the pass kernel keeps p only from l = 0 on
  if (pmf && ((uintptr_t)pmf & 15)) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (iter >= 1 && (!is_device_ptr(w_in) || !is_device_ptr(hard))) return NBLDPC_ERR_INVALID_ARGUMENT;
  if ((u_out && !is_device_ptr(u_out)) || (soft && !is_device_ptr(soft))) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (vn_algorithm != 0 && vn_algorithm != 1) return NBLDPC_ERR_INVALID_ARGUMENT;
  if (!c->row_regular || !c->colw2) return NBLDPC_ERR_UNSUPPORTED;  // internal slots == canonical order only then
  if (vn_algorithm == 0 && !c->cluster_ok) return NBLDPC_ERR_UNSUPPORTED;
  std::lock_guard<std::mutex> lk(c->mu);
  NB_TRY(cudaSetDevice(c->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  nbldpc_status_t rs = ensure_workspace(c, frames, st);
  if (rs != NBLDPC_OK) return rs;
  Workspace& w = c->ws;
  const size_t msg = (size_t)frames * c->E * c->q * sizeof(float);
  CallDev call{};
  call.llr = llr;
  if (pmf) {
    rs = grow_buffer(w, &w.p0buf, &w.p0buf_bytes, (size_t)frames * c->N * c->q * sizeof(float), st);
    if (rs != NBLDPC_OK) return rs;
    call.pmf = pmf;
    call.p0buf = w.p0buf;
  }
  call.frames = frames;
  call.max_iters = 1 << 30;
  call.mode = 0;
  call.early_stop = 1;
  call.want_soft = soft != nullptr;
  nb::nb_step_setup_kernel<<<(frames + 255) / 256, 256, 0, st>>>(w.dev, call, iter);
  NB_TRY(cudaGetLastError());
  if (!pmf) {
    nb::nb_tanh_kernel<<<256, 256, 0, st>>>(llr, w.dev.Tt, (size_t)frames * c->N, c->m);
    NB_TRY(cudaGetLastError());
  }
  // the direct pass kernel selects buffers by iteration parity, the persistent one by epoch (0)
  const int in_buf = vn_algorithm ? (iter & 1) : 0;
  float* wcur = w.dev.W + (size_t)in_buf * frames * c->E * c->q;
  float* wnxt = w.dev.W + (size_t)(in_buf ^ 1) * frames * c->E * c->q;
  if (iter >= 1) {
    if (vn_algorithm) {
      NB_TRY(cudaMemcpyAsync(wcur, w_in, msg, cudaMemcpyDeviceToDevice, st));
    } else {  // the cluster kernel keeps messages in its chunk-swizzled order (linear unless soft outputs)
      NB_TRY(launch_layout(c, w_in, wcur, frames, 1, soft == nullptr && c->m >= 7, st));
    }
  }
  if (vn_algorithm) {
    PassParams P = make_params(c, 1, u_out);
    NB_TRY(launch_pass(c, P, 1, st, soft != nullptr));
  } else {
    nb::ClusterParams PP = make_cparams(c, 1, iter, u_out);
    NB_TRY(launch_cluster(c, PP, std::min(frames, c->p_ncl), st, pmf != nullptr, 0, 0, soft != nullptr));
  }
  if (vn_algorithm) {
    NB_TRY(cudaMemcpyAsync(w_out, wnxt, msg, cudaMemcpyDeviceToDevice, st));
  } else {
    NB_TRY(launch_layout(c, wnxt, w_out, frames, 0, soft == nullptr && c->m >= 7, st));
  }
  if (iter >= 1) {
    NB_TRY(cudaMemcpyAsync(hard, w.dev.xhat, (size_t)frames * c->N, cudaMemcpyDeviceToDevice, st));
    if (soft)
      NB_TRY(cudaMemcpyAsync(soft, w.dev.soft, (size_t)frames * c->N * c->m * sizeof(float), cudaMemcpyDeviceToDevice,
                             st));
  }
  return mark_done(w, st);
}
}  // namespace

extern "C" {

nbldpc_status_t nbldpc_step(nbldpc_code_t c, const float* llr, int frames, int iter, const float* w_in, float* w_out,
                            float* u_out, uint8_t* hard, float* soft, int vn_algorithm, void* stream) {
  return step_impl(c, llr, nullptr, frames, iter, w_in, w_out, u_out, hard, soft, vn_algorithm, stream);
}

nbldpc_status_t nbldpc_step_pmf(nbldpc_code_t c, const float* pmf, int frames, int iter, const float* w_in,
                                float* w_out, float* u_out, uint8_t* hard, float* soft, void* stream) {
  return step_impl(c, nullptr, pmf, frames, iter, w_in, w_out, u_out, hard, soft, 0, stream);
}

}  // extern "C"
