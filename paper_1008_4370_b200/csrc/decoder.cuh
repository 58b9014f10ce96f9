// decoder.cuh -- device side of the B200 Log-Fourier SP decoder (arXiv:1008.4370).
//
// One kernel, nb_pass_kernel<m>, advances every resident frame slot by one
// flooding iteration.  It is check-centric and fuses, per check c and edge
// e = (c, v) with partner edge e' = (c', v):
//   VARIABLE TO CHECK   U_e = normalise(P_v^0 (*) W_e')    [signed XOR-convolution]
//   TENTATIVE DECISION  at the variable's first edge only: M_v at 0, alpha^i
//   CHECK TO VARIABLE   W_e(next) = TOT_c(pi^-1 z) - U_e(z), TOT_c = sum_j U_j(pi_j .)
// and, in the last CTA that finishes a slot, the syndrome (PAPER.md:427 or
// :521-526), early termination and the refill of the slot
// with the next pending frame.
//
// Work decomposition: CTA (g, y) owns check group g and the
// frame slots y, y+Y, y+2Y, ...; it keeps its edge table in registers and walks
// its slots one after another, prefetching the next slot's messages into a
// second shared-memory buffer with cp.async while it computes the current one.
//
// Numerics: messages live in HBM/L2 as float32 whose
// magnitude is -log2|x| (>= 0) and whose IEEE sign bit is the message sign
// (the paper's Gamma, in base 2).  The signed log-convolution
// Gamma(sum_y Gamma^-1(L1(y) + L2(z^y))) is evaluated through the exact identity
// Gamma^-1(a + b) = Gamma^-1(a) Gamma^-1(b): ex2 on the inputs,
// an FFMA2 XOR-convolution, lg2 on the outputs.  The channel spectrum is the
// closed form P_v^0(z) = prod_{i in z} tanh(L_{v,i}/2) (= WHT of the factorised
// prior).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace nb {

constexpr float kFloor = 200.0f;  // -log2 of a "zero" entry; ex2(-200) flushes to 0 in float32
constexpr uint32_t kSign = 0x80000000u;
constexpr int kMaxSlotsPerCta = 64;

struct EdgeDev {      // 32 bytes, one per internal edge slot c*kpad + j (var < 0: padding)
  int32_t partner;    // internal index of the variable's other edge
  int32_t var;        // variable index v
  uint8_t h, hinv;    // h_cv and its inverse
  uint8_t is_a;       // 1 if e is v's first edge (owner of v's tentative decision)
  uint8_t logh;       // log_alpha h_cv
  uint8_t pib[8];     // pi_h(e_i)    = H_cv alpha^i     (i < m), bit j = bit i of h*alpha^j
  uint8_t pinvb[8];   // pi_h^-1(e_i) = H_cv^-1 alpha^i  (= pi_{h^-1}(e_i))
  uint8_t plogh;      // log_alpha of the partner edge's coefficient
  uint8_t kind_a;     // q = 256 split decision: 1 if e evaluates the high half (one of v's two edges; the host
                      // orients them so that both edge slots of a warp are of the same kind)
  uint8_t pad[2];
};
static_assert(sizeof(EdgeDev) == 32, "EdgeDev layout");

struct CodeDev {
  int m, M, N, E, k_max;      // E = M * kpad internal edge slots
  int kpad;                   // edge-slot stride per check: next power of two >= max(4, k_max)
  const EdgeDev* edges;       // [E]
  const uint8_t* gf_exp;      // [2(q-1)+1] alpha^i
  const uint8_t* gf_log;      // [q]
  const uint64_t* pinv_tab;   // [q] byte i of entry h: pi_h^-1(alpha^i) (entry 0 unused)
};

struct CallDev {            // per-call arguments, written on the stream before the pass loop
  const float* llr;
  uint8_t* hard;
  uint8_t* ok;
  int32_t* iters;
  float* soft_out;
  int32_t* events_out;
  int frames, max_iters, mode, early_stop;
  int want_soft;
  int pad[3];
  const float* pmf;   // nbldpc_decode_pmf: [frames][N][q] channel pmf (else NULL)
  float* p0buf;       // nbldpc_decode_pmf: [S][N][q] P_v^0 = WHT(pmf) / sum(pmf) per slot
  float* post_out;    // symbol posterior [frames][N][q] (or NULL), rewritten at every iteration
  uint8_t* map_out;   // symbol-MAP decision [frames][N] (or NULL), idem: the last write is the stopping one
  const int32_t* chunk_flags;  // nbldpc_decode_host: flag c != 0 once frames [c*chunk_frames, ..) are in HBM
  int chunk_frames;
  int pad2;
};

struct WorkDev {
  int S;
  float* W;              // [2][S][E][q] packed messages (ping-pong by iteration parity)
  float* Tt;             // [S][N][8]  tanh(L/2) (m used)
  uint8_t* xhat;         // [S][N]
  float* soft;           // [S][N][m]
  uint8_t* con;          // [S][con_stride] per-edge syndrome contribution h_cv xhat_v (or paper bits)
  int con_stride;        // round_up(E, 16)
  int32_t* slot_frame;   // [S] frame index or -1
  int32_t* slot_iter;    // [S] CHECK-TO-VARIABLE steps completed (l)
  int32_t* slot_events;  // [S]
  int32_t* slot_counter; // [S] CTAs finished in the current pass
  int32_t* slot_epoch;   // [S] passes completed (persistent kernel)
  int32_t* glob;         // [0] next frame, [1] active slots, [2] WHILE-body iterations
  CallDev* call;
};

struct PassParams {
  CodeDev code;
  WorkDev ws;
  int groups;           // G: check groups (CTAs per slot)
  int slot_lanes;       // Y: CTA (g, y) handles slots y, y+Y, ...
  int checks_per_cta;
  int tpc;              // threads per check: k_max*TT padded to a power of two <= 32 or a multiple of 32
  int step_mode;        // 1: nbldpc_step (no syndrome / finish / refill)
  float* u_out;         // step mode: optional U^(l) dump [S][E][q]
};

template <int MB>
struct Cfg {
  static constexpr int Q = 1 << MB;
  static constexpr int LR = MB < 4 ? MB : 4;   // log2 of outputs per thread
  static constexpr int R = 1 << LR;
  static constexpr int TT = Q / R;             // threads per convolution team
  static constexpr int PAD = (TT > 1 && TT < 8) ? 4 * TT : 0;
  static constexpr int VEC = Q + PAD;          // floats per team vector in smem
  // per team: A (P^0, then T_j) | B[2] (W_e') | D[2] (W_e) | TH[2][8]
  static constexpr int TEAM_FLOATS = 5 * VEC + 16;
};

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2a(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// packed (sign | -log2|x|) -> linear x
__device__ __forceinline__ float to_lin(float p) {
  float v = ex2a(-fabsf(p));
  return __uint_as_float(__float_as_uint(v) | (__float_as_uint(p) & kSign));
}
__device__ __forceinline__ float pack(float mag, uint32_t sign) {
  mag = fminf(fmaxf(mag, 0.0f), kFloor);
  if (mag >= kFloor) sign = 0;  // a zero carries sign 0 (reading R6)
  return __uint_as_float(__float_as_uint(mag) | (sign & kSign));
}

// ---- the tentative decision in fp64 (soft outputs, reading R22)
// M_v(z) = sum_y raw(y) D(z ^ y) at z = 0 and z = alpha^i, raw = P^0 (*) B, computed
// in fp64 from the stored (packed fp32) spectra B = W_e' and D = W_e of the deciding edge.  The fp32
// evaluation is accurate enough for the hard bits (their signs) but not for the posterior
// log-magnitudes ln|M(alpha^i)/M(0)| where P^0 (*) B cancels strongly: the result can be 1e5 times
// more sensitive than its inputs, so even the fp32 rounding of Gamma^-1 (2^-24 relative) moves it by
// 5e-3 (measured at GF(256); tools/soft_bar.py).  Hence Gamma^-1 itself is evaluated in fp64 (lin64)
// and every later operation too.  Used only when soft outputs are requested (decode soft_out,
// nbldpc_step), never on the plain hot path (a separate kernel instantiation).
//
// Gamma^-1 of a packed entry (sign | -log2|x|) in fp64: 2^-mag = 2^-n e^{-g ln 2}, n = floor(mag),
// g = mag - n (exact), e^y by its Taylor series to degree 17 (|y| < ln 2: truncation < 2e-18).
__device__ __forceinline__ double lin64(float p) {
  const float mag = fabsf(p);
  if (!(mag < 1022.0f)) return 0.0;  // below the normal doubles (the oracle's floor is 2^-1075)
  const int n = (int)mag;
  const double y = -((double)mag - (double)n) * 0.6931471805599453094172321;
  constexpr double c[18] = {1.0, 1.0, 1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040, 1.0 / 40320,
                            1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800, 1.0 / 479001600, 1.0 / 6227020800.0,
                            1.0 / 87178291200.0, 1.0 / 1307674368000.0, 1.0 / 20922789888000.0,
                            1.0 / 355687428096000.0};
  double e = c[17];
#pragma unroll
  for (int k = 16; k >= 0; --k) e = fma(e, y, c[k]);
  const double r = e * __hiloint2double((1023 - n) << 20, 0);
  return (__float_as_uint(p) & 0x80000000u) ? -r : r;
}

// Layout: phase A -- lane t of a team of TT = 2^(MB-LR) contiguous lanes holds z = R t + r, r < R;
// bpk / dpk are those R entries of B and D as stored (packed), plin (PMF) the pmf p_v(z).  PMF:
// raw = WHT(p . WHT(B)) / q (a general symbol pmf), else raw = (x)_i (1, t_i) applied to B (the
// separable channel spectrum, th[i] = tanh(L_i / 2)).  Returns the team totals md[0..MB] in every lane;
// lanes of non-deciding teams pass zero spectra.
template <int MB, int LR, bool PMF>
__device__ __noinline__ void decision_f64(const float* bpk, const float* dpk, const float* plin, const float* th,
                                          int t, double* md) {
  constexpr int R = 1 << LR;
  constexpr int TT = 1 << (MB - LR);
  double x[R], d[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    x[r] = lin64(bpk[r]);
    d[r] = lin64(dpk[r]);
  }
  auto wht64 = [&]() {
#pragma unroll
    for (int b = 0; b < LR; ++b)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (!(r & (1 << b))) {
          const double u = x[r], w = x[r | (1 << b)];
          x[r] = u + w;
          x[r | (1 << b)] = u - w;
        }
#pragma unroll
    for (int b = LR; b < MB; ++b) {
      const int off = 1 << (b - LR);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_xor_sync(0xffffffffu, x[r], off);
        x[r] = (t & off) ? o - x[r] : x[r] + o;
      }
    }
  };
  if constexpr (PMF) {
    wht64();
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] *= (double)plin[r];
    wht64();  // q raw: the factor q cancels in every ratio and sign
  } else {
#pragma unroll
    for (int b = 0; b < LR; ++b) {
      const double tb = (double)th[b];
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (!(r & (1 << b))) {
          const double u = x[r], w = x[r | (1 << b)];
          x[r] = fma(tb, w, u);
          x[r | (1 << b)] = fma(tb, u, w);
        }
    }
#pragma unroll
    for (int b = LR; b < MB; ++b) {
      const double tb = (double)th[b];
      const int off = 1 << (b - LR);
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = fma(tb, __shfl_xor_sync(0xffffffffu, x[r], off), x[r]);
    }
  }
#pragma unroll
  for (int b = 0; b <= MB; ++b) md[b] = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    md[0] = fma(x[r], d[r], md[0]);
#pragma unroll
    for (int b = 0; b < LR; ++b) md[b + 1] = fma(x[r], d[r ^ (1 << b)], md[b + 1]);
  }
#pragma unroll
  for (int b = LR; b < MB; ++b) {
    const int off = 1 << (b - LR);
#pragma unroll
    for (int r = 0; r < R; ++r) md[b + 1] = fma(x[r], __shfl_xor_sync(0xffffffffu, d[r], off), md[b + 1]);
  }
  if constexpr (TT > 1) {
#pragma unroll
    for (int off = TT / 2; off >= 1; off >>= 1)
#pragma unroll
      for (int b = 0; b <= MB; ++b) md[b] += __shfl_xor_sync(0xffffffffu, md[b], off);
  }
}

// ln|M(alpha^b) / M(0)| from fp64 totals (a ratio below 2^-126 is reported as ln 2^-126)
__device__ __forceinline__ float soft_ratio(double mb, double m0) {
  const double r = fabs(mb) / fabs(m0);
  return __logf((float)fmax(r, 1.1754944e-38));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// chunk-major smem index of element y (block y/R, 16-byte chunk (y%R)/4): keeps the
// XOR-permuted block reads of a team conflict-free
template <int MB>
__device__ __forceinline__ int cm_idx(int y) {
  using C = Cfg<MB>;
  constexpr int R = C::R, NB = C::TT;
  if constexpr (C::TT > 1) {
    return ((((y & (R - 1)) >> 2) * NB + (y >> C::LR)) << 2) | (y & 3);
  } else {
    return y;
  }
}

// acc(2p, 2p+1) += sum_yl a[yl] (b[2p ^ yl], b[2p ^ yl ^ 1]): the thread's share of
// raw[z] = sum_y a[y] b[z ^ y].  (b[w], b[w^1]) is a natural pair when yl is even and
// the swapped natural pair when yl is odd -- both free operand forms of FFMA2, whose
// scalar operand is broadcast.
template <int R>
__device__ __forceinline__ void conv_block(const float (&a)[R], const float (&b)[R], float2 (&acc)[R / 2]) {
#pragma unroll
  for (int p = 0; p < R / 2; ++p) {
#pragma unroll
    for (int yl = 0; yl < R; ++yl) {
      const int w = (2 * p) ^ yl;
      const float2 bp = (yl & 1) ? make_float2(b[w], b[w - 1]) : make_float2(b[w], b[w + 1]);
      acc[p] = __ffma2_rn(make_float2(a[yl], a[yl]), bp, acc[p]);
    }
  }
}

// One stage of the separable XOR-convolution with P^0 = (x)_i (1, t_i):
// x(z) <- x(z) + t_i x(z ^ e_i) on the bit i of the thread's register index (i < LR), as
// FFMA2 with the broadcast t_i and a natural or swapped pair.
template <int R, int I>
__device__ __forceinline__ void bfly_reg(float (&x)[R], float ti) {
  constexpr int S = 1 << I;
  if constexpr (I == 0) {
#pragma unroll
    for (int p = 0; p < R / 2; ++p) {
      const float2 v = make_float2(x[2 * p], x[2 * p + 1]);
      const float2 r = __ffma2_rn(make_float2(ti, ti), make_float2(v.y, v.x), v);
      x[2 * p] = r.x;
      x[2 * p + 1] = r.y;
    }
  } else {
    float y[R];
#pragma unroll
    for (int p = 0; p < R / 2; ++p) {
      const int lo = 2 * p, pa = lo ^ S;
      const float2 r = __ffma2_rn(make_float2(ti, ti), make_float2(x[pa], x[pa + 1]), make_float2(x[lo], x[lo + 1]));
      y[lo] = r.x;
      y[lo + 1] = r.y;
    }
#pragma unroll
    for (int z = 0; z < R; ++z) x[z] = y[z];
  }
}
template <int R, int I, int LR>
__device__ __forceinline__ void bfly_regs(float (&x)[R], const float* th) {
  if constexpr (I < LR) {
    bfly_reg<R, I>(x, th[I]);
    bfly_regs<R, I + 1, LR>(x, th);
  }
}

// In-place Walsh-Hadamard transform x(z) <- sum_y x(y) (-1)^{z.y} of a vector spread over a team of
// TT = 2^(MB-LR) consecutive lanes holding R = 2^LR entries each (entry t*R + zl in x[zl] of team
// lane t): LR stages in registers, MB - LR across the team by shuffles.  Every lane of the warp
// must call it (full-mask shuffles).
template <int MB, int LR, int R>
__device__ __forceinline__ void wht_team(float (&x)[R], int t) {
#pragma unroll
  for (int b = 0; b < LR; ++b)
#pragma unroll
    for (int zl = 0; zl < R; ++zl)
      if (!(zl & (1 << b))) {
        const float u = x[zl], w = x[zl | (1 << b)];
        x[zl] = u + w;
        x[zl | (1 << b)] = u - w;
      }
#pragma unroll
  for (int b = LR; b < MB; ++b) {
    const int off = 1 << (b - LR);
#pragma unroll
    for (int zl = 0; zl < R; ++zl) {
      const float o = __shfl_xor_sync(0xffffffffu, x[zl], off);
      x[zl] = (t & off) ? o - x[zl] : x[zl] + o;
    }
  }
}

// barrier over the threads of one check: the warp when a check fits in it, else a named barrier
__device__ __forceinline__ void check_sync(int lc, int tpc) {
  if (tpc <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(lc + 1), "r"(tpc) : "memory");
  }
}
__device__ __forceinline__ int atom_add_release_gpu(int* p, int v) {
  int old;
  asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// SOFT = true: soft outputs (the fp64 decision, reading R22) -- a separate instantiation so that the plain
// kernel carries none of its registers (with the call site inline: 12 -> 132 spilled bytes, C2 9% slower)
template <int MB, int MAXB, bool DIRECT, bool PMF = false, bool SOFT = false>
__global__ void __launch_bounds__(MAXB, (MAXB <= 256 ? 2 : 1)) nb_pass_kernel(PassParams P) {
  static_assert(DIRECT || !PMF, "a general channel pmf needs the direct convolution");
  using C = Cfg<MB>;
  constexpr int Q = C::Q, R = C::R, TT = C::TT, LR = C::LR, NB = C::TT;
  extern __shared__ __align__(16) float smem[];
  __shared__ int sh_frame[kMaxSlotsPerCta], sh_iter[kMaxSlotsPerCta], sh_list[kMaxSlotsPerCta];
  __shared__ int sh_nact;

  const CodeDev& cd = P.code;
  const WorkDev& ws = P.ws;
  const int g = blockIdx.x % P.groups;
  const int yl0 = blockIdx.x / P.groups;
  const int Y = P.slot_lanes;
  const int nmy = (ws.S - yl0 + Y - 1) / Y;  // my slots: s = yl0 + i*Y, i < nmy

  // ---- my edge (the same for every slot I process)
  const int TPC = P.tpc;
  const int lc = threadIdx.x / TPC;
  const int c = g * P.checks_per_cta + lc;
  const int j = (threadIdx.x - lc * TPC) / TT;
  const int t = threadIdx.x & (TT - 1);
  const bool cvalid = (lc < P.checks_per_cta) && (c < cd.M) && (j < cd.k_max);
  const int e = c * cd.kpad + j;  // internal edge slot
  EdgeDev ed;
  {
    int4 w0 = make_int4(0, -1, 0, 0), w1 = make_int4(0, 0, 0, 0);
    if (cvalid) {
      const int4* ep = reinterpret_cast<const int4*>(cd.edges + e);
      w0 = __ldg(ep);
      w1 = __ldg(ep + 1);
    }
    *reinterpret_cast<int4*>(&ed) = w0;
    *(reinterpret_cast<int4*>(&ed) + 1) = w1;
  }
  const bool active = cvalid && ed.var >= 0;
  const bool is_a = active && ed.is_a;

  // ---- my slots' states; list of the active ones
  for (int i = threadIdx.x; i < nmy; i += blockDim.x) {
    const int s = yl0 + i * Y;
    sh_frame[i] = ws.slot_frame[s];
    sh_iter[i] = ws.slot_iter[s];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int i = 0; i < nmy; ++i)
      if (sh_frame[i] >= 0) sh_list[n++] = i;
    sh_nact = n;
  }
  __syncthreads();
  const int nact = sh_nact;
  if (nact == 0) return;

  const int lane = threadIdx.x & 31;
  const int slot_target = P.groups * (int)(blockDim.x >> 5);  // warps that process every slot
  const CallDev* call = ws.call;
  const float* llr = call->llr;
  const int max_iters = call->max_iters;
  const int mode = call->mode;
  constexpr bool want_soft = SOFT;  // soft outputs exactly when the host launches a SOFT kernel
  const size_t EQ = (size_t)cd.E * Q;

  // team vectors (offsets computed arithmetically so the compiler keeps shared-space accesses)
  const int team_off = (threadIdx.x / TT) * C::TEAM_FLOATS;
  float* A = smem + team_off;
#define NB_BV(b) (smem + team_off + (1 + (b)) * C::VEC)
#define NB_DV(b) (smem + team_off + (3 + (b)) * C::VEC)
#define NB_TH(b) (smem + team_off + 5 * C::VEC + 8 * (b))
  float* TOT = smem + (blockDim.x / TT) * C::TEAM_FLOATS + lc * Q;

  // issue the asynchronous loads of slot list entry kk into buffer buf
  auto stage = [&](int kk, int buf) {
    if (!active) return;
    const int i = sh_list[kk];
    const int s = yl0 + i * Y;
    const int f = sh_frame[i], ell = sh_iter[i];
    float* th = NB_TH(buf);
    if (!PMF && t == 0) {
      const float* src = ell == 0 ? llr + ((size_t)f * cd.N + ed.var) * MB : ws.Tt + ((size_t)s * cd.N + ed.var) * 8;
#pragma unroll
      for (int b = 0; b < MB; ++b) cp_async4(th + b, src + b);
    }
    if (ell == 0) return;
    const float* Wc = ws.W + ((size_t)(ell & 1) * ws.S + s) * EQ;
    const float* sb = Wc + (size_t)ed.partner * Q + t * R;
    const float* sd = Wc + (size_t)e * Q + t * R;
    if constexpr (R >= 4) {
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4) cp_async16(NB_BV(buf) + cm_idx<MB>(t * R + 4 * c4), sb + 4 * c4);
      if (is_a) {
#pragma unroll
        for (int c4 = 0; c4 < R / 4; ++c4) cp_async16(NB_DV(buf) + cm_idx<MB>(t * R + 4 * c4), sd + 4 * c4);
      }
    } else {
      cp_async8(NB_BV(buf), sb);
      if (is_a) cp_async8(NB_DV(buf), sd);
    }
  };

  stage(0, 0);
  cp_async_commit();
#pragma unroll 1
  for (int kk = 0; kk < nact; ++kk) {
    const int buf = kk & 1;
    if (kk + 1 < nact) stage(kk + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();

    const int si = sh_list[kk];
    const int s = yl0 + si * Y;
    const int f = sh_frame[si];
    const int ell = sh_iter[si];
    const bool do_dec = ell >= 1;
    const bool do_cn = P.step_mode || ell < max_iters;
    float* B = NB_BV(buf);
    float* D = NB_DV(buf);

    // ---- channel terms t_i = tanh(L_{v,i}/2): computed at l = 0, cached per slot after
    float th[MB];
#pragma unroll
    for (int b = 0; b < MB; ++b) th[b] = (active && !PMF) ? NB_TH(buf)[b] : 0.0f;
    if (!PMF && ell == 0 && active) {
#pragma unroll
      for (int b = 0; b < MB; ++b) th[b] = tanhf(0.5f * th[b]);
      if (is_a && t == 0) {
#pragma unroll
        for (int b = 0; b < MB; ++b) ws.Tt[((size_t)s * cd.N + ed.var) * 8 + b] = th[b];
      }
    }
    // P_v^0(z) for the thread's block z = t*R + zl (closed form)
    float p0[R];
    if constexpr (PMF) {
      // general pmf: at l = 0 the row is scaled to a probability vector p,
      // kept per slot (p0buf) for the later passes, and P^0 = WHT(p) is the initial message;
      // at l >= 1 p0 holds p (the variable node works in the probability domain, below)
      const float* src = ell == 0 ? call->pmf + ((size_t)f * cd.N + (active ? ed.var : 0)) * Q
                                  : call->p0buf + ((size_t)s * cd.N + (active ? ed.var : 0)) * Q;
      if constexpr (R >= 4) {
#pragma unroll
        for (int c4 = 0; c4 < R / 4; ++c4) {
          const float4 v = active ? __ldcg(reinterpret_cast<const float4*>(src + t * R) + c4) : make_float4(0, 0, 0, 0);
          p0[4 * c4] = v.x; p0[4 * c4 + 1] = v.y; p0[4 * c4 + 2] = v.z; p0[4 * c4 + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int zl = 0; zl < R; ++zl) p0[zl] = active ? __ldcg(src + t * R + zl) : 0.0f;
      }
      if (ell == 0) {
        float tot = 0.0f;
#pragma unroll
        for (int zl = 0; zl < R; ++zl) tot += p0[zl];
        if constexpr (TT > 1) {
#pragma unroll
          for (int off = TT / 2; off >= 1; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
        }
        const float inv = tot > 0.0f ? 1.0f / tot : 0.0f;  // degenerate row: all zero -> event below
#pragma unroll
        for (int zl = 0; zl < R; ++zl) p0[zl] *= inv;
        if (is_a) {
          float* dst = call->p0buf + ((size_t)s * cd.N + ed.var) * Q + t * R;
#pragma unroll
          for (int zl = 0; zl < R; ++zl) dst[zl] = p0[zl];
        }
        wht_team<MB, LR, R>(p0, t);
      }
    } else {
      float hi = 1.0f;
#pragma unroll
      for (int b = LR; b < MB; ++b)
        if ((t >> (b - LR)) & 1) hi *= th[b];
      p0[0] = hi;
#pragma unroll
      for (int b = 0; b < LR; ++b)
#pragma unroll
        for (int jj = 0; jj < (1 << b); ++jj) p0[(1 << b) + jj] = p0[jj] * th[b];
    }

    // ---- VARIABLE TO CHECK: raw = P^0 (*) W_e'  (at l = 0, U = Lambda^0: INITIALIZATION)
    float raw[R];
    float dreg[TT == 1 ? Q : 1];  // W_e linear for the decision (register path)
    if (ell == 0) {
#pragma unroll
      for (int zl = 0; zl < R; ++zl) raw[zl] = p0[zl];
    } else if constexpr (TT == 1) {
      float b[Q];
#pragma unroll
      for (int y = 0; y < Q; ++y) b[y] = active ? to_lin(B[y]) : 0.0f;
      if (is_a) {
#pragma unroll
        for (int y = 0; y < Q; ++y) {
          dreg[y] = to_lin(D[y]);
          D[y] = dreg[y];  // linear copy for the paper-mode points
        }
      }
      if constexpr (PMF) {
        // raw = P^0 (*) W_e' = WHT(p . IWHT(W_e')) up to the factor q (XOR-convolution theorem;
        // 2 m q butterfly operations instead of q^2 FMAs -- the normalisation removes q)
        wht_team<MB, LR, R>(b, t);
#pragma unroll
        for (int zl = 0; zl < R; ++zl) b[zl] *= p0[zl];
        wht_team<MB, LR, R>(b, t);
#pragma unroll
        for (int zl = 0; zl < R; ++zl) raw[zl] = b[zl];
      } else if constexpr (DIRECT) {
        float2 acc[R / 2];
#pragma unroll
        for (int p = 0; p < R / 2; ++p) acc[p] = make_float2(0.0f, 0.0f);
        conv_block<R>(p0, b, acc);
#pragma unroll
        for (int p = 0; p < R / 2; ++p) { raw[2 * p] = acc[p].x; raw[2 * p + 1] = acc[p].y; }
      } else {
        bfly_regs<R, 0, LR>(b, th);  // raw = P^0 (*) W_e' through the m separable stages
#pragma unroll
        for (int zl = 0; zl < R; ++zl) raw[zl] = b[zl];
      }
    } else if constexpr (!DIRECT) {
      // separable path: own block of W_e' to linear; the m - LR high stages pair threads of
      // the team (lane ^ 2^(i-LR)), the LR low stages stay in registers
      float b[R];
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4) {
        float4 v = *reinterpret_cast<const float4*>(B + cm_idx<MB>(t * R + 4 * c4));
        b[4 * c4] = to_lin(v.x); b[4 * c4 + 1] = to_lin(v.y); b[4 * c4 + 2] = to_lin(v.z); b[4 * c4 + 3] = to_lin(v.w);
      }
      if (is_a) {
#pragma unroll
        for (int c4 = 0; c4 < R / 4; ++c4) {
          float4* pd = reinterpret_cast<float4*>(D + cm_idx<MB>(t * R + 4 * c4));
          float4 v = *pd;
          *pd = make_float4(to_lin(v.x), to_lin(v.y), to_lin(v.z), to_lin(v.w));
        }
      }
      bfly_regs<R, 0, LR>(b, th);
#pragma unroll
      for (int i = LR; i < MB; ++i) {
        const int off = 1 << (i - LR);
#pragma unroll
        for (int zl = 0; zl < R; ++zl) b[zl] = fmaf(th[i], __shfl_xor_sync(0xffffffffu, b[zl], off), b[zl]);
      }
#pragma unroll
      for (int zl = 0; zl < R; ++zl) raw[zl] = b[zl];
      __syncwarp();  // D conversions visible to the team
    } else if constexpr (PMF) {
      // probability-domain variable node as above, the team's high stages by shuffles
      float b[R];
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4) {
        float4 v = active ? *reinterpret_cast<const float4*>(B + cm_idx<MB>(t * R + 4 * c4)) : make_float4(0, 0, 0, 0);
        b[4 * c4] = to_lin(v.x); b[4 * c4 + 1] = to_lin(v.y); b[4 * c4 + 2] = to_lin(v.z); b[4 * c4 + 3] = to_lin(v.w);
      }
      if (is_a) {
#pragma unroll
        for (int c4 = 0; c4 < R / 4; ++c4) {
          float4* pd = reinterpret_cast<float4*>(D + cm_idx<MB>(t * R + 4 * c4));
          float4 v = *pd;
          *pd = make_float4(to_lin(v.x), to_lin(v.y), to_lin(v.z), to_lin(v.w));
        }
      }
      wht_team<MB, LR, R>(b, t);
#pragma unroll
      for (int zl = 0; zl < R; ++zl) b[zl] *= p0[zl];
      wht_team<MB, LR, R>(b, t);
#pragma unroll
      for (int zl = 0; zl < R; ++zl) raw[zl] = b[zl];
      __syncwarp();  // D conversions visible to the team
    } else {
      if (active) {
        // A <- P^0 (natural layout); B, D converted in place to linear (own chunks)
#pragma unroll
        for (int c4 = 0; c4 < R / 4; ++c4) {
          *reinterpret_cast<float4*>(A + t * R + 4 * c4) =
              make_float4(p0[4 * c4], p0[4 * c4 + 1], p0[4 * c4 + 2], p0[4 * c4 + 3]);
          float4* pb = reinterpret_cast<float4*>(B + cm_idx<MB>(t * R + 4 * c4));
          float4 v = *pb;
          *pb = make_float4(to_lin(v.x), to_lin(v.y), to_lin(v.z), to_lin(v.w));
        }
        if (is_a) {
#pragma unroll
          for (int c4 = 0; c4 < R / 4; ++c4) {
            float4* pd = reinterpret_cast<float4*>(D + cm_idx<MB>(t * R + 4 * c4));
            float4 v = *pd;
            *pd = make_float4(to_lin(v.x), to_lin(v.y), to_lin(v.z), to_lin(v.w));
          }
        }
      }
      __syncwarp();
      float2 acc[R / 2];
#pragma unroll
      for (int p = 0; p < R / 2; ++p) acc[p] = make_float2(0.0f, 0.0f);
      if (active) {
#pragma unroll 1
        for (int yh = 0; yh < NB; ++yh) {
          float a[R], b[R];
#pragma unroll
          for (int c4 = 0; c4 < R / 4; ++c4) {
            float4 va = *reinterpret_cast<const float4*>(A + yh * R + 4 * c4);
            a[4 * c4] = va.x; a[4 * c4 + 1] = va.y; a[4 * c4 + 2] = va.z; a[4 * c4 + 3] = va.w;
            float4 vb = *reinterpret_cast<const float4*>(B + cm_idx<MB>((t ^ yh) * R + 4 * c4));
            b[4 * c4] = vb.x; b[4 * c4 + 1] = vb.y; b[4 * c4 + 2] = vb.z; b[4 * c4 + 3] = vb.w;
          }
          conv_block<R>(a, b, acc);
        }
      }
#pragma unroll
      for (int p = 0; p < R / 2; ++p) { raw[2 * p] = acc[p].x; raw[2 * p + 1] = acc[p].y; }
    }

    // ---- normalise so that entry 0 is (0,0), Gamma in base 2, packed
    float raw0 = raw[0];
    if constexpr (TT > 1) raw0 = __shfl_sync(0xffffffffu, raw[0], lane & ~(TT - 1));
    uint32_t up[R];
    {
      const bool neutral = !(raw0 > 0.0f);  // DC term <= 0: numerical event (reading R10)
      const float lg0 = lg2a(raw0);
#pragma unroll
      for (int zl = 0; zl < R; ++zl) {
        float pk = pack(lg0 - lg2a(fabsf(raw[zl])), __float_as_uint(raw[zl]));
        if (neutral) pk = (t == 0 && zl == 0) ? 0.0f : kFloor;
        up[zl] = __float_as_uint(pk);
      }
      if (neutral && active && t == 0) atomicAdd(&ws.slot_events[s], 1);
    }
    if (P.u_out != nullptr && active) {
      float* dst = P.u_out + ((size_t)s * cd.E + e) * Q + t * R;
#pragma unroll
      for (int zl = 0; zl < R; ++zl) dst[zl] = __uint_as_float(up[zl]);
    }

    // ---- TENTATIVE DECISION at the variable's first edge:  M_v(z) = sum_y raw(y) W_e(z ^ y)
    // (raw is the unnormalised VN output, so M_v is exact up to a positive factor; per-thread
    // partial sums in fp32, the cross-thread reduction in fp64)
    if (do_dec) {
      float mf[MB + 1];  // the thread's partial sums (<= 16 terms) in fp32, reduced across the team in fp64
#pragma unroll
      for (int b = 0; b <= MB; ++b) mf[b] = 0.0f;
      if (is_a) {
        if constexpr (TT == 1) {
#pragma unroll
          for (int y = 0; y < Q; ++y) {
            mf[0] = fmaf(raw[y], dreg[y], mf[0]);
#pragma unroll
            for (int b = 0; b < MB; ++b) mf[b + 1] = fmaf(raw[y], dreg[y ^ (1 << b)], mf[b + 1]);
          }
        } else {
          float dv[R];
#pragma unroll
          for (int c4 = 0; c4 < R / 4; ++c4) {
            float4 v = *reinterpret_cast<const float4*>(D + cm_idx<MB>(t * R + 4 * c4));
            dv[4 * c4] = v.x; dv[4 * c4 + 1] = v.y; dv[4 * c4 + 2] = v.z; dv[4 * c4 + 3] = v.w;
          }
#pragma unroll
          for (int zl = 0; zl < R; ++zl) {
            mf[0] = fmaf(raw[zl], dv[zl], mf[0]);
#pragma unroll
            for (int b = 0; b < LR; ++b) mf[b + 1] = fmaf(raw[zl], dv[zl ^ (1 << b)], mf[b + 1]);
          }
#pragma unroll
          for (int b = LR; b < MB; ++b) {
            const int bb = t ^ (1 << (b - LR));
#pragma unroll
            for (int c4 = 0; c4 < R / 4; ++c4) {
              float4 v = *reinterpret_cast<const float4*>(D + cm_idx<MB>(bb * R + 4 * c4));
              mf[b + 1] = fmaf(raw[4 * c4], v.x, mf[b + 1]);
              mf[b + 1] = fmaf(raw[4 * c4 + 1], v.y, mf[b + 1]);
              mf[b + 1] = fmaf(raw[4 * c4 + 2], v.z, mf[b + 1]);
              mf[b + 1] = fmaf(raw[4 * c4 + 3], v.w, mf[b + 1]);
            }
          }
        }
      }
      double mv[MB + 1];
#pragma unroll
      for (int b = 0; b <= MB; ++b) mv[b] = (double)mf[b];
      if constexpr (TT > 1) {
#pragma unroll
        for (int off = TT / 2; off >= 1; off >>= 1)
#pragma unroll
          for (int b = 0; b <= MB; ++b) mv[b] += __shfl_xor_sync(0xffffffffu, mv[b], off);
      }
      if (want_soft) {
        // soft outputs: the whole decision in fp64 from the linear spectra (decision_f64, reading R22)
        float bl[R], dl[R], pl[PMF ? R : 1];
        const float* Wc = ws.W + ((size_t)(ell & 1) * ws.S + s) * EQ;  // this pass's input messages (packed)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int z = t * R + r;
          bl[r] = is_a ? __ldcg(Wc + (size_t)ed.partner * Q + z) : 1000.0f;  // 1000: Gamma^-1 = 0
          dl[r] = is_a ? __ldcg(Wc + (size_t)e * Q + z) : 1000.0f;
          if constexpr (PMF) pl[r] = is_a ? p0[r] : 0.0f;
        }
        decision_f64<MB, LR, PMF>(bl, dl, pl, th, t, mv);
      }
      const uint32_t s0z = mv[0] < 0.0 ? 1u : 0u;  // sgn_GF2 M(0); an exact zero has sign 0
      if (is_a && t == 0) {
        int x = 0;
#pragma unroll
        for (int b = 0; b < MB; ++b) x |= (int)(((mv[b + 1] < 0.0) ? 1u : 0u) ^ s0z) << b;
        ws.xhat[(size_t)s * cd.N + ed.var] = (uint8_t)x;
        if (mode == 0) {  // syndrome contributions h_cv xhat_v to both checks of v
          int ca = 0, cb = 0;
          if (x != 0) {
            const int lx = __ldg(&cd.gf_log[x]);
            ca = __ldg(&cd.gf_exp[ed.logh + lx]);
            cb = __ldg(&cd.gf_exp[ed.plogh + lx]);
          }
          ws.con[(size_t)s * ws.con_stride + e] = (uint8_t)ca;
          ws.con[(size_t)s * ws.con_stride + ed.partner] = (uint8_t)cb;
        }
        if (want_soft) {
#pragma unroll
          for (int b = 0; b < MB; ++b) ws.soft[((size_t)s * cd.N + ed.var) * MB + b] = soft_ratio(mv[b + 1], mv[0]);
        }
      }
      if constexpr (DIRECT) {
        if (call->post_out != nullptr || call->map_out != nullptr) {
          // symbol-level decision: mu_v(x) = sum_z M_v(z) (-1)^{z.x} with
          // M_v = raw (*) W_e, i.e. mu_v = WHT(raw) . WHT(W_e) (the XOR-convolution theorem);
          // clamped at 0 and normalised to a posterior, argmax ties -> lowest x
          float a[R], b[R];
#pragma unroll
          for (int zl = 0; zl < R; ++zl) a[zl] = raw[zl];
          if constexpr (TT == 1) {
#pragma unroll
            for (int y = 0; y < Q; ++y) b[y] = is_a ? dreg[y] : 0.0f;
          } else {
#pragma unroll
            for (int c4 = 0; c4 < R / 4; ++c4) {
              float4 v = is_a ? *reinterpret_cast<const float4*>(D + cm_idx<MB>(t * R + 4 * c4)) : make_float4(0, 0, 0, 0);
              b[4 * c4] = v.x; b[4 * c4 + 1] = v.y; b[4 * c4 + 2] = v.z; b[4 * c4 + 3] = v.w;
            }
          }
          wht_team<MB, LR, R>(a, t);
          wht_team<MB, LR, R>(b, t);
          float tot = 0.0f, best = 0.0f;
          int bx = 0;
#pragma unroll
          for (int zl = 0; zl < R; ++zl) {
            a[zl] = fmaxf(a[zl] * b[zl], 0.0f);  // mu >= 0; rounding residues below 0 clamp to 0
            tot += a[zl];
            if (zl == 0 || a[zl] > best) { best = a[zl]; bx = t * R + zl; }
          }
          if constexpr (TT > 1) {
#pragma unroll
            for (int off = TT / 2; off >= 1; off >>= 1) {
              tot += __shfl_xor_sync(0xffffffffu, tot, off);
              const float ob = __shfl_xor_sync(0xffffffffu, best, off);
              const int ox = __shfl_xor_sync(0xffffffffu, bx, off);
              if (ob > best || (ob == best && ox < bx)) { best = ob; bx = ox; }
            }
          }
          // written straight to the frame's output rows at every iteration: the stopping
          // iteration's write is the last one (no per-slot copy when the frame finishes)
          if (is_a && call->post_out) {
            const float inv = tot > 0.0f ? 1.0f / tot : 0.0f;
            float* dst = call->post_out + ((size_t)f * cd.N + ed.var) * Q + t * R;
            if constexpr (R >= 4) {
#pragma unroll
              for (int c4 = 0; c4 < R / 4; ++c4)
                reinterpret_cast<float4*>(dst)[c4] =
                    make_float4(a[4 * c4] * inv, a[4 * c4 + 1] * inv, a[4 * c4 + 2] * inv, a[4 * c4 + 3] * inv);
            } else {
#pragma unroll
              for (int zl = 0; zl < R; ++zl) dst[zl] = a[zl] * inv;
            }
          }
          if (is_a && t == 0 && call->map_out) call->map_out[(size_t)f * cd.N + ed.var] = (uint8_t)bx;
        }
      }
      if (mode == 1) {
        // paper-mode fast syndrome: sign bits of M_v(H_cv alpha^i) for both checks
        uint64_t pa = 0, pbv = 0;
        if (is_a) {
          const uint32_t* ea = reinterpret_cast<const uint32_t*>(cd.edges + e) + 3;
          const uint32_t* eb = reinterpret_cast<const uint32_t*>(cd.edges + ed.partner) + 3;
          pa = (uint64_t)__ldg(ea) | ((uint64_t)__ldg(ea + 1) << 32);
          pbv = (uint64_t)__ldg(eb) | ((uint64_t)__ldg(eb + 1) << 32);
        }
        int ma = 0, mb = 0;
#pragma unroll 1
        for (int i = 0; i < 2 * MB; ++i) {
          const int z = (int)(((i < MB ? pa : pbv) >> (8 * (i < MB ? i : i - MB))) & 0xFF);
          float accf = 0.0f;
          if (is_a) {
#pragma unroll
            for (int zl = 0; zl < R; ++zl) {
              const int yy = (t * R + zl) ^ z;
              accf = fmaf(raw[zl], D[cm_idx<MB>(yy)], accf);
            }
          }
          double acc = (double)accf;
          if constexpr (TT > 1) {
#pragma unroll
            for (int off = TT / 2; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
          }
          const int bit = (int)(((acc < 0.0) ? 1u : 0u) ^ s0z);
          if (i < MB) ma |= bit << i; else mb |= bit << (i - MB);
        }
        if (is_a && t == 0) {
          ws.con[(size_t)s * ws.con_stride + e] = (uint8_t)ma;
          ws.con[(size_t)s * ws.con_stride + ed.partner] = (uint8_t)mb;
        }
      }
    }

    // ---- CHECK TO VARIABLE: T_j(w) = U_j(pi_j w);  W_j(z) = sum_{j' != j} T_j'(pi_j^-1 z)
    if (do_cn) {
      int pl[R];  // pi_h^-1 of the thread's outputs (linear map: XOR of basis images)
      {
        int base = 0;
#pragma unroll
        for (int b = LR; b < MB; ++b)
          if ((t >> (b - LR)) & 1) base ^= ed.pinvb[b];
        pl[0] = base;
#pragma unroll
        for (int b = 0; b < LR; ++b)
#pragma unroll
          for (int jj = 0; jj < (1 << b); ++jj) pl[(1 << b) + jj] = pl[jj] ^ ed.pinvb[b];
      }
      if constexpr (TT > 1) __syncwarp();  // team done reading A in the convolution
      if (active) {
#pragma unroll
        for (int zl = 0; zl < R; ++zl) A[pl[zl]] = __uint_as_float(up[zl]);
      } else if (cvalid) {
#pragma unroll
        for (int zl = 0; zl < R; ++zl) A[t * R + zl] = 0.0f;  // padding edge: neutral (0, 0)
      }
      check_sync(lc, TPC);
      if (lc < P.checks_per_cta && c < cd.M) {
        const float* Ab = smem + (size_t)(lc * (TPC / TT)) * C::TEAM_FLOATS;
        for (int w = threadIdx.x - lc * TPC; w < Q; w += TPC) {
          float mag = 0.0f;
          uint32_t sg = 0;
          for (int jj = 0; jj < cd.k_max; ++jj) {
            const float x = Ab[(size_t)jj * C::TEAM_FLOATS + w];
            mag += fabsf(x);
            sg ^= __float_as_uint(x);
          }
          TOT[w] = __uint_as_float(__float_as_uint(mag) | (sg & kSign));
        }
      }
      check_sync(lc, TPC);
      if (active) {
        float out[R];
#pragma unroll
        for (int zl = 0; zl < R; ++zl) {
          const float x = TOT[pl[zl]];
          const float u = __uint_as_float(up[zl]);
          out[zl] = pack(fabsf(x) - fabsf(u), __float_as_uint(x) ^ up[zl]);
        }
        float* dst = ws.W + ((size_t)((ell + 1) & 1) * ws.S + s) * EQ + (size_t)e * Q + t * R;
        if constexpr (R >= 4) {
#pragma unroll
          for (int c4 = 0; c4 < R / 4; ++c4)
            reinterpret_cast<float4*>(dst)[c4] = make_float4(out[4 * c4], out[4 * c4 + 1], out[4 * c4 + 2], out[4 * c4 + 3]);
        } else {
#pragma unroll
          for (int zl = 0; zl < R; ++zl) dst[zl] = out[zl];
        }
      }
    }

    // ---- slot bookkeeping, per warp: the warp that finishes the slot last (over all CTAs of
    // the slot) runs the syndrome, the stopping rule and the refill.  The release add is
    // cumulative over the warp's writes (ordered by __syncwarp); the finisher acquires.
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atom_add_release_gpu(&ws.slot_counter[s], 1) == slot_target - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) continue;
    fence_acquire_gpu();
    if (lane == 0) ws.slot_counter[s] = 0;
    if (P.step_mode) continue;
    if (ell == 0) {
      if (lane == 0) ws.slot_iter[s] = 1;
      continue;
    }
    // syndrome: s_c = XOR of the contribution bytes on the check's kpad edge slots, read as
    // 16-byte vectors; a check spans kpad/16 consecutive lanes when kpad > 16
    int bad = 0;
    {
      const uint4* cs = reinterpret_cast<const uint4*>(ws.con + (size_t)s * ws.con_stride);
      const int nvec = ws.con_stride >> 4;
      const int kp = cd.kpad;
#pragma unroll 4
      for (int it = 0; it < (nvec + 31) / 32; ++it) {
        const int v = lane + 32 * it;
        const uint4 x = v < nvec ? __ldcg(cs + v) : make_uint4(0, 0, 0, 0);
        uint32_t f0, f1 = 0, f2 = 0, f3 = 0;
        if (kp == 4) {
          f0 = x.x; f1 = x.y; f2 = x.z; f3 = x.w;
        } else if (kp == 8) {
          f0 = x.x ^ x.y; f1 = x.z ^ x.w;
        } else {
          f0 = x.x ^ x.y ^ x.z ^ x.w;
          for (int off = 1; off < (kp >> 4); off <<= 1) f0 ^= __shfl_xor_sync(0xffffffffu, f0, off);
        }
        f0 ^= f0 >> 16; f1 ^= f1 >> 16; f2 ^= f2 >> 16; f3 ^= f3 >> 16;
        f0 ^= f0 >> 8; f1 ^= f1 >> 8; f2 ^= f2 >> 8; f3 ^= f3 >> 8;
        bad |= (int)((f0 | f1 | f2 | f3) & 0xFFu);
      }
    }
    const int ok = !__any_sync(0xffffffffu, bad != 0);
    const bool done = (call->early_stop && ok) || ell >= max_iters;
    if (!done) {
      if (lane == 0) ws.slot_iter[s] = ell + 1;
      continue;
    }
    const int N = cd.N;
    if ((N & 15) == 0) {  // 16-byte copies (the frame's rows are 16-byte aligned)
      const uint4* src = reinterpret_cast<const uint4*>(ws.xhat + (size_t)s * N);
      uint4* dst = reinterpret_cast<uint4*>(call->hard + (size_t)f * N);
#pragma unroll 4
      for (int v = lane; v < (N >> 4); v += 32) dst[v] = __ldcg(src + v);
    } else {
      for (int v = lane; v < N; v += 32) call->hard[(size_t)f * N + v] = __ldcg(&ws.xhat[(size_t)s * N + v]);
    }
    if (want_soft) {
#pragma unroll 4
      for (int i = lane; i < N * MB; i += 32)
        call->soft_out[(size_t)f * N * MB + i] = __ldcg(&ws.soft[(size_t)s * N * MB + i]);
    }
    if (lane == 0) {
      call->ok[f] = (uint8_t)ok;
      call->iters[f] = ell;
      if (call->events_out) call->events_out[f] = ws.slot_events[s];
      ws.slot_events[s] = 0;
      const int nf = atomicAdd(&ws.glob[0], 1);
      if (nf < call->frames) {
        ws.slot_frame[s] = nf;
        ws.slot_iter[s] = 0;
      } else {
        ws.slot_frame[s] = -1;
        atomicSub(&ws.glob[1], 1);
      }
    }
  }
  cp_async_wait<0>();
#undef NB_BV
#undef NB_DV
#undef NB_TH
}

// the small control kernels are defined in nbldpc.cu's translation unit only (NB_CONTROL_KERNELS)
#ifdef NB_CONTROL_KERNELS
__global__ void nb_setup_kernel(WorkDev ws, CallDev call) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    *ws.call = call;
    const int n = call.frames < ws.S ? call.frames : ws.S;
    ws.glob[0] = n;
    ws.glob[1] = n;
    ws.glob[2] = 0;
  }
  if (i < ws.S) {
    ws.slot_frame[i] = i < call.frames ? i : -1;
    ws.slot_iter[i] = 0;
    ws.slot_events[i] = 0;
    ws.slot_counter[i] = 0;
    ws.slot_epoch[i] = 0;
  }
}

// cluster kernel: frames are taken from glob[0] starting at 0; slot = cluster
__global__ void nb_cluster_setup_kernel(WorkDev ws, CallDev call) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    *ws.call = call;
    ws.glob[0] = 0;
    ws.glob[1] = 0;
    ws.glob[2] = 0;
  }
  if (i < ws.S) ws.slot_events[i] = 0;
}

// step mode: slots hold frames 0..frames-1 at iteration `iter`
__global__ void nb_step_setup_kernel(WorkDev ws, CallDev call, int iter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *ws.call = call;
  if (i < ws.S) {
    ws.slot_frame[i] = i;
    ws.slot_iter[i] = iter;
    ws.slot_events[i] = 0;
    ws.slot_counter[i] = 0;
    ws.slot_epoch[i] = 0;
  }
}

// Tt[fv][b] = tanh(L_{fv,b} / 2), rows of 8 floats (m used)
__global__ void nb_tanh_kernel(const float* llr, float* Tt, size_t nvar, int m) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nvar * m; i += (size_t)gridDim.x * blockDim.x)
    Tt[(i / m) * 8 + i % m] = tanhf(0.5f * llr[i]);
}

__global__ void nb_control_kernel(int32_t* glob, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0) {
    glob[2] += 1;  // WHILE-body iterations (launch accounting)
    if (*(volatile const int32_t*)&glob[1] == 0) cudaGraphSetConditional(h, 0);
  }
}
#endif  // NB_CONTROL_KERNELS

}  // namespace nb
