// logsp.cuh -- the conventional logarithm-domain SP decoder (Log-SP) on sm_100a:
// the paper's comparison algorithm (Table 1, made empirical).
//
// Messages are log2-probability vectors lambda(x), x in GF(2^m) (natural order, one float per entry).
// One CTA decodes one frame at a time (persistent over frames, a global frame counter); a flooding
// iteration is three phases separated by __syncthreads:
//   CHECK TO VARIABLE: per check, lambda~_vc(x) = lambda_vc(h^-1 x) with the
//     variable-to-check message lambda_vc = lambda_v^0 + lambda_c'v (degree-2 variable node, :262-266,
//     fused here); the leave-one-out log-convolutions [x]_{v' != v} by forward-backward: 3(k-2)
//     log-convolutions of q^2 terms per check.  Each log-convolution is evaluated through the exact
//     identity e^{a+b} = e^a e^b (reading R8): the inputs are exponentiated once (ex2, after removing
//     their maximum), convolved with FFMA2 (the direct-VN kernel's conv_block), and the outputs take
//     one lg2 each.  Entries below 2^-126 of their vector's maximum underflow to "zero" (reading R25).
//   TENTATIVE DECISION: mu_v(x) = lambda_v^0(x) + sum_c' lambda_c'v(x),
//     xhat_v = argmax (ties: lowest x) -- the symbol-MAP decision of Log-SP.
//   syndrome of xhat (exact), early termination.
// A check is owned by a team of TT = max(1, q/16) threads holding R = min(q, 16) entries each; the
// team's vectors (the forward products F_i, the current input, the backward product) live in shared
// memory.
#pragma once
#include "decoder.cuh"

namespace nb {

struct LsParams {
  CodeDev code;
  float* W;         // [2][S][E][q] check-to-variable messages (ping-pong), log2, natural order
  float* L0s;       // [S][N][q] lambda_v^0 (log2), per slot
  uint8_t* xh;      // [S][N] decisions of the current iteration
  int32_t* glob;    // [0] next frame
  const float* llr; // [frames][N*m] or NULL
  const float* pmf; // [frames][N][q] or NULL
  uint8_t* hard;
  uint8_t* ok;
  int32_t* iters;
  int frames, max_iters, early_stop;
  int teams;        // check teams per CTA
  int kmax;
};

template <int MB>
struct LsCfg {
  static constexpr int Q = 1 << MB;
  static constexpr int R = Q < 16 ? Q : 16;
  static constexpr int TT = Q / R;
  static constexpr int LR = MB < 4 ? MB : 4;
};

// maximum over the TT lanes of a team (tmask: the team's lanes; teams may diverge from each other)
template <int TT>
__device__ __forceinline__ float team_max(float v, unsigned tmask) {
#pragma unroll
  for (int off = TT / 2; off >= 1; off >>= 1) v = fmaxf(v, __shfl_xor_sync(tmask, v, off));
  return v;
}

// out block t (R entries, natural layout) of A (*) B over GF(2)^m: sum_yh conv_block(A_yh, B_{t^yh})
template <int MB>
__device__ __forceinline__ void ls_conv(const float* A, const float* B, int t, float (&out)[LsCfg<MB>::R]) {
  using C = LsCfg<MB>;
  constexpr int R = C::R, TT = C::TT;
  float2 acc[R / 2];
#pragma unroll
  for (int p = 0; p < R / 2; ++p) acc[p] = make_float2(0.0f, 0.0f);
#pragma unroll 1
  for (int yh = 0; yh < TT; ++yh) {
    float a[R], b[R];
    if constexpr (R >= 4) {
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4) {
        const float4 va = *reinterpret_cast<const float4*>(A + yh * R + 4 * c4);
        const float4 vb = *reinterpret_cast<const float4*>(B + (t ^ yh) * R + 4 * c4);
        a[4 * c4] = va.x; a[4 * c4 + 1] = va.y; a[4 * c4 + 2] = va.z; a[4 * c4 + 3] = va.w;
        b[4 * c4] = vb.x; b[4 * c4 + 1] = vb.y; b[4 * c4 + 2] = vb.z; b[4 * c4 + 3] = vb.w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) { a[r] = A[r]; b[r] = B[r]; }
    }
    conv_block<R>(a, b, acc);
  }
#pragma unroll
  for (int p = 0; p < R / 2; ++p) { out[2 * p] = acc[p].x; out[2 * p + 1] = acc[p].y; }
}

template <int MB>
__global__ void __launch_bounds__(256) ls_frame_kernel(LsParams P) {
  using C = LsCfg<MB>;
  constexpr int Q = C::Q, R = C::R, TT = C::TT;
  extern __shared__ __align__(16) float smem[];
  __shared__ int sh_frame;
  const CodeDev& cd = P.code;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
  const int team = tid / TT, t = tid & (TT - 1);
  const bool in_team = team < P.teams;
  // the team's lanes: teams run their own loops (checks of different degrees, ragged counts), so
  // every team-level shuffle and barrier names only them
  const unsigned tmask = TT >= 32 ? 0xffffffffu : (((1u << TT) - 1u) << (lane & ~(TT - 1)));
  const int VS = P.kmax + 1;                      // vectors per team: F_0..F_{kmax-2}, Pbuf, Bbuf
  float* const Tb = smem + (size_t)(in_team ? team : 0) * VS * Q;
  float* const Pbuf = Tb + (P.kmax - 1) * Q;
  float* const Bbuf = Pbuf + Q;
  int* const gexp = reinterpret_cast<int*>(smem + (size_t)P.teams * VS * Q);  // [2q] alpha^i
  int* const glog = gexp + 2 * Q;                                              // [q]
  for (int i = tid; i < 2 * (Q - 1) + 1; i += nthr) gexp[i] = cd.gf_exp[i];
  for (int i = tid; i < Q; i += nthr) glog[i] = cd.gf_log[i];
  __syncthreads();
  auto gmul = [&](int h, int x) { return x == 0 ? 0 : gexp[glog[h] + glog[x]]; };

  const int slot = blockIdx.x;
  const int S = gridDim.x;
  const size_t EQ = (size_t)cd.E * Q;
  float* const L0 = P.L0s + (size_t)slot * cd.N * Q;
  uint8_t* const xh = P.xh + (size_t)slot * cd.N;

  // ---- one input vector: lambda~(h y) = lambda_v^0(y) + lambda_c'v(y); the team's block y = tR..,
  // exponentiated after removing the team maximum, scattered to dst at h*y
  auto load_p = [&](int e, const float* Win, bool first, float* dst) {
    const EdgeDev ed = cd.edges[e];
    float l[R];
    const float* l0 = L0 + (size_t)ed.var * Q + t * R;
    const float* wi = Win + (size_t)ed.partner * Q + t * R;
    if constexpr (R >= 4) {  // 16-byte loads of the two rows
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4) {
        const float4 a = reinterpret_cast<const float4*>(l0)[c4];
        const float4 w = first ? make_float4(0.f, 0.f, 0.f, 0.f) : reinterpret_cast<const float4*>(wi)[c4];
        l[4 * c4] = a.x + w.x; l[4 * c4 + 1] = a.y + w.y; l[4 * c4 + 2] = a.z + w.z; l[4 * c4 + 3] = a.w + w.w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) l[r] = l0[r] + (first ? 0.0f : wi[r]);
    }
    float mx = l[0];
#pragma unroll
    for (int r = 1; r < R; ++r) mx = fmaxf(mx, l[r]);
    mx = team_max<TT>(mx, tmask);
#pragma unroll
    for (int r = 0; r < R; ++r) dst[gmul(ed.h, t * R + r)] = ex2a(l[r] - mx);
  };
  // ---- one output vector: lambda_cv(x) = lambda~_cv(h x), log2, maximum removed
  auto store_w = [&](int e, const float* src, float* Wout) {
    const int h = cd.edges[e].h;
    float v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[gmul(h, t * R + r)];
    float mx = v[0];
#pragma unroll
    for (int r = 1; r < R; ++r) mx = fmaxf(mx, v[r]);
    mx = team_max<TT>(mx, tmask);
    const float lmx = mx > 0.0f ? lg2a(mx) : 0.0f;
    float* dst = Wout + (size_t)e * Q + t * R;
    float o[R];
#pragma unroll
    for (int r = 0; r < R; ++r) o[r] = v[r] > 0.0f ? lg2a(v[r]) - lmx : -kFloor;
    if constexpr (R >= 4) {
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4)
        reinterpret_cast<float4*>(dst)[c4] = make_float4(o[4 * c4], o[4 * c4 + 1], o[4 * c4 + 2], o[4 * c4 + 3]);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) dst[r] = o[r];
    }
  };
  auto team_sync = [&]() {
    if constexpr (TT > 1) __syncwarp(tmask);  // a one-thread team owns its vectors alone
  };

#pragma unroll 1
  for (;;) {
    if (tid == 0) sh_frame = atomicAdd(P.glob, 1);
    __syncthreads();
    const int f = sh_frame;
    if (f >= P.frames) break;
    // lambda_v^0 in log2, normalised to lambda(0) = 0 for LLRs:
    // ln Pr(x) - ln Pr(0) = -sum_{i in x} L_i; ln p(x) for a pmf (0 -> floor)
    for (int i = tid; i < cd.N * Q; i += nthr) {
      const int v = i / Q, x = i - v * Q;
      float val;
      if (P.pmf) {
        const float p = P.pmf[((size_t)f * cd.N + v) * Q + x];
        val = p > 0.0f ? lg2a(p) : -kFloor;
      } else {
        float s = 0.0f;
        for (int b = 0; b < MB; ++b)
          if ((x >> b) & 1) s += P.llr[((size_t)f * cd.N + v) * MB + b];
        val = -s * 1.4426950408889634f;
      }
      L0[i] = val;
    }
    __syncthreads();
    int ell = 0, okv = 0;
#pragma unroll 1
    for (;;) {
      const float* Win = P.W + ((size_t)(ell & 1) * S + slot) * EQ;
      float* Wout = P.W + ((size_t)((ell + 1) & 1) * S + slot) * EQ;
      // ---- CHECK TO VARIABLE, forward-backward over the check's edges
      if (in_team) {
#pragma unroll 1
        for (int c = team; c < cd.M; c += P.teams) {
          const int e0 = c * cd.kpad;
          int kc = 0;
          while (kc < cd.kpad && cd.edges[e0 + kc].var >= 0) ++kc;
          load_p(e0, Win, ell == 0, Tb);  // F_0 = P_0
          team_sync();
          for (int i = 1; i + 1 < kc; ++i) {  // F_i = F_{i-1} (*) P_i
            load_p(e0 + i, Win, ell == 0, Pbuf);
            team_sync();
            float o[R];
            ls_conv<MB>(Tb + (i - 1) * Q, Pbuf, t, o);
            float mx = o[0];
#pragma unroll
            for (int r = 1; r < R; ++r) mx = fmaxf(mx, o[r]);
            mx = team_max<TT>(mx, tmask);
            const float inv = mx > 0.0f ? 1.0f / mx : 0.0f;  // rescale: the vectors stay O(1)
#pragma unroll
            for (int r = 0; r < R; ++r) Tb[i * Q + t * R + r] = o[r] * inv;
            team_sync();
          }
          load_p(e0 + kc - 1, Win, ell == 0, Bbuf);  // B = P_{k-1}
          team_sync();
          store_w(e0 + kc - 1, Tb + (kc - 2) * Q, Wout);  // out_{k-1} = F_{k-2}
          for (int i = kc - 2; i >= 1; --i) {
            float o[R], nb[R];
            ls_conv<MB>(Tb + (i - 1) * Q, Bbuf, t, o);  // out_i = F_{i-1} (*) B_{i+1}
            team_sync();
            load_p(e0 + i, Win, ell == 0, Pbuf);
            team_sync();
            ls_conv<MB>(Pbuf, Bbuf, t, nb);  // B_i = P_i (*) B_{i+1}
            float mx = nb[0];
#pragma unroll
            for (int r = 1; r < R; ++r) mx = fmaxf(mx, nb[r]);
            mx = team_max<TT>(mx, tmask);
            const float inv = mx > 0.0f ? 1.0f / mx : 0.0f;
            team_sync();
#pragma unroll
            for (int r = 0; r < R; ++r) {
              Pbuf[t * R + r] = o[r];
              Bbuf[t * R + r] = nb[r] * inv;
            }
            team_sync();
            store_w(e0 + i, Pbuf, Wout);
            team_sync();
          }
          store_w(e0, Bbuf, Wout);  // out_0 = B_1
          team_sync();
        }
      }
      ++ell;
      __syncthreads();
      // ---- TENTATIVE DECISION at every variable's first edge: argmax of mu_v
      if (in_team) {
#pragma unroll 1
        for (int e = team; e < cd.E; e += P.teams) {
          const EdgeDev ed = cd.edges[e];
          if (ed.var < 0 || !ed.is_a) continue;
          const float* l0 = L0 + (size_t)ed.var * Q + t * R;
          const float* wa = Wout + (size_t)e * Q + t * R;
          const float* wb = Wout + (size_t)ed.partner * Q + t * R;
          float best = -3.0e38f;
          int bx = 0;
          float mu[R];
          if constexpr (R >= 4) {
#pragma unroll
            for (int c4 = 0; c4 < R / 4; ++c4) {
              const float4 a = reinterpret_cast<const float4*>(l0)[c4];
              const float4 b = reinterpret_cast<const float4*>(wa)[c4];
              const float4 d = reinterpret_cast<const float4*>(wb)[c4];
              mu[4 * c4] = a.x + b.x + d.x; mu[4 * c4 + 1] = a.y + b.y + d.y;
              mu[4 * c4 + 2] = a.z + b.z + d.z; mu[4 * c4 + 3] = a.w + b.w + d.w;
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) mu[r] = l0[r] + wa[r] + wb[r];
          }
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (mu[r] > best) { best = mu[r]; bx = t * R + r; }
#pragma unroll
          for (int off = TT / 2; off >= 1; off >>= 1) {
            const float ob = __shfl_xor_sync(tmask, best, off);
            const int ox = __shfl_xor_sync(tmask, bx, off);
            if (ob > best || (ob == best && ox < bx)) { best = ob; bx = ox; }
          }
          if (t == 0) xh[ed.var] = (uint8_t)bx;
        }
      }
      __syncthreads();
      // ---- exact syndrome of xhat and the stopping rule
      int bad = 0;
      for (int c = tid; c < cd.M; c += nthr) {
        int s = 0;
        for (int j = 0; j < cd.kpad; ++j) {
          const EdgeDev ed = cd.edges[c * cd.kpad + j];
          if (ed.var < 0) break;
          s ^= gmul(ed.h, xh[ed.var]);
        }
        bad |= s;
      }
      okv = !__syncthreads_or(bad != 0);
      if ((P.early_stop && okv) || ell >= P.max_iters) break;
    }
    for (int v = tid; v < cd.N; v += nthr) P.hard[(size_t)f * cd.N + v] = xh[v];
    if (tid == 0) {
      P.ok[f] = (uint8_t)okv;
      P.iters[f] = ell;
    }
    __syncthreads();
  }
}

}  // namespace nb
