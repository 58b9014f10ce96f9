// lf_general.cuh -- Log-Fourier SP for any column weight j >= 1 (PAPER.md:101
// "the extension to general j is straightforward"), and for any code through NBLDPC_VN_GENERAL.
//
// A variable of degree d sends U_i = normalise(P^0 (*) W_1 (*) .. (*) W_d without W_i) to its i-th
// check (PAPER.md:486-494 with |C_v| = d).  The (d-1)-fold XOR-convolution is evaluated in the
// probability domain (the XOR-convolution theorem): w_i = WHT(W_i) / q, the
// leave-one-out products p^0 prod_{i' != i} w_i', and U_i = WHT of that -- 2 transforms of m q
// butterflies per edge instead of (d-1) q^2-term convolutions.  The decision needs only
// mu = p^0 prod_i w_i: M_v(0) = sum_x mu(x), M_v(alpha^b) = sum_x mu(x) (-1)^{x_b},
// and the symbol posterior mu / M_v(0).  The check node is the Log-Fourier one
// (PAPER.md:474-482): TOT(w) = sum_k U_k(pi_k w) (log-magnitudes add, signs XOR), then
// W_j(z) = TOT(pi_j^-1 z) - U_j(z).
//
// One CTA decodes one frame at a time (persistent over frames); an iteration is two phases
// (check node, then variable node + decision) and the syndrome, separated by __syncthreads.  Teams of
// TT = max(1, q/16) threads hold R = min(q, 16) entries of a vector each (natural layout z = tR + r).
// Messages (U and W, packed sign | -log2|x| like the other kernels) live per slot in HBM: J3's 444 slots x
// 1.6 MB exceed the 126 MB L2 (ncu, profiles/r01_ncu_j3_general.txt: 63% L2 hit rate, 123 GB of DRAM traffic).
#pragma once
#include "decoder.cuh"

namespace nb {

struct GenParams {
  CodeDev code;
  const int32_t* v_ptr;   // [N+1] variable -> its edges v_edges[v_ptr[v] .. v_ptr[v+1]-1] (internal slots)
  const int32_t* v_edges;
  float* U;               // [S][E][q] variable-to-check messages
  float* W;               // [S][E][q] check-to-variable messages
  uint8_t* xh;            // [S][N]
  int32_t* glob;          // [0] next frame
  const float* llr;       // [frames][N*m] or NULL
  const float* pmf;       // [frames][N][q] or NULL
  uint8_t* hard;
  uint8_t* ok;
  int32_t* iters;
  float* soft_out;        // [frames][N*m] or NULL (rewritten every iteration; the last write is the stopping one)
  int32_t* events_out;    // [frames] or NULL
  float* post_out;        // [frames][N][q] or NULL
  uint8_t* map_out;       // [frames][N] or NULL
  int frames, max_iters, early_stop;
  int teams;              // teams per CTA
  int jmax;               // largest column weight
};

// The decision in fp64 for soft outputs (reading R22, as decision_f64 of the degree-2 kernels):
// mu = p0 prod_i w_i with w_i = WHT(Gamma^-1(W_i)) evaluated in fp64 from the fp32 spectra, then
// M_v(0) = sum mu and M_v(alpha^b) = sum mu (-1)^{x_b} (the 1/q factors are positive
// and cancel in every sign and ratio).  Team layout z = R t + r; tmask: the team's lanes.
template <int MB, int LR>
__device__ __noinline__ void general_decision_f64(const float* W, const int32_t* edges, int d, const float* p0, int t,
                                                  unsigned tmask, double* md) {
  constexpr int Q = 1 << MB, R = 1 << LR, TT = Q / R;
  double mu[R];
#pragma unroll
  for (int r = 0; r < R; ++r) mu[r] = (double)p0[r];
  for (int i = 0; i < d; ++i) {
    double x[R];
    const float* src = W + (size_t)edges[i] * Q + t * R;
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = lin64(src[r]);  // Gamma^-1 in fp64 (see decision_f64)
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
        const double o = __shfl_xor_sync(tmask, x[r], off);
        x[r] = (t & off) ? o - x[r] : x[r] + o;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) mu[r] *= x[r];
  }
  double s = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) s += mu[r];
  md[0] = s;
#pragma unroll
  for (int b = 0; b < MB; ++b) {
    double sb = 0.0;
    if (b < LR) {
#pragma unroll
      for (int r = 0; r < R; ++r) sb += ((r >> b) & 1) ? -mu[r] : mu[r];
    } else {
      sb = ((t >> (b - LR)) & 1) ? -s : s;
    }
    md[b + 1] = sb;
  }
  if constexpr (TT > 1) {
#pragma unroll
    for (int off = TT / 2; off >= 1; off >>= 1)
#pragma unroll
      for (int b = 0; b <= MB; ++b) md[b] += __shfl_xor_sync(tmask, md[b], off);
  }
}

// SOFT = true: soft outputs requested (the fp64 decision); a separate instantiation so the plain kernel keeps
// its 80 registers (with the fp64 call site in it: 128 registers and spills, J3 7% slower)
template <int MB, bool SOFT = false>
__global__ void __launch_bounds__(256) lfg_frame_kernel(GenParams P) {
  constexpr int Q = 1 << MB, R = Q < 16 ? Q : 16, TT = Q / R, LR = MB < 4 ? MB : 4;
  extern __shared__ __align__(16) float smem[];
  __shared__ int sh_frame, sh_events;
  const CodeDev& cd = P.code;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
  const int team = tid / TT, t = tid & (TT - 1);
  const bool in_team = team < P.teams;
  const unsigned tmask = TT >= 32 ? 0xffffffffu : (((1u << TT) - 1u) << (lane & ~(TT - 1)));
  // team vectors: w_1..w_d (variable phase) / TOT and one staged U row (check phase)
  const int VS = P.jmax > 2 ? P.jmax : 2;
  // team stride padded to TT (mod 32): the per-thread vector entries at [i][r][t] of the teams of a
  // warp then fall in 32 distinct banks
  const int TS = VS * Q + ((TT - (VS * Q) % 32) & 31);
  float* const Tb = smem + (size_t)(in_team ? team : 0) * TS;
  int* const gexp = reinterpret_cast<int*>(smem + (size_t)P.teams * TS);
  int* const glog = gexp + 2 * Q;
  for (int i = tid; i < 2 * (Q - 1) + 1; i += nthr) gexp[i] = cd.gf_exp[i];
  for (int i = tid; i < Q; i += nthr) glog[i] = cd.gf_log[i];
  __syncthreads();
  auto gmul = [&](int h, int x) { return x == 0 ? 0 : gexp[glog[h] + glog[x]]; };
  auto team_sum = [&](float v) {
#pragma unroll
    for (int off = TT / 2; off >= 1; off >>= 1) v += __shfl_xor_sync(tmask, v, off);
    return v;
  };
  // in-place WHT of the team's vector (LR register stages, the rest by shuffles within the team)
  auto wht = [&](float (&x)[R]) {
#pragma unroll
    for (int b = 0; b < LR; ++b)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (!(r & (1 << b))) {
          const float u = x[r], w = x[r | (1 << b)];
          x[r] = u + w;
          x[r | (1 << b)] = u - w;
        }
#pragma unroll
    for (int b = LR; b < MB; ++b) {
      const int off = 1 << (b - LR);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float o = __shfl_xor_sync(tmask, x[r], off);
        x[r] = (t & off) ? o - x[r] : x[r] + o;
      }
    }
  };
  // pi_h images of the thread's z = tR + r (linear over GF(2): XOR of the basis images b[i] = pi(e_i))
  auto perm_block = [&](const uint8_t* b, int (&idx)[R]) {
    int base = 0;
#pragma unroll
    for (int i = LR; i < MB; ++i)
      if ((t >> (i - LR)) & 1) base ^= b[i];
    idx[0] = base;
#pragma unroll
    for (int i = 0; i < LR; ++i)
#pragma unroll
      for (int jj = 0; jj < (1 << i); ++jj) idx[(1 << i) + jj] = idx[jj] ^ b[i];
  };

  auto ld_block = [&](const float* src, float (&x)[R]) {  // R consecutive floats (16-byte aligned when R >= 4)
    if constexpr (R >= 4) {
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(src) + c4);
        x[4 * c4] = v.x; x[4 * c4 + 1] = v.y; x[4 * c4 + 2] = v.z; x[4 * c4 + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = __ldcg(src + r);
    }
  };
  auto st_block = [&](float* dst, const float (&x)[R]) {
    if constexpr (R >= 4) {
#pragma unroll
      for (int c4 = 0; c4 < R / 4; ++c4)
        reinterpret_cast<float4*>(dst)[c4] = make_float4(x[4 * c4], x[4 * c4 + 1], x[4 * c4 + 2], x[4 * c4 + 3]);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) dst[r] = x[r];
    }
  };
#define TW(i, r) Tb[(i) * Q + (r) * TT + t]

  const int slot = blockIdx.x;
  const size_t EQ = (size_t)cd.E * Q;
  float* const U = P.U + (size_t)slot * EQ;
  float* const W = P.W + (size_t)slot * EQ;
  uint8_t* const xh = P.xh + (size_t)slot * cd.N;
  constexpr float kInvQ = 1.0f / (float)Q;

#pragma unroll 1
  for (;;) {
    if (tid == 0) {
      sh_frame = atomicAdd(P.glob, 1);
      sh_events = 0;
    }
    __syncthreads();
    const int f = sh_frame;
    if (f >= P.frames) break;

    // ---- VARIABLE TO CHECK (and, for l >= 1, the TENTATIVE DECISION), one team per variable
    auto variable_phase = [&](int ell) {
      if (!in_team) return;
#pragma unroll 1
      for (int v = team; v < cd.N; v += P.teams) {
        const int e0 = P.v_ptr[v], d = P.v_ptr[v + 1] - e0;
        // p_v^0(x) for x = tR + r: the bit product, or the scaled pmf row
        float p0[R];
        if (P.pmf) {
          ld_block(P.pmf + ((size_t)f * cd.N + v) * Q + t * R, p0);
          float s = 0.0f;
#pragma unroll
          for (int r = 0; r < R; ++r) s += p0[r];
          s = team_sum(s);
          const float inv = s > 0.0f ? 1.0f / s : 0.0f;
#pragma unroll
          for (int r = 0; r < R; ++r) p0[r] *= inv;
        } else {
          float pz[MB], po[MB];
#pragma unroll
          for (int b = 0; b < MB; ++b) {
            const float L = P.llr[((size_t)f * cd.N + v) * MB + b];
            pz[b] = 1.0f / (1.0f + __expf(-L));  // Pr(b = 0 | L)
            po[b] = 1.0f / (1.0f + __expf(L));
          }
          float hi = 1.0f;
#pragma unroll
          for (int b = LR; b < MB; ++b) hi *= ((t >> (b - LR)) & 1) ? po[b] : pz[b];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            float pr = hi;
#pragma unroll
            for (int b = 0; b < LR; ++b) pr *= ((r >> b) & 1) ? po[b] : pz[b];
            p0[r] = pr;
          }
        }
        // w_i = WHT(W_i) / q, kept in the team's vectors (each thread its own block)
        if (ell > 0) {
          for (int i = 0; i < d; ++i) {
            float x[R];
            ld_block(W + (size_t)P.v_edges[e0 + i] * Q + t * R, x);
#pragma unroll
            for (int r = 0; r < R; ++r) x[r] = to_lin(x[r]);
            wht(x);
#pragma unroll
            for (int r = 0; r < R; ++r) TW(i, r) = x[r] * kInvQ;
          }
          // decision: mu = p0 prod_i w_i; M(0) and M(alpha^b) by signed sums
          float mu[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            float a = p0[r];
            if (d == 3) {  // the loop's order, unrolled
              a *= TW(0, r);
              a *= TW(1, r);
              a *= TW(2, r);
            } else {
              for (int i = 0; i < d; ++i) a *= TW(i, r);
            }
            mu[r] = a;
          }
          float Ms[MB + 1];
          {
            float s = 0.0f;
#pragma unroll
            for (int r = 0; r < R; ++r) s += mu[r];
            Ms[0] = s;
#pragma unroll
            for (int b = 0; b < MB; ++b) {
              float sb = 0.0f;
              if (b < LR) {
#pragma unroll
                for (int r = 0; r < R; ++r) sb += ((r >> b) & 1) ? -mu[r] : mu[r];
              } else {
                sb = ((t >> (b - LR)) & 1) ? -s : s;
              }
              Ms[b + 1] = sb;
            }
#pragma unroll
            for (int b = 0; b <= MB; ++b) Ms[b] = team_sum(Ms[b]);
          }
          int s0 = Ms[0] < 0.0f ? 1 : 0;
          int xv = 0;
#pragma unroll
          for (int b = 0; b < MB; ++b) xv |= ((Ms[b + 1] < 0.0f ? 1 : 0) ^ s0) << b;
          if constexpr (SOFT) {  // soft outputs: the decision again in fp64 (reading R22); its signs decide
            double md[MB + 1];
            general_decision_f64<MB, LR>(W, P.v_edges + e0, d, p0, t, tmask, md);
            s0 = md[0] < 0.0 ? 1 : 0;
            xv = 0;
#pragma unroll
            for (int b = 0; b < MB; ++b) xv |= ((md[b + 1] < 0.0 ? 1 : 0) ^ s0) << b;
            if (t == 0) {
#pragma unroll
              for (int b = 0; b < MB; ++b) P.soft_out[((size_t)f * cd.N + v) * MB + b] = soft_ratio(md[b + 1], md[0]);
            }
          }
          if (t == 0) xh[v] = (uint8_t)xv;
          if (P.post_out || P.map_out) {  // symbol posterior mu / sum mu and its argmax
            float tot = 0.0f, best = 0.0f;
            int bx = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const float a = fmaxf(mu[r], 0.0f);
              tot += a;
              if (r == 0 || a > best) { best = a; bx = t * R + r; }
            }
            tot = team_sum(tot);
#pragma unroll
            for (int off = TT / 2; off >= 1; off >>= 1) {
              const float ob = __shfl_xor_sync(tmask, best, off);
              const int ox = __shfl_xor_sync(tmask, bx, off);
              if (ob > best || (ob == best && ox < bx)) { best = ob; bx = ox; }
            }
            const float inv = tot > 0.0f ? 1.0f / tot : 0.0f;
            if (P.post_out) {
              float* dst = P.post_out + ((size_t)f * cd.N + v) * Q + t * R;
#pragma unroll
              for (int r = 0; r < R; ++r) dst[r] = fmaxf(mu[r], 0.0f) * inv;
            }
            if (P.map_out && t == 0) P.map_out[(size_t)f * cd.N + v] = (uint8_t)bx;
          }
        }
        // U_i = normalise(WHT(p0 prod_{i' != i} w_i'))
        for (int i = 0; i < d; ++i) {
          float x[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            float a = p0[r];
            if (ell > 0) {
              // the common small column weights unrolled (no loop and index test per entry; J3: 25% of the
              // stall samples sat on this product), others by the loop
              if (d == 3) {
                a *= TW(i == 0 ? 1 : 0, r) * TW(i == 2 ? 1 : 2, r);
              } else if (d == 2) {
                a *= TW(1 - i, r);
              } else if (d == 4) {
                const int i0 = i == 0 ? 1 : 0, i1 = i <= 1 ? 2 : 1, i2 = i <= 2 ? 3 : 2;
                a *= TW(i0, r) * TW(i1, r) * TW(i2, r);
              } else {
                for (int i2 = 0; i2 < d; ++i2)
                  if (i2 != i) a *= TW(i2, r);
              }
            }
            x[r] = a;
          }
          wht(x);
          float raw0 = x[0];
          if constexpr (TT > 1) raw0 = __shfl_sync(tmask, x[0], lane & ~(TT - 1));
          const bool neutral = !(raw0 > 0.0f);  // reading R10
          const float lg0 = lg2a(raw0);
          float pk[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            pk[r] = pack(lg0 - lg2a(fabsf(x[r])), __float_as_uint(x[r]));
            if (neutral) pk[r] = (t == 0 && r == 0) ? 0.0f : kFloor;
          }
          st_block(U + (size_t)P.v_edges[e0 + i] * Q + t * R, pk);
          if (neutral && t == 0) atomicAdd(&sh_events, 1);
        }
      }
    };

    variable_phase(0);  // INITIALIZATION: U = Lambda^0
    __syncthreads();
    int ell = 0, okv = 0;
#pragma unroll 1
    for (;;) {
      // ---- CHECK TO VARIABLE, one team per check
      if (in_team) {
#pragma unroll 1
        for (int c = team; c < cd.M; c += P.teams) {
          const int eb = c * cd.kpad;
          int kc = 0;
          while (kc < cd.kpad && cd.edges[eb + kc].var >= 0) ++kc;
          // TOT(w) = sum_k U_k(pi_k w) for my block of w
          float mag[R];
          uint32_t sg[R];
#pragma unroll
          for (int r = 0; r < R; ++r) { mag[r] = 0.0f; sg[r] = 0u; }
          // each U_k row is loaded coalesced (16-byte loads, the next one prefetched into registers) and staged
          // in the team's second vector in the interleaved layout z = tR + r -> r TT + t (conflict-free stores);
          // the permuted gather then reads shared memory instead of issuing scattered 4-byte L2 loads
          // (ncu, J3: 26% of the stall samples waited on those loads)
          float* const SG = Tb + Q;
          auto spos = [&](int z) { return ((z & (R - 1)) * TT) | (z >> LR); };  // a bit permutation: XOR-linear
          float nxt[R];
          if (kc > 0) ld_block(U + (size_t)eb * Q + t * R, nxt);
          for (int k = 0; k < kc; ++k) {
            const EdgeDev ed = cd.edges[eb + k];
#pragma unroll
            for (int r = 0; r < R; ++r) SG[r * TT + t] = nxt[r];
            if (k + 1 < kc) ld_block(U + (size_t)(eb + k + 1) * Q + t * R, nxt);
            uint8_t bp[8];
#pragma unroll
            for (int i = 0; i < MB; ++i) bp[i] = (uint8_t)spos(ed.pib[i]);
            int idx[R];
            perm_block(bp, idx);
            if constexpr (TT > 1) __syncwarp(tmask);
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const float u = SG[idx[r]];
              mag[r] += fabsf(u);
              sg[r] ^= __float_as_uint(u);
            }
            if constexpr (TT > 1) __syncwarp(tmask);
          }
          {
            // scalar stores: the padded team stride keeps Tb only 4-byte aligned
#pragma unroll
            for (int r = 0; r < R; ++r) Tb[t * R + r] = __uint_as_float(__float_as_uint(mag[r]) | (sg[r] & kSign));
          }
          if constexpr (TT > 1) __syncwarp(tmask);
          // W_j(z) = TOT(pi_j^-1 z) - U_j(z)
          for (int j = 0; j < kc; ++j) {
            const EdgeDev ed = cd.edges[eb + j];
            int idx[R];
            perm_block(ed.pinvb, idx);
            float uj[R], o[R];
            ld_block(U + (size_t)(eb + j) * Q + t * R, uj);
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const float tt = Tb[idx[r]];
              o[r] = pack(fabsf(tt) - fabsf(uj[r]), __float_as_uint(tt) ^ __float_as_uint(uj[r]));
            }
            st_block(W + (size_t)(eb + j) * Q + t * R, o);
          }
          if constexpr (TT > 1) __syncwarp(tmask);
        }
      }
      ++ell;
      __syncthreads();
      variable_phase(ell);
      __syncthreads();
      // ---- exact syndrome and the stopping rule
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
      if (P.events_out) P.events_out[f] = sh_events;
    }
    __syncthreads();
  }
#undef TW
}

}  // namespace nb
