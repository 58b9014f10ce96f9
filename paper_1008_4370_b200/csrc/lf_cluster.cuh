// lf_cluster.cuh -- cluster-per-frame kernel of the B200 Log-Fourier SP decoder (arXiv:1008.4370),
// separable variable node (NBLDPC_VN_SEPARABLE).
//
// One launch decodes the whole batch.  The grid is the number of thread-block clusters that fit on
// the GPU at once (persistent); each cluster of CS CTAs decodes one frame at a time, start to finish,
// then takes the next frame from a global counter.  CTA rank r of the cluster owns the check chunks
// r, r + CS, ... (checks_per_cta checks each, CPC * TPC threads).  One flooding iteration is one
// pass of every CTA over its chunks (the next chunk's messages bulk-copied into shared memory while the
// current one computes) followed by a hardware cluster barrier; the frame's two message buffers live in
// HBM (148 frames x 2 E 2^m x 4 bytes exceed the L2: every pass streams one set in and one out, DESIGN.md
// 7.6).  After the barrier each CTA folds its checks'
// syndrome bytes, ORs a "not a codeword" flag into rank 0's shared memory (DSMEM), and a second
// barrier makes the stopping decision cluster-uniform.
//
// Per check c and edge e = (c, v) with partner edge e' = (c', v) one pass computes
//   VARIABLE TO CHECK  raw = P_v^0 (*) Gamma^-1(W_e'), U_e = normalise(Gamma(raw)),
//       with P^0 = (x)_i (1, tanh(L_i/2)): the XOR-convolution is m butterfly stages
//       x(z) <- x(z) + t_i x(z ^ alpha^i)
//   TENTATIVE DECISION at v's deciding edge: M_v(z) = sum_y raw(y) W_e(z ^ y) at
//       z = 0, alpha^i (and H_cv alpha^i in paper mode); q = 256 hot path: split over
//       v's two edges (SPLITDEC below)
//   CHECK TO VARIABLE X_e(pi_e^-1 z) = U_e(z) (scatter), TOT(w) = sum_j X_j(w),
//       W_e(next)(z) = TOT(pi_e^-1 z) - U_e(z) (log-magnitudes add, signs XOR).
//
// Thread layout: an edge is owned by a team of TT = max(1, q/16) threads holding R = min(q, 16)
// entries each.  Phase A: thread t holds z = 16t + r (register bits = z bits 0..3); phase B (after
// one shared-memory transposition): z = jl | t << (8-m) | h << 4 with r = jl + 2^(8-m) h.
#pragma once
#include <assert.h>

#include <cuda_fp16.h>

#include "decoder.cuh"

// NB_BOUNDS_CHECK=1 (debug builds, `NBLDPC_DEFS=-DNB_BOUNDS_CHECK`): device asserts on every computed
// shared-memory index and global message row (compute-sanitizer is not available on the GPU pool)
#ifdef NB_BOUNDS_CHECK
#define NB_CHECK(cond) assert(cond)
#else
#define NB_CHECK(cond) ((void)0)
#endif

namespace nb {

struct ClusterParams {
  CodeDev code;
  WorkDev ws;          // slots = clusters (decode) or frames (step mode)
  int chunks;          // G = ceil(M / checks_per_cta)
  int checks_per_cta;  // CPC
  int tpc;             // threads per check (power of two)
  int step_mode;       // 1: nbldpc_step (frames 0..F-1 at iteration step_iter, one pass each)
  int step_iter;
  int rec_per_cta;     // compact edge records per CTA in shared memory (max over ranks)
  float* u_out;        // step mode: optional U dump [F][E][q]
};

// compact per-edge record kept in shared memory for the CTA's chunks (8 bytes); the Fourier
// permutation images of h come from a per-field table (CodeDev::pinv_tab, copied to shared memory)
struct EdgeRec {
  int32_t partner_a;  // partner edge << 9 | h of the partner edge << 1 | is_a ; -1: padding slot
  uint32_t var_h;     // variable << 8 | h_cv, bit 31: kind_a (q = 256 split decision)
};

// alignment of the cluster kernels' dynamic shared memory: one message row (q floats, q <= 256)
constexpr uint32_t kSmemAlignPad = 1024;

template <int MB>
struct CCfg {
  static constexpr int Q = 1 << MB;
  static constexpr int LR = MB < 4 ? MB : 4;
  static constexpr int R = 1 << LR;                 // entries per thread
  static constexpr int TT = Q / R;                  // threads per edge team
  static constexpr int LJ = MB >= 4 ? 8 - MB : 0;   // phase-B low register bits (TT > 1)
  static constexpr int V = 1 << LJ;                 // phase-B contiguous run (floats)
  static constexpr int CH = R >= 4 ? R / 4 : 1;     // 16-byte chunks per thread
  static constexpr int QS = Q < 4 ? 4 : Q;          // row stride (floats) of a staged message
  static constexpr bool BULK = Q >= 4;  // message rows are whole 16-byte chunks: bulk-copied
  // channel-term row: prefetched into registers for one- or two-thread teams (measured: C5 651 -> 546
  // ns per frame-iteration), bulk-copied beside the message rows for wider teams (C3 902 vs 1017 ns)
#ifndef NB_THREG_MAX_TT
#define NB_THREG_MAX_TT 2
#endif
  static constexpr bool THREG = TT <= NB_THREG_MAX_TT;
  static constexpr int THW = THREG ? 0 : 8;          // channel-term floats per team and stage buffer
  // shared memory per team (floats): message row x 2 stage buffers (+ channel terms x 2); the consumed
  // row doubles as the transposition buffer, the decision buffer and the check node's scatter target
#ifndef NB_NSTAGE
#define NB_NSTAGE 2
#endif
  static constexpr int NS = NB_NSTAGE;               // stage buffers per group (chunks in flight + 1)
  // q >= 64: one more row per team, the work row of the F32 kernels (transposition, decision buffer, check-node
  // scatter): the staged rows are then only read by the generic proxy, so no proxy fence and no end-of-chunk
  // barrier is needed before their next bulk fill
  static constexpr int NW = MB >= 6 ? 1 : 0;
  static constexpr int RB = NS + NW;                 // row buffers per team
  static constexpr int TEAMW = RB * QS + NS * THW;
};

// Message storage ("reader-ordered rows"): row r holds the message CONSUMED by edge slot r, i.e. the
// check-to-variable message of r's partner edge, so that a chunk's variable-node inputs are one
// contiguous block (one bulk copy per group).  Entry z of row r sits at mpos(z, r): the 16-byte chunks
// are XOR-swizzled by the block index and by low row bits, so that the phase-A reads of the staged
// rows (rows at a stride of q floats) are bank-conflict free.
template <int MB>
__host__ __device__ __forceinline__ int mpos(int z, int row) {
  constexpr int Q = 1 << MB;
  if constexpr (MB == 8) {
    // q = 256: 16-byte chunk c (= (z >> 2) & 3) of block b (= z >> 4) at chunk 16 c + (b ^ c).  A thread holding a
    // block (phase A) writes or reads it as four 16-byte chunks, and the 16 blocks' chunk c are one contiguous
    // 256-byte run (coalesced stores, conflict-free 16-byte shared loads); a phase-B lane (z = t | h << 4) reads
    // word 64 c + 4 (h ^ c) + (t & 3): its team's 16 lanes hit 16 distinct banks
    const int b = z >> 4, c = (z >> 2) & 3;
    (void)row;
    return (c << 6) | ((b ^ c) << 2) | (z & 3);
  } else if constexpr (MB >= 5) {
    constexpr int TT = Q / 16;
    const int b = z >> 4, c = (z >> 2) & 3;
    const int f = TT <= 4 ? (row & (8 / TT - 1)) : 0;
    return (b << 4) | (((c ^ b ^ (b >> 2) ^ f) & 3) << 2) | (z & 3);
  } else if constexpr (MB >= 2) {
    constexpr int CH = Q / 4;                           // chunks per row (1, 2, 4)
    const int key = (row / (8 / CH)) & (CH - 1);
    return ((((z >> 2) ^ key) & (CH - 1)) << 2) | (z & 3);
  } else {
    return z;
  }
}

// F16 message rows (NBLDPC_MSG_F16, q >= 8): entry z of row r at mposh(z, r), in 16-byte units of 8
// halves XOR-swizzled by the row's position in its 128-byte line (the phase-A unit reads of the rows of
// a quarter warp hit distinct bank quads), and for rows of >= 16 units by the unit's own bit 3
template <int MB>
__host__ __device__ __forceinline__ int mposh(int z, int row) {
  constexpr int U = (1 << MB) / 8;  // units per row
  int unit = z >> 3;
  if constexpr (U >= 16) unit ^= (unit >> 3) & 1;
  const int key = U >= 8 ? row : (row * U) >> 3;
  return ((unit ^ (key & (U - 1))) << 3) | (z & 7);
}
#ifdef NB_MSG16_FIXED
// experiment: sign | 15-bit fixed-point magnitude with step 2^-9 (saturating at 64)
__device__ __forceinline__ float fx2f(uint32_t h) {
  return __uint_as_float(__float_as_uint((float)(h & 0x7FFFu) * (1.0f / 512.0f)) | ((h & 0x8000u) << 16));
}
__device__ __forceinline__ uint32_t f2fx(float a) {
  const uint32_t m = (uint32_t)fminf(rintf(fabsf(a) * 512.0f), 32767.0f);
  return m | ((__float_as_uint(a) >> 16) & 0x8000u);
}
__device__ __forceinline__ float2 h2f2(uint32_t v) { return make_float2(fx2f(v & 0xFFFFu), fx2f(v >> 16)); }
__device__ __forceinline__ uint32_t f22h(float a, float b) { return f2fx(a) | (f2fx(b) << 16); }
#define NB_F2H1(a) __ushort_as_half((unsigned short)f2fx(a))
#else
__device__ __forceinline__ float2 h2f2(uint32_t v) { return __half22float2(*reinterpret_cast<const __half2*>(&v)); }
__device__ __forceinline__ uint32_t f22h(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
#define NB_F2H1(a) __float2half_rn(a)
#endif

__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* mb, uint32_t tx) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(mb)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(mb)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mb))
               : "memory");
}

// W_e rows are written once and next read a whole pass later (never from L2: the in-flight frames' message sets
// exceed it): NB_STCS stores them evict-first so that the L2 keeps the rows that are read twice
// within a pass (as a partner row and as the decision's own row)
__device__ __forceinline__ void st_w4(float* p, float4 v) {
#ifdef NB_STCS
  __stcs(reinterpret_cast<float4*>(p), v);
#else
  *reinterpret_cast<float4*>(p) = v;
#endif
}

// NB_STCS >= 2: the decision's own-row copy with an L2 evict-first policy (the row's other read is the partner's
// block copy, which keeps the default policy)
__device__ __forceinline__ void bulk_g2s_ef(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
#if defined(NB_STCS) && NB_STCS >= 2
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mb)), "l"(pol)
               : "memory");
#else
  bulk_g2s(dst, src, bytes, mb);
#endif
}

// the same on shared-window addresses computed once (no generic-to-shared conversion in the loop)
__device__ __forceinline__ void mbar_arrive_tx_s(uint32_t mb, uint32_t tx) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(mb), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t mb, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(mb),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mb)
               : "memory");
}

// transposition layout: 16-byte chunk c of block b at chunk c ^ ((b ^ (b >> 2)) & 3): the phase-A
// 128-bit stores (8 threads per quarter warp) and the phase-B reads are bank-conflict free
__device__ __forceinline__ int tpos(int z) {
  return (z & ~15) | ((((z >> 2) ^ (z >> 4) ^ (z >> 6)) & 3) << 2) | (z & 3);
}

// decision buffer: row tb (16 floats) holds D at the phase-B coordinates (tb, rb); its 16-byte chunks
// are XOR-swizzled by (tb >> 1) & 3 so that 8 consecutive rows read in one LDS.128 hit 8 bank quads
__device__ __forceinline__ int db_word(int tb, int rb) { return 16 * tb + ((((rb >> 2) ^ (tb >> 1)) & 3) << 2) + (rb & 3); }

// Sum NV per-lane values over the TT lanes of a team by recursive halving (reduce-scatter): each level
// exchanges half of the remaining slots with the partner lane.  Returns the OR over the team of
// [total < 0] << index; lane-local slot k then holds the total of value index off + k (k < nfin).
template <int NV, int TT>
__device__ __forceinline__ uint32_t team_sign_bits(float (&v)[NV], int lane, int& off, int& nfin) {
  int n = NV, nv = NV;  // n: slots (compile-time sequence), nv: this lane's slots holding real values
  off = 0;
#pragma unroll
  for (int o = TT / 2; o >= 1; o >>= 1) {
    const int h = (n + 1) / 2;
    const bool upper = (lane & o) != 0;
    nv = upper ? (nv > h ? nv - h : 0) : (nv < h ? nv : h);
#pragma unroll
    for (int k = 0; k < (NV + 1) / 2; ++k) {
      if (k < h) {
        const float lo = v[k];
        const float hi = (h + k < n) ? v[h + k] : 0.0f;
        const float send = upper ? lo : hi;
        const float keep = upper ? hi : lo;
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    if (upper) off += h;
    n = h;
  }
  nfin = nv;
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < NV; ++k)
    if (k < n && k < nv && v[k] < 0.0f) bits |= 1u << (off + k);
  const unsigned tmask = (TT >= 32) ? 0xffffffffu : (((1u << TT) - 1u) << (lane & ~(TT - 1) & 31));
  return __reduce_or_sync(tmask, bits);
}

// The five totals of the split decision (q = 256: two 16-lane teams per warp) by recursive halving as in
// team_sign_bits; the totals of values 0..4 end in team lanes 0, 2, 4, 8 and 10, whose sign bits are collected by
// one warp-wide ballot (no per-team REDUX, which the two teams' masks serialise)
__device__ __forceinline__ uint32_t split_sign_bits(float (&v)[5], int lane) {
  int off = 0, nfin = 0;
  constexpr int NV = 5, TT = 16;
  int n = NV, nv = NV;
#pragma unroll
  for (int o = TT / 2; o >= 1; o >>= 1) {
    const int h = (n + 1) / 2;
    const bool upper = (lane & o) != 0;
    nv = upper ? (nv > h ? nv - h : 0) : (nv < h ? nv : h);
#pragma unroll
    for (int k = 0; k < (NV + 1) / 2; ++k) {
      if (k < h) {
        const float lo = v[k];
        const float hi = (h + k < n) ? v[h + k] : 0.0f;
        const float send = upper ? lo : hi;
        const float keep = upper ? hi : lo;
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    if (upper) off += h;
    n = h;
  }
  nfin = nv;
  (void)off;
  const uint32_t bal = __ballot_sync(0xffffffffu, nfin > 0 && v[0] < 0.0f) >> (lane & 16);
  return (bal & 1u) | ((bal >> 1) & 2u) | ((bal >> 2) & 4u) | ((bal >> 5) & 8u) | ((bal >> 6) & 16u);
}

template <int CH>
__device__ __forceinline__ int cswz(int c, int key) { return c ^ (key & (CH - 1)); }

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nrank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (a shared variable of this CTA) in CTA `rank`
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsmem_st(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ int dsmem_ld(uint32_t addr) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void dsmem_or(uint32_t addr, int v) {
  asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// TOT(w) = sum_j X_j(w) over the thread's WPT w's (stride TT*JPT) and JPT teams (stride TEAM words)
template <int R, int JPT, int TT, int TEAM>
__device__ __forceinline__ void tot_sum(const float* smem, int gbase, float* TOT, int wgrp, int split, int pck,
                                        bool cvalid, int ix = 0) {
  // ix: XOR on the w-group index i (the odd check of a warp holding two checks takes its w's in the order
  // i ^ 1, so the two checks' loads and TOT stores fall in different bank halves)
  constexpr int WPT = R / JPT;
  const float* g = smem + gbase;
  // one w split over lanes (WPT == 1): the lanes of a w read rows JPT apart, which for TEAM * JPT = 0 mod 32
  // words are the same banks -- so odd split lanes take the rows in the order jj ^ 1 (a different bank half
  // when TEAM = 16; the sum does not depend on the order up to rounding)
  const int jx = (WPT == 1 && TEAM % 32 != 0) ? (pck & 1) : 0;
#pragma unroll
  for (int i = 0; i < WPT; ++i) {
    float mag = 0.0f;
    uint32_t sg = 0;
    const int iw = WPT > 1 ? (i ^ ix) : i;
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) {
      const float v = g[((JPT > 1 ? jj ^ jx : jj)) * TEAM + iw * TT * JPT];
      mag += fabsf(v);
      sg ^= __float_as_uint(v);
    }
    if constexpr (WPT == 1) {
      for (int off = 1; off < split; off <<= 1) {
        mag += __shfl_xor_sync(0xffffffffu, mag, off);
        sg ^= __shfl_xor_sync(0xffffffffu, sg, off);
      }
    }
    if (cvalid && (WPT > 1 || (pck & (split - 1)) == 0))
      TOT[wgrp + TT * JPT * iw] = __uint_as_float(__float_as_uint(mag) | (sg & kSign));
  }
}

// TOT for one-thread teams (q <= 16) from the lane-major scatter buffer xs[w][32] (X_j(w) of the team in
// lane j of the warp at xs[32 w + j]): the scatter of every lane hits its own bank, and here the threads of
// a w read the check's lanes in an order rotated by w, so that every load instruction covers 32 banks.
// c0: the check's first lane in the warp; the rest as tot_sum.
template <int R, int JPT>
__device__ __forceinline__ void tot_sum_lm(const float* xs, int c0, float* TOT, int wgrp, int split, int pck,
                                           bool cvalid) {
  constexpr int WPT = R / JPT;
  const int jb = c0 + (pck % split) * JPT;
#pragma unroll
  for (int i = 0; i < WPT; ++i) {
    const int w = wgrp + JPT * i;
    const float* g = xs + 32 * w + jb;
    NB_CHECK(w < R * (32 / (JPT * split) > 0 ? 32 : 32) && jb + JPT <= 32);
    float mag = 0.0f;
    uint32_t sg = 0;
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) {
      const float v = g[(jj + wgrp) & (JPT - 1)];
      mag += fabsf(v);
      sg ^= __float_as_uint(v);
    }
    if constexpr (WPT == 1) {
      for (int off = 1; off < split; off <<= 1) {
        mag += __shfl_xor_sync(0xffffffffu, mag, off);
        sg ^= __shfl_xor_sync(0xffffffffu, sg, off);
      }
    }
    if (cvalid && (WPT > 1 || (pck & (split - 1)) == 0)) TOT[w] = __uint_as_float(__float_as_uint(mag) | (sg & kSign));
  }
}

// LIN: the leave-one-out PRODUCTS of the check node on linear messages: thread pck owns
// WPT w's x JPT teams of its check; each X_j(w) is replaced in place by prod_{j' != j} X_j'(w) (prefix and
// suffix products in registers; when one w is split over SPLIT lanes the other lanes' products come by a
// butterfly of exclusive products).  No division: a zero factor stays exact.
template <int R, int JPT, int TT, int TEAM>
__device__ __forceinline__ void tot_prod(float* smem, int gbase, int split, bool cvalid) {
  constexpr int WPT = R / JPT;
  float* g = smem + gbase;
#pragma unroll
  for (int i = 0; i < WPT; ++i) {
    float v[JPT], ex[JPT];
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) v[jj] = g[jj * TEAM + i * TT * JPT];
    if constexpr (JPT >= 4) {
      if (split == 1) {
        // packed (FMUL2) form: the two halves' prefix products side by side, then their suffix products started
        // from the other half's total, so (ex[k], ex[k + H]) = (prefix_A, prefix_B) * (suffix_A * total_B,
        // suffix_B * total_A): 3 H FMUL2 instead of 3 JPT FMUL, the same products reassociated
        constexpr int H = JPT / 2;
        float2 pp[H];
        float2 c = make_float2(1.0f, 1.0f);
#pragma unroll
        for (int k = 0; k < H; ++k) {
          pp[k] = c;
          c = __fmul2_rn(c, make_float2(v[k], v[k + H]));
        }
        float2 sc = make_float2(c.y, c.x);  // (total_B, total_A)
#pragma unroll
        for (int k = H - 1; k >= 0; --k) {
          const float2 e2 = __fmul2_rn(pp[k], sc);
          ex[k] = e2.x;
          ex[k + H] = e2.y;
          sc = __fmul2_rn(sc, make_float2(v[k], v[k + H]));
        }
        if (cvalid) {
#pragma unroll
          for (int jj = 0; jj < JPT; ++jj) g[jj * TEAM + i * TT * JPT] = ex[jj];
        }
        continue;
      }
    }
    float pre = 1.0f;
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) {
      ex[jj] = pre;
      pre *= v[jj];
    }
    float suf = 1.0f;
#pragma unroll
    for (int jj = JPT - 1; jj >= 0; --jj) {
      ex[jj] *= suf;
      suf *= v[jj];
    }
    if constexpr (WPT == 1) {
      float other = 1.0f, incl = pre;  // the product of the other split lanes' factors
      for (int off = 1; off < split; off <<= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, incl, off);
        other *= o;
        incl *= o;
      }
#pragma unroll
      for (int jj = 0; jj < JPT; ++jj) ex[jj] *= other;
    }
    if (cvalid) {
#pragma unroll
      for (int jj = 0; jj < JPT; ++jj) g[jj * TEAM + i * TT * JPT] = ex[jj];
    }
  }
}

// LIN at q = 256 (two teams per warp): the pair of a warp's two team rows holds X_{2p}(w) and X_{2p+1}(w)
// interleaved at 2w and 2w + 1, so the two teams' scatters use the even and the odd banks (measured
// row-major: 2.9 wavefronts per scatter instruction); the column threads then read j in the order jj ^ flip
// (flip: the upper half-warp, or the odd split lane) so that their loads still cover 32 banks.
template <int R, int JPT, int TT, int QS>
__device__ __forceinline__ void tot_prod_il(float* rows, int wgrp, int jbase, int flip, int split, bool cvalid) {
  constexpr int WPT = R / JPT;
#pragma unroll
  for (int i = 0; i < WPT; ++i) {
    const int w = wgrp + TT * JPT * i;
    float v[JPT], ex[JPT];
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) {
      const int j = jbase + (jj ^ flip);
      v[jj] = rows[(j & ~1) * QS + 2 * w + (j & 1)];
    }
    float pre = 1.0f;
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) {
      ex[jj] = pre;
      pre *= v[jj];
    }
    float suf = 1.0f;
#pragma unroll
    for (int jj = JPT - 1; jj >= 0; --jj) {
      ex[jj] *= suf;
      suf *= v[jj];
    }
    if constexpr (WPT == 1) {
      float other = 1.0f, incl = pre;
      for (int off = 1; off < split; off <<= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, incl, off);
        other *= o;
        incl *= o;
      }
#pragma unroll
      for (int jj = 0; jj < JPT; ++jj) ex[jj] *= other;
    }
    if (cvalid) {
#pragma unroll
      for (int jj = 0; jj < JPT; ++jj) {
        const int j = jbase + (jj ^ flip);
        rows[(j & ~1) * QS + 2 * w + (j & 1)] = ex[jj];
      }
    }
  }
}

// linear message entry -> the packed (sign | -log2|x|) format of nbldpc_step (0 -> the zero, 200)
__device__ __forceinline__ float lin_to_packed(float u) {
  const float mag = fminf(fmaxf(-lg2a(fabsf(u)), 0.0f), kFloor);
  return __uint_as_float(__float_as_uint(mag) | (mag >= kFloor ? 0u : (__float_as_uint(u) & kSign)));
}

// One Walsh-Hadamard butterfly stage (u, w) -> (u + w, u - w) on register bit I of a thread's R entries.
template <int R, int I>
__device__ __forceinline__ void wht_reg(float (&x)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (!(r & (1 << I))) {
      const float u = x[r], w = x[r | (1 << I)];
      x[r] = u + w;
      x[r | (1 << I)] = u - w;
    }
}
// The full WHT of a team's vector held in the phase-B coordinates zr (pmf input):
// every register bit, then the z bits LJ..3 that index the team's lanes by shuffles.
template <int MB, int R, int LR, int LJ, int TT>
__device__ __forceinline__ void wht_phase_b(float (&x)[R], int t) {
  if constexpr (LR > 0) wht_reg<R, 0>(x);
  if constexpr (LR > 1) wht_reg<R, 1>(x);
  if constexpr (LR > 2) wht_reg<R, 2>(x);
  if constexpr (LR > 3) wht_reg<R, 3>(x);
  if constexpr (TT > 1) {
#pragma unroll
    for (int k = 0; k < 4 - LJ; ++k) {
      const int off = 1 << k;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float o = __shfl_xor_sync(0xffffffffu, x[r], off);
        x[r] = (t & off) ? o - x[r] : x[r] + o;
      }
    }
  }
}
// position of entry z of a normalised pmf row in the per-slot buffer: thread t of the team reads its R
// phase-B entries zr(t, r) as one contiguous run at t R + r
template <int MB>
__device__ __forceinline__ int ppos(int z) {
  if constexpr (MB > 4) {
    constexpr int LJ = 8 - MB, TT = 1 << (MB - 4), R = 16;
    const int jl = z & ((1 << LJ) - 1), tt = (z >> LJ) & (TT - 1), h = z >> 4;
    return tt * R + (jl | (h << LJ));
  } else {
    return z;
  }
}

// PMF = true: nbldpc_decode_pmf.  The channel prior is a general symbol pmf p_v, so P_v^0 is not a
// tensor product; the variable node runs in the probability domain instead (XOR-convolution
// theorem): raw = P^0 (*) W_e' = WHT(p_v . WHT(W_e')) / q -- 2m butterfly stages and a product per
// entry (the factor q cancels in the normalisation).
// F16 = true: messages stored in HBM / L2 as IEEE half (sign | -log2|x|), the paper's reduced-precision
// motivation: half the message bytes.  The staged rows are halves;
// a float work row per team takes the transposition, the decision's D and the check node's scatter.
// KP > 0: the code's edge-slot stride kpad, known at compile time with full CTAs (NTHR threads,
// NTHR / (KP TT) checks each), so that the chunk geometry constant-folds; 0: taken from P.
// SYM = true: also the symbol-level decision at every iteration, written to the
// frame's output rows: mu_v = WHT(raw) . WHT(W_e) in the phase-B coordinates (M_v = raw (*) W_e).
// SOFT = true: soft outputs (decode soft_out, nbldpc_step): the decision in fp64 (decision_f64, reading
// R22); a separate instantiation so that the plain hot-path kernels carry none of its registers.
template <int MB, int NTHR, bool PMF = false, bool F16 = false, int KP = 0, bool SYM = false, bool SOFT = false>
#ifndef NB_CLUSTER_MINB
#define NB_CLUSTER_MINB 2
#endif
__global__ void __launch_bounds__(NTHR, (NTHR <= 256 ? NB_CLUSTER_MINB : 1)) lf_cluster_kernel(ClusterParams P) {
  using C = CCfg<MB>;
  constexpr int Q = C::Q, R = C::R, TT = C::TT, LR = C::LR, LJ = C::LJ, CH = C::CH;
  extern __shared__ __align__(1024) float smem_raw[];
  // LIN (q >= 128): the dynamic region starts on a 1 KB (message-row) boundary of the shared window (the
  // declared alignment; checked once below), so that a team row's shared address ORs with an entry's byte
  // offset -- the check node's scatter / read-back addresses are then the XOR chain itself
  float* const smem = smem_raw;
  __shared__ int sh_frame, sh_flag[2], sh_bad;
  // lazy decision (SPLITDEC): sh_skip = stamp of the pass in which some probe check of the cluster was
  // proven unsatisfied (the pass cannot stop the frame, so the rest of its tentative decision is skipped);
  // sh_pc[team] = the probe chunk's tag << 8 | h_e x_v of the team's edge
  __shared__ int sh_skip;
  __shared__ uint32_t sh_pc[64];
  __shared__ __align__(8) uint64_t sh_mbar[8 * C::NS];  // [group][buffer]: the group's teams arrive, bulk copies complete_tx
  __shared__ __align__(8) uint64_t sh_cbar[8];  // SPLITDEC: [group] "every warp of the check has scattered" (one arrival per warp)

  if (MB >= 7 && (smem_u32(smem_raw) & (kSmemAlignPad - 1)) != 0) __trap();  // the row alignment LIN relies on
  const CodeDev& cd = P.code;
  const WorkDev& ws = P.ws;
  const int tid = threadIdx.x;
  const int nthr = KP ? NTHR : (int)blockDim.x;
  const int lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t csz = cluster_nrank();
  const int clid = (int)cluster_id();
  const int ncl = (int)cluster_count();
  const int KPAD = KP ? KP : cd.kpad;  // edge-slot stride per check
  const int TPC = KP ? KP * TT : P.tpc;
  const int CPC = KP ? NTHR / (KP * TT) : P.checks_per_cta;
  const int KT = TPC / TT;                       // teams per check (incl. padding teams)
  const int nch = ((int)P.chunks - (int)rank + (int)csz - 1) / (int)csz;  // my chunks: rank + k*csz
  // independent groups of GT = max(32, TPC) threads (a warp, or one check): each runs its own stage
  // pipeline (mbarriers) over the chunks, so warps of a CTA never wait for one another inside a pass
  const int GT = TPC > 32 ? TPC : 32;
  const int ngrp = nthr / GT;
  const int grp = threadIdx.x / GT;
  constexpr int NS = C::NS;
  uint64_t* const gmbar = &sh_mbar[NS * grp];
  auto group_sync = [&]() {
    if (GT == 32) {
      __syncwarp();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(GT) : "memory");
    }
  };

  // ---- my position in a chunk (fixed)
  const int lc = tid / TPC;
  const int pck = tid - lc * TPC;
  const int j = pck / TT;
  const int t = pck & (TT - 1);
  const bool in_check = lc < CPC;
  const int team = tid / TT;
  const int nteams = nthr / TT;
  // shared memory: per group [2 stage buffers][GT/TT team rows][QS] | TH [2][nteams][8] | TOT | PT | ...
  const int TG = GT / TT;                        // teams per group
  const int CPG = GT / TPC;                      // checks per group
  const int GBLK = TG * C::QS;                   // one stage buffer of a group (floats)
  float* const GST = smem + grp * C::RB * GBLK;  // the group's stage buffers (+ its work rows, q >= 128)
  const int trow = team - grp * TG;              // my team's row within a group stage buffer
  // F16: the group's region holds two stage buffers of half rows (GBLKH floats each) and the float
  // work rows (GBLK floats), the same bytes as two float stage buffers
  const int GBLKH = GBLK / 2;
  float* const WK = F16 ? GST + NS * GBLKH + trow * C::QS : nullptr;  // my work row
  float* const THB = smem + nteams * C::RB * C::QS + team * 8;  // + b * nteams * 8 (wide teams only)
  float* const TOT = smem + nteams * C::TEAMW + lc * Q;
  uint64_t* const PT = reinterpret_cast<uint64_t*>(smem + nteams * C::TEAMW + CPC * Q);  // [q] pi_h^-1 images
  EdgeRec* const recs = reinterpret_cast<EdgeRec*>(PT + Q);
  uint8_t* const GL = reinterpret_cast<uint8_t*>(recs + P.rec_per_cta);  // [q] log_alpha
  uint8_t* const GE = GL + Q;                                            // [2q] alpha^i
  // pmf input, one-thread teams (q <= 16): the teams' pmf rows staged one chunk ahead beside the message
  // rows ([NS][nteams][q], LDGSTS on the stage mbarrier), instead of an L2 load at the chunk's start
  // (ncu, C5 pmf: 33% of the stall samples waited on that load)
  constexpr bool PSTAGE = PMF && TT == 1 && Q >= 4;
  float* const PB = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(GL) + 3 * Q + 15) & ~(uintptr_t)15);
  // SPLITDEC (q = 256): each team's own message W_e bulk-copied one chunk ahead ([NS][nteams] rows of q + 16
  // words after the GF tables, on the stage mbarrier) instead of a register load at the chunk's start (ncu: the
  // decision waited on that load) -- the region of PB, which only one-thread teams use
  // (offset arithmetic on smem, not an integer round trip, so that the compiler keeps shared-space accesses)
  float* const WE = smem + ((((reinterpret_cast<const char*>(GL) - reinterpret_cast<const char*>(smem)) + 3 * Q + 15) & ~15) >> 2);

  // TOT(w) gather offsets: thread pck owns WPT w's x JPT teams of its check (R terms, natural X)
  const int SPLIT = KT > R ? KT / R : 1;
  const int JPT = KT / SPLIT;
  const int wgrp = pck / SPLIT;
  const int jbase = (pck % SPLIT) * JPT;
  const int tix = (TPC == 16) ? (lc & 1) : 0;  // tot_sum's i rotation for the odd check of a warp
  const int gbase = in_check ? (int)(GST - smem) + (F16 ? NS * GBLKH : 0) + ((lc - grp * CPG) * KT + jbase) * C::QS + wgrp
                             : 0;  // + buf * GBLK (F32: the consumed stage rows; F16: the work rows)
  // my phase-B z's
  int zr[R];
#pragma unroll
  for (int r = 0; r < R; ++r) zr[r] = TT > 1 ? ((r & ((1 << LJ) - 1)) | (t << LJ) | ((r >> LJ) << 4)) : r;

  // ---- compact edge records of my chunks -> shared memory (once)
  for (int i = tid; i < nch * CPC * KT; i += nthr) {
    const int kc = i / (CPC * KT), rem = i - kc * CPC * KT;
    const int l = rem / KT, jj = rem - l * KT;
    const int c = ((int)rank + kc * (int)csz) * CPC + l;
    EdgeRec rr{-1, 0};
    if (c < cd.M && jj < cd.k_max) {
      const EdgeDev* ep = cd.edges + (size_t)c * KPAD + jj;
      if (ep->var >= 0) {
        rr.partner_a = (ep->partner << 9) | ((int)cd.edges[ep->partner].h << 1) | (ep->is_a ? 1 : 0);
        rr.var_h = ((uint32_t)ep->var << 8) | ep->h | ((uint32_t)(ep->kind_a ? 1 : 0) << 31);
      }
    }
    recs[i] = rr;
  }
  for (int h = tid; h < Q; h += nthr) {
    PT[h] = cd.pinv_tab[h];
    GL[h] = cd.gf_log[h];
  }
  for (int i = tid; i < 2 * Q - 1; i += nthr) GE[i] = cd.gf_exp[i < 2 * (Q - 1) + 1 ? i : 0];
  if (tid == 0) {
    sh_flag[0] = 0;
    sh_flag[1] = 0;
    sh_skip = -1;
    for (int gg = 0; gg < ngrp; ++gg) {
      for (int b = 0; b < NS; ++b) mbar_init(&sh_mbar[NS * gg + b], (uint32_t)(GT / TT));
      mbar_init(&sh_cbar[gg], (uint32_t)(GT / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_sync_all();
  uint32_t mb_parity = 0;
  uint32_t cb_parity = 0;  // SPLITDEC: parity of the next completion of my group's sh_cbar  // bit b: parity of the next completion of stage buffer b  // every CTA of the cluster has started before any DSMEM access

  const CallDev* call = ws.call;
  const int max_iters = call->max_iters;
  const int mode = call->mode;
  constexpr bool want_soft = SOFT;  // soft outputs are requested exactly when the host launches a SOFT kernel
  // LIN: messages stored as linear fp32 values -- the F32 hot path at q >= 128, where dropping
  // the ex2 / lg2 / sign work of the log format outweighs the check node's extra write-back (measured: C3
  // -2.5%, C4 -2% time; C2 +5%, C5 +12%, so q <= 64 keeps the log format); the F16 format and the
  // soft-output kernels (whose fp64 decision needs the exact log-magnitudes) always keep the packed log format
  constexpr bool LIN = !F16 && !SOFT && MB >= 7;
  // one-thread teams (q <= 16): the check node's scatter goes to the group's consumed stage buffer in a
  // lane-major layout xs[w][lane] (conflict-free; ncu, C5: the row-major scatter replayed 3.6x)
#ifdef NB_LANEMAJOR_F16
  constexpr bool LANEMAJOR = TT == 1 && Q >= 2;
#else
  constexpr bool LANEMAJOR = TT == 1 && !F16 && Q >= 2;
#endif
  // the interleaved team pairs of tot_prod_il: measured neutral on C4 (conflict replays -14%, instructions
  // +7%), kept off; NB_PAIRIL=1 builds it
#ifdef NB_PAIRIL
  constexpr bool PAIRIL = LIN && TT == 16;
#else
  constexpr bool PAIRIL = false;
#endif
  // SPLITDEC (q = 256 hot path, exact syndrome): the tentative decision is split over the variable's two
  // edge teams instead of being computed whole by one of them.  M_v = raw_a (*) W_a = raw_b (*) W_b
  // (raw_e = P^0 (*) W_partner(e)), so the is_a team evaluates M_v(0) and M_v(alpha^i),
  // i = 4..7 (its phase-B register bits: W_e transposed into phase B), the other team M_v(0) and i = 0..3
  // (its phase-A register bits: raw_e transposed into phase A, W_e straight from its phase-A load) -- every
  // point is an in-thread FFMA2 dot product, no partner-row reads, and every team does the same ~half
  // decision (no deciding / idle imbalance at the check barriers).  Each team stores its nibble of the
  // fast bit rule in con[e]; at the end of the pass x_v = the two nibbles and each CTA forms its checks'
  // exact syndromes from them.  The paper syndrome (mode 1) keeps the whole decision.
  constexpr bool SPLITDEC_CT = LIN && TT == 16 && !SYM && !SOFT;
  // F32 kernels at q >= 64: the transposition, decision buffer and scatter go to a per-team work row (CCfg::NW)
  // (the q = 64 symbol-output variant keeps its registers: no work rows -- C2 symbol outputs 3.71e9 -> 4.44e9;
  // the q >= 128 linear-format check node's read-back assumes separate work rows, so SYM keeps them there)
  constexpr bool WROW = !F16 && MB >= 6 && !(SYM && MB < 7);
  const bool split = SPLITDEC_CT && mode == 0;
  const int step = P.step_mode;
  const size_t EQ = (size_t)cd.E * Q;
  const uint32_t flag0 = dsmem_addr(&sh_flag[0], 0), flag1 = dsmem_addr(&sh_flag[1], 0);

  int round = 0;
#pragma unroll 1
  for (;;) {
    // ---- next frame for the cluster
    int f, slot;
    if (step) {
      f = clid + round * ncl;
      slot = f;
      if (f >= call->frames) break;
    } else {
      if (rank == 0 && tid == 0) {
        const int nf = atomicAdd(&ws.glob[0], 1);
        if (call->chunk_flags != nullptr && nf < call->frames) {
          // end-to-end decode: this frame's LLRs are still being copied in (nbldpc_decode_host
          // overlaps the host-to-device copy with the decode); the copy stream raises the flag
          const int32_t* fl = call->chunk_flags + nf / call->chunk_frames;
          int v;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
            if (v != 0) break;
            __nanosleep(200);
          }
        }
        for (uint32_t r = 0; r < csz; ++r) dsmem_st(dsmem_addr(&sh_frame, r), nf);
      }
      cluster_sync_all();
      f = sh_frame;
      slot = clid;
      if (f >= call->frames) break;
      if (rank == 0 && tid == 0) {
        sh_flag[0] = 0;
        sh_flag[1] = 0;
      }
    }
    ++round;
    uint8_t* const xout = step ? ws.xhat + (size_t)f * cd.N : call->hard + (size_t)f * cd.N;
    float* const sout = step ? ws.soft + (size_t)f * cd.N * MB : call->soft_out + (size_t)f * cd.N * MB;
    float* const Tt = ws.Tt + (size_t)slot * cd.N * 8;
    uint8_t* const con = ws.con + (size_t)slot * ws.con_stride;
    float* const Pp = PMF ? call->p0buf + (size_t)slot * cd.N * Q : nullptr;
    if (PMF) {  // (also in step mode: nbldpc_step_pmf, slot = frame)
      // the frame's pmf rows scaled to probabilities p_v, several rows per warp, stored at
      // ppos(z) for the teams' phase-B reads; a row with a non-positive sum becomes all zero (its
      // variable-node outputs are then neutral and counted as numerical events, reading R23)
      const float* pf = call->pmf + (size_t)f * cd.N * Q;
      const int nwarp = nthr >> 5;
      if constexpr (Q >= 4) {
        // each lane takes EL consecutive entries of a row (16-byte loads), LN = Q / EL lanes per row, 32 / LN
        // rows per warp and pass (q = 16: 8 rows per warp-pass instead of 1 with half the lanes idle)
        constexpr int EL = Q / 32 > 4 ? Q / 32 : 4, LN = Q / EL, RW = 32 / LN;
        const int sub = lane / LN, zl = (lane % LN) * EL;
        for (int v0 = ((int)rank * nwarp + (tid >> 5)) * RW; v0 < cd.N; v0 += (int)csz * nwarp * RW) {
          const int v = v0 + sub;
          float pv[EL], sum = 0.0f;
#pragma unroll
          for (int k = 0; k < EL / 4; ++k) {
            const float4 x4 = v < cd.N ? __ldcs(reinterpret_cast<const float4*>(pf + (size_t)v * Q + zl) + k)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);  // streamed: read once
            pv[4 * k] = x4.x; pv[4 * k + 1] = x4.y; pv[4 * k + 2] = x4.z; pv[4 * k + 3] = x4.w;
            sum += (x4.x + x4.y) + (x4.z + x4.w);
          }
#pragma unroll
          for (int off = LN / 2; off >= 1; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
          const float inv = sum > 0.0f ? 1.0f / sum : 0.0f;
          if (v < cd.N) {
#pragma unroll
            for (int k = 0; k < EL; ++k) Pp[(size_t)v * Q + ppos<MB>(zl + k)] = pv[k] * inv;
          }
        }
      } else {
        constexpr int PER = 1;
        for (int v = (int)rank * nwarp + (tid >> 5); v < cd.N; v += (int)csz * nwarp) {
          float pv[PER], sum = 0.0f;
          const int z = lane;
          pv[0] = z < Q ? __ldcs(pf + (size_t)v * Q + z) : 0.0f;
          sum = pv[0];
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
          const float inv = sum > 0.0f ? 1.0f / sum : 0.0f;
          if (z < Q) Pp[(size_t)v * Q + ppos<MB>(z)] = pv[0] * inv;
        }
      }
      cluster_sync_all();
    } else if (!step) {
      // channel terms of the frame, computed once and cooperatively by the cluster's CTAs:
      // Tt[v][i] = tanh(L_{v,i} / 2), the factors of P_v^0 = (x)_i (1, t_i)
      const float* lf = call->llr + (size_t)f * cd.N * MB;
      for (int i = (int)rank * nthr + tid; i < cd.N * MB; i += (int)csz * nthr) {
        const int v = i / MB;
        Tt[(size_t)v * 8 + (i - v * MB)] = tanhf(0.5f * __ldcs(lf + i));  // streamed: read once
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");  // read next by bulk copies (async proxy)
      cluster_sync_all();
    }

#pragma unroll 1
    for (int ell = step ? P.step_iter : 0;; ++ell) {
      const int rb_ = step ? 0 : (ell & 1);
      const float* const Win = ws.W + ((size_t)rb_ * ws.S + slot) * EQ;
      float* const Wout = ws.W + ((size_t)(rb_ ^ 1) * ws.S + slot) * EQ;
      const __half* const WinH = reinterpret_cast<const __half*>(ws.W) + ((size_t)rb_ * ws.S + slot) * EQ;
      __half* const WoutH = reinterpret_cast<__half*>(ws.W) + ((size_t)(rb_ ^ 1) * ws.S + slot) * EQ;
      const bool do_dec = ell >= 1;
      const bool do_cn = step || ell < max_iters;
      // lazy decision: a pass that also runs the check node (ell < max_iters) needs its tentative decision only to
      // test the stopping rule (the estimate is returned for the last pass alone).  The first
      // NB_NPROBE chunks of every CTA are probes: their teams evaluate both halves of the split decision, so the
      // chunk's checks know their syndromes at once; the first unsatisfied probe check proves that the pass does
      // not stop the frame, and the remaining chunks of the cluster skip the decision and the own-row copy.
      // A pass whose probes are all satisfied, the last pass and step mode decide in full (outputs unchanged).
#ifndef NB_NPROBE
#define NB_NPROBE 128
#endif
      // probes per CTA and pass: at most an eighth of its chunks (a probe chunk costs an extra half decision)
#ifndef NB_PROBE_SHIFT
#define NB_PROBE_SHIFT 3
#endif
      const int nprobe = NB_NPROBE < (nch >> NB_PROBE_SHIFT) ? NB_NPROBE : ((nch >> NB_PROBE_SHIFT) > 1 ? (nch >> NB_PROBE_SHIFT) : 1);
      const int ps = round * 4099 + ell;  // pass stamp (max_iters < 4000: distinct over the frames of this CTA)
      const bool lazy = SPLITDEC_CT && NB_NPROBE > 0 && split && do_dec && do_cn && !step && max_iters < 4000;
      const bool lazy_all = lazy && !call->early_stop;  // no stopping rule: only the last pass decides
      auto we_needed = [&](int kcs) -> bool {  // does chunk kcs read its teams' own rows (warp-uniform)
        if (!lazy) return true;
        if (lazy_all) return false;
        if (kcs < nprobe) return true;
        int v = *reinterpret_cast<volatile int*>(&sh_skip);
        v = __shfl_sync(0xffffffffu, v, 0);
        return v != ps;
      };

      // stage chunk kc into buffer b of my group (one arrival per team on gmbar[b]): the group leader
      // bulk-copies the group's block of message rows (contiguous: reader-ordered storage), wide teams
      // bulk-copy their channel-term row; plain loads for q = 2
      auto stage = [&](int kc, int b, bool need_we) {
        if (t != 0) return;
        uint32_t tx = 0;
        EdgeRec rr{-1, 0};
        if (in_check) rr = recs[(kc * CPC + lc) * KT + j];
        const bool act = in_check && rr.partner_a >= 0;
        const int cg0 = ((int)rank + kc * (int)csz) * CPC + grp * CPG;  // the group's first check
        const bool lead = (tid - grp * GT) == 0;
        uint32_t blk = 0;
        if (lead && C::BULK && ell != 0 && cg0 < cd.M)
          blk = (uint32_t)((cd.M - cg0 < CPG ? cd.M - cg0 : CPG) * KPAD * Q * (F16 ? 2 : 4));
        if (act && !C::BULK && ell != 0) {
          const float* sp = Win + ((size_t)((((int)rank + kc * (int)csz) * CPC + lc) * KPAD + j)) * Q;
          float* dst = GST + b * GBLK + trow * C::QS;
#pragma unroll
          for (int r = 0; r < Q; ++r) dst[r] = __ldcg(sp + r);
        }
#ifdef NB_TT_BULK
        if (act && !C::THREG && !PMF) tx += 32;
#else
        // the team's channel-term row by two LDGSTS tracked by the same mbarrier (the pending count
        // is raised before this thread's own arrival, so the phase waits for them): a bulk copy from a
        // divergent thread would cost a uniform-register waterfall loop over the warp's team leaders
        if constexpr (PSTAGE) {
          if (act) {
            const float* srcp = call->p0buf + ((size_t)slot * cd.N + (rr.var_h >> 8 & 0x7FFFFFu)) * Q;
            float* dstp = PB + ((size_t)b * nteams + team) * Q;
            NB_CHECK((rr.var_h >> 8 & 0x7FFFFFu) < (uint32_t)cd.N && b < NS && team < nteams);
#pragma unroll
            for (int c4 = 0; c4 < Q / 4; ++c4)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dstp + 4 * c4)), "l"(srcp + 4 * c4)
                           : "memory");
            asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(&gmbar[b])) : "memory");
          }
        }
        if (act && !C::THREG && !PMF) {
          const float* srcT = Tt + (size_t)(rr.var_h >> 8 & 0x7FFFFFu) * 8;
          float* dstT = THB + b * nteams * 8;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dstT)), "l"(srcT) : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dstT + 4)), "l"(srcT + 4) : "memory");
          asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(&gmbar[b])) : "memory");
        }
#endif
        tx += blk;
        // SPLITDEC: my edge's own message W_e (row prow, contiguous) into my WE row, on the same mbarrier
        const bool wecp = SPLITDEC_CT && split && ell >= 1 && act && need_we;
        if (wecp) tx += Q * 4;
        mbar_arrive_tx(&gmbar[b], tx);
        if constexpr (SPLITDEC_CT) {
          if (wecp) bulk_g2s_ef(WE + ((size_t)b * nteams + team) * (Q + 16), Win + (size_t)(rr.partner_a >> 9) * Q, Q * 4, &gmbar[b]);
        }
        // the block in pieces of <= NB_BLK_PIECE bytes (several TMA transfers in flight)
#ifndef NB_BLK_PIECE
#define NB_BLK_PIECE 16384
#endif
        if constexpr (F16) {
          NB_CHECK(blk == 0 || ((size_t)cg0 * KPAD * Q * 2 + blk <= (size_t)cd.E * Q * 2 && blk <= (uint32_t)GBLKH * 4));
          for (uint32_t o = 0; o < blk; o += NB_BLK_PIECE)
            bulk_g2s(GST + b * GBLKH + o / 4, WinH + (size_t)cg0 * KPAD * Q + o / 2,
                     blk - o < NB_BLK_PIECE ? blk - o : NB_BLK_PIECE, &gmbar[b]);
        } else {
          NB_CHECK(blk == 0 || ((size_t)cg0 * KPAD * Q * 4 + blk <= (size_t)cd.E * Q * 4 && blk <= (uint32_t)GBLK * 4));
          for (uint32_t o = 0; o < blk; o += NB_BLK_PIECE)
            bulk_g2s(GST + b * GBLK + o / 4, Win + (size_t)cg0 * KPAD * Q + o / 4,
                     blk - o < NB_BLK_PIECE ? blk - o : NB_BLK_PIECE, &gmbar[b]);
        }
#ifdef NB_TT_BULK
        if (act && !C::THREG && !PMF) bulk_g2s(THB + b * nteams * 8, Tt + (size_t)(rr.var_h >> 8 & 0x7FFFFFu) * 8, 32, &gmbar[b]);
#endif
      };
      // channel-term row of chunk kc's variable, prefetched into registers one chunk ahead
      auto th_load = [&](int kc, float4 (&dst)[2]) {
        dst[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        dst[1] = dst[0];
        if (PMF || !C::THREG || !in_check || kc >= nch) return;
        const EdgeRec rr = recs[(kc * CPC + lc) * KT + j];
        if (rr.partner_a < 0) return;
        const float4* src = reinterpret_cast<const float4*>(Tt + (size_t)(rr.var_h >> 8 & 0x7FFFFFu) * 8);
        dst[0] = __ldcg(src);
        if constexpr (MB > 4) dst[1] = __ldcg(src + 1);
      };

      int buf = 0;
      for (int k0 = 0; k0 < NS - 1 && k0 < nch; ++k0) {  // prologue: NS - 1 chunks in flight
        const bool nw = we_needed(k0);
        stage(k0, k0, nw);
      }
      float4 thn[2];
      th_load(0, thn);
#pragma unroll 1
      for (int kc = 0; kc < nch; ++kc) {
        if (kc + NS - 1 < nch) {
          const bool nw = we_needed(kc + NS - 1);
          stage(kc + NS - 1, buf == 0 ? NS - 1 : buf - 1, nw);
        }
        // lazy decision: this chunk skips the decision (skipc) or is a probe
        bool skipc = lazy_all, probe = false;
        if (lazy && !lazy_all) {
          int v = *reinterpret_cast<volatile int*>(&sh_skip);
          v = __shfl_sync(0xffffffffu, v, 0);
          skipc = v == ps;
          probe = !skipc && kc < nprobe;
        }
        const uint32_t ptag = ((uint32_t)ps * 256u + (uint32_t)kc) & 0xFFFFFFu;  // kc < nprobe <= 128
        const float4 thc[2] = {thn[0], thn[1]};
        th_load(kc + 1, thn);
        mbar_wait(&gmbar[buf], (mb_parity >> buf) & 1u);
        mb_parity ^= 1u << buf;

        const int c = ((int)rank + kc * (int)csz) * CPC + lc;
        const bool cvalid = in_check && c < cd.M;
        EdgeRec rr{-1, 0};
        if (in_check) rr = recs[(kc * CPC + lc) * KT + j];
        const bool active = cvalid && rr.partner_a >= 0;
        const bool is_a = active && (rr.partner_a & 1);  // v's deciding edge (whole decision)
        const bool kind_a = active && (rr.var_h >> 31);  // SPLITDEC: the edge that evaluates the high half
        const int e = c * KPAD + j;
        const int var = (int)(rr.var_h >> 8 & 0x7FFFFFu);
        // my row: the message consumed by edge e (F32; it doubles as the work row), or (F16) the half
        // stage row sth, read only in phase A, and the float work row
        // LIN: the staged row stg is only read (phase A); st is my work row
        float* const stg = GST + buf * GBLK + trow * C::QS;
        float* st = F16 ? WK : WROW ? GST + NS * GBLK + trow * C::QS : stg;
        const __half* sth = reinterpret_cast<const __half*>(GST + buf * GBLKH) + trow * C::QS;

        // ---- channel terms t_i = tanh(L_i / 2)
        float th[MB];
        {
          const float tv[8] = {thc[0].x, thc[0].y, thc[0].z, thc[0].w, thc[1].x, thc[1].y, thc[1].z, thc[1].w};
#pragma unroll
          float tb8[8];
          if constexpr (!C::THREG) {  // the team's staged row of 8 channel terms: two 16-byte loads (broadcast)
            const float4 a4 = *reinterpret_cast<const float4*>(THB + buf * nteams * 8);
            const float4 b4 = *reinterpret_cast<const float4*>(THB + buf * nteams * 8 + 4);
            tb8[0] = a4.x; tb8[1] = a4.y; tb8[2] = a4.z; tb8[3] = a4.w; tb8[4] = b4.x; tb8[5] = b4.y; tb8[6] = b4.z; tb8[7] = b4.w;
          }
#pragma unroll
          // (an inactive padding team's terms are never used: its outputs become the neutral message below;
          // the log-format kernels keep the select, which their register allocation prefers)
          for (int b = 0; b < MB; ++b) th[b] = (!PMF && (LIN || active)) ? (C::THREG ? tv[b] : tb8[b]) : 0.0f;
        }
        // pmf input: my R entries of p_v at the phase-B coordinates zr, straight from L2
        float pv[PMF ? R : 1];
        if constexpr (PSTAGE) {
          const float* src = PB + ((size_t)buf * nteams + team) * Q;
#pragma unroll
          for (int ch = 0; ch < CH; ++ch) {
            const float4 v = active ? *reinterpret_cast<const float4*>(src + 4 * ch) : make_float4(0.f, 0.f, 0.f, 0.f);
            pv[4 * ch] = v.x; pv[4 * ch + 1] = v.y; pv[4 * ch + 2] = v.z; pv[4 * ch + 3] = v.w;
          }
        } else if constexpr (PMF) {
          const float* src = Pp + (size_t)var * Q + t * R;
          if constexpr (R >= 4) {
#pragma unroll
            for (int ch = 0; ch < CH; ++ch) {
              const float4 v = active ? __ldcg(reinterpret_cast<const float4*>(src) + ch) : make_float4(0.f, 0.f, 0.f, 0.f);
              pv[4 * ch] = v.x; pv[4 * ch + 1] = v.y; pv[4 * ch + 2] = v.z; pv[4 * ch + 3] = v.w;
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) pv[r] = active ? __ldcg(src + r) : 0.0f;
          }
        }
        // W_e (own message, for v's decision at its first edge) straight from L2 into registers;
        // consumed after the variable node
        float4 wo4[CH];
        uint4 woh[F16 ? (R >= 8 ? R / 8 : 1) : 1];  // F16: the raw half units, converted at the decision
#ifdef NB_DIAG_DEC_NOLOAD
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) wo4[ch] = make_float4(0.5f, 0.25f, 0.125f, 1.0f);
#endif
        auto load_wo = [&]() {
#ifdef NB_DIAG_DEC_NOLOAD
          if (false) {
#else
          if (is_a && do_dec && !split) {
#endif
            const int prow = rr.partner_a >> 9;  // W_e is stored in the row its reader (the partner edge) consumes
            if constexpr (F16) {
              const __half* so = WinH + (size_t)prow * Q;
#pragma unroll
              for (int u = 0; u < R / 8; ++u) woh[u] = __ldcg(reinterpret_cast<const uint4*>(so + mposh<MB>(t * R + 8 * u, prow)));
            } else if constexpr (R >= 4) {
              const float* so = Win + (size_t)prow * Q;
#pragma unroll
              for (int ch = 0; ch < CH; ++ch) wo4[ch] = __ldcg(reinterpret_cast<const float4*>(so + mpos<MB>(t * R + 4 * ch, prow)));
            } else {
              const float2 v2 = __ldcg(reinterpret_cast<const float2*>(Win + (size_t)prow * Q));
              wo4[0] = make_float4(v2.x, v2.y, 0.f, 0.f);
            }
          }
        };
#ifndef NB_WO_LATE
        if (!split) load_wo();  // (SPLITDEC: W_e comes staged)
#endif

        // ---- VARIABLE TO CHECK: x (phase B) = P^0 (*) Gamma^-1(W_e'); at l = 0, x = P^0
        float x[R];
        if (PMF && ell == 0) {
          // P^0 = WHT(p_v)
#pragma unroll
          for (int r = 0; r < R; ++r) x[r] = pv[r];
          wht_phase_b<MB, R, LR, LJ, TT>(x, t);
        } else if (ell == 0) {
          float base = 1.0f;
          if constexpr (TT > 1) {
#pragma unroll
            for (int b = 0; b < MB - 4; ++b)
              if ((t >> b) & 1) base *= th[LJ + b];
          }
          x[0] = base;
#pragma unroll
          for (int rb = 0; rb < LR; ++rb) {
            const int zb = (TT > 1) ? (rb < LJ ? rb : 4 + rb - LJ) : rb;
#pragma unroll
            for (int jj = 0; jj < (1 << rb); ++jj) x[(1 << rb) + jj] = x[jj] * th[zb];
          }
        } else {
          if constexpr (F16) {
#pragma unroll
            for (int u = 0; u < R / 8; ++u) {
              const uint4 v = *reinterpret_cast<const uint4*>(sth + mposh<MB>(t * R + 8 * u, e));
              const float2 a = h2f2(v.x), b = h2f2(v.y), cc = h2f2(v.z), d = h2f2(v.w);
              x[8 * u] = to_lin(a.x); x[8 * u + 1] = to_lin(a.y); x[8 * u + 2] = to_lin(b.x); x[8 * u + 3] = to_lin(b.y);
              x[8 * u + 4] = to_lin(cc.x); x[8 * u + 5] = to_lin(cc.y); x[8 * u + 6] = to_lin(d.x); x[8 * u + 7] = to_lin(d.y);
            }
          } else if constexpr (R >= 4) {
#pragma unroll
            for (int ch = 0; ch < CH; ++ch) {
              const float4 v = *reinterpret_cast<const float4*>(stg + mpos<MB>(t * R + 4 * ch, e));
              if constexpr (LIN) {
                x[4 * ch] = v.x; x[4 * ch + 1] = v.y; x[4 * ch + 2] = v.z; x[4 * ch + 3] = v.w;
              } else {
                x[4 * ch] = to_lin(v.x); x[4 * ch + 1] = to_lin(v.y); x[4 * ch + 2] = to_lin(v.z); x[4 * ch + 3] = to_lin(v.w);
              }
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) x[r] = LIN ? stg[r] : to_lin(stg[r]);
          }
          if constexpr (PMF) {
            if constexpr (LR > 0) wht_reg<R, 0>(x);  // z bits 0..LR-1 of WHT(W_e')
            if constexpr (LR > 1) wht_reg<R, 1>(x);
            if constexpr (LR > 2) wht_reg<R, 2>(x);
            if constexpr (LR > 3) wht_reg<R, 3>(x);
          } else {
#ifndef NB_ABL_NOVN
            bfly_regs<R, 0, LR>(x, th);  // z bits 0..LR-1
#endif
          }
          if constexpr (TT > 1) {
            // transposition through the consumed stage buffer, chunk-swizzled layout tpos(z); at q = 64 two
            // teams share each quarter warp and their rows are 64 words apart (the same banks), so the odd
            // team XORs its words by 16 (the other half of the bank quads): conflict-free both ways
            const int tpx = (TT == 4 && (trow & 1)) ? 16 : 0;
            // q = 256 (two teams per warp, rows 1 KB apart): the odd team stores 16-entry block b at block
            // (b + 1) mod 16 of its row, so that in every phase-B read the two teams' words differ in bank
            // bit 4 (ncu: the unshifted reads replayed 2x); the phase-A stores stay conflict-free
            const int tsh = (TT == 16 && (trow & 1)) ? 1 : 0;
            __syncwarp();  // every thread of the team has read its phase-A chunks
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              const int wa = TT == 16 ? (16 * ((t + tsh) & 15) + (tpos(16 * t + 4 * ch) & 15)) : (tpx ^ tpos(16 * t + 4 * ch));
              *reinterpret_cast<float4*>(st + wa) = make_float4(x[4 * ch], x[4 * ch + 1], x[4 * ch + 2], x[4 * ch + 3]);
            }
            __syncwarp();
            // LJ <= 1 (q >= 128): tpos((t << LJ) | (h << 4)) = 16 h + (((a ^ h ^ (h >> 2)) & 3) << 2) + ((t << LJ) & 3)
            // with a = ((t << LJ) >> 2) & 3 -- four row pointers, then every read is [pointer + 64 h bytes]
            // (q = 256, odd team: + 16 words, and block 15 wraps to block 0)
            const float* pc[4];
            if constexpr (LJ <= 1) {
#pragma unroll
              for (int c = 0; c < 4; ++c) pc[c] = st + 16 * tsh + (((((t << LJ) >> 2) ^ c) & 3) << 2) + ((t << LJ) & 3);
            }
#pragma unroll
            for (int h = 0; h < TT; ++h) {
              if constexpr (LJ == 0) {
                x[h] = (TT == 16 && h == 15) ? pc[0][tsh ? -16 : 240] : pc[(h ^ (h >> 2)) & 3][16 * h];
              } else if constexpr (LJ == 1) {
                const float2 v = *reinterpret_cast<const float2*>(pc[(h ^ (h >> 2)) & 3] + 16 * h);
                x[2 * h] = v.x; x[2 * h + 1] = v.y;
              } else {
#pragma unroll
                for (int q4 = 0; q4 < (1 << LJ) / 4; ++q4) {
                  const float4 v = *reinterpret_cast<const float4*>(st + (tpx ^ tpos(((t << LJ) | (h << 4)) + 4 * q4)));
                  x[(h << LJ) + 4 * q4] = v.x; x[(h << LJ) + 4 * q4 + 1] = v.y;
                  x[(h << LJ) + 4 * q4 + 2] = v.z; x[(h << LJ) + 4 * q4 + 3] = v.w;
                }
              }
            }
            // z bits 4..MB-1 = register bits LJ..3
            if constexpr (PMF) {
              if constexpr (LJ <= 0) wht_reg<R, 0>(x);
              if constexpr (LJ <= 1) wht_reg<R, 1>(x);
              if constexpr (LJ <= 2) wht_reg<R, 2>(x);
              if constexpr (LJ <= 3) wht_reg<R, 3>(x);
            } else {
#ifdef NB_ABL_NOVN
              if constexpr (false)
#endif
              if constexpr (LJ <= 0) bfly_reg<R, 0>(x, th[4 - LJ]);
#ifdef NB_ABL_NOVN
              if constexpr (false)
#endif
              if constexpr (LJ <= 1) bfly_reg<R, 1>(x, th[(5 - LJ) < MB ? 5 - LJ : 0]);
              if constexpr (LJ <= 2) bfly_reg<R, 2>(x, th[(6 - LJ) < MB ? 6 - LJ : 0]);
              if constexpr (LJ <= 3) bfly_reg<R, 3>(x, th[(7 - LJ) < MB ? 7 - LJ : 0]);
            }
          }
          if constexpr (PMF) {
            // q w'(x) = WHT(W_e')(x) at x = zr[r]: times p_v(x), back with the second WHT -> q raw
#pragma unroll
            for (int r = 0; r < R; ++r) x[r] *= pv[r];
            wht_phase_b<MB, R, LR, LJ, TT>(x, t);
          }
        }

        // ---- normalise so that entry 0 is (0, 0), Gamma in base 2, packed
        float raw0 = x[0];
        if constexpr (TT > 1) raw0 = __shfl_sync(0xffffffffu, x[0], lane & ~(TT - 1));
        uint32_t up[R];
        if constexpr (LIN) {
          // U = raw / raw(0): entry 0 is 1; |U| <= 1 up to rounding
          float inv0;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv0) : "f"(raw0));
          if constexpr (R >= 2) {
#pragma unroll
            for (int r = 0; r < R; r += 2) {  // FMUL2 with a broadcast factor
              const float2 u2 = __fmul2_rn(make_float2(x[r], x[r + 1]), make_float2(inv0, inv0));
              up[r] = __float_as_uint(u2.x);
              up[r + 1] = __float_as_uint(u2.y);
            }
          } else {
            up[0] = __float_as_uint(x[0] * inv0);
          }
          if (__builtin_expect(!(active && raw0 > 0.0f), 0)) {  // rare: one branch instead of per-entry selects
            if (!active) {  // padding edge: the neutral factor 1 in every entry
#pragma unroll
              for (int r = 0; r < R; ++r) up[r] = 0x3f800000u;
            } else {  // DC term <= 0: neutral message + numerical event (reading R10)
#pragma unroll
              for (int r = 0; r < R; ++r) up[r] = zr[r] == 0 ? 0x3f800000u : 0u;
              if (t == 0) atomicAdd(&ws.slot_events[step ? 0 : slot], 1);
            }
          }
        } else {
          const float lg0 = lg2a(raw0);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            // |x| >= 2^-120 keeps the magnitude finite (<= lg0 + 120); a rounding-negative magnitude
            // loses its sign bit to the message sign in the same LOP3
            const float mag = lg0 - lg2a(fmaxf(fabsf(x[r]), 7.52316385e-37f));
            up[r] = (__float_as_uint(mag) & ~kSign) | (__float_as_uint(x[r]) & kSign);
          }
          if (!active) {  // padding edge: the neutral message (0, 0) in every entry
#pragma unroll
            for (int r = 0; r < R; ++r) up[r] = 0u;
          } else if (!(raw0 > 0.0f)) {  // DC term <= 0: neutral message + numerical event (reading R10)
#pragma unroll
            for (int r = 0; r < R; ++r) up[r] = __float_as_uint(zr[r] == 0 ? 0.0f : kFloor);
            if (t == 0) atomicAdd(&ws.slot_events[step ? 0 : slot], 1);
          }
        }
        if (P.u_out != nullptr && active) {
          float* dst = P.u_out + ((size_t)f * cd.E + e) * Q;
#pragma unroll
          for (int r = 0; r < R; ++r) dst[zr[r]] = LIN ? lin_to_packed(__uint_as_float(up[r])) : __uint_as_float(up[r]);
        }

        // ---- TENTATIVE DECISION, split over the two edge teams (SPLITDEC above)
        float md5[5];
        // the sign bits over the team (a chain of shuffles) and my nibble: run after the check-node scatter, between
        // this warp's arrival on the group's scatter barrier and its wait, when the check node follows
        auto split_finish = [&]() {
          int s_off = 0, s_n = 5;
#ifdef NB_ABL_NORED
          uint32_t sb = 0;
          for (int b = 0; b < 5; ++b) sb |= (md5[b] < 0.0f ? 1u : 0u) << b;
          (void)s_off; (void)s_n;
#else
          const uint32_t sb = split_sign_bits(md5, lane);
          (void)s_off; (void)s_n;
#endif
          if (active && t == 0) {
            const uint32_t nib = ((sb >> 1) ^ ((sb & 1u) ? 0xFu : 0u)) & 0xFu;  // bit = sgn M(alpha^i) ^ sgn M(0)
            con[e] = (uint8_t)(kind_a ? nib << 4 : nib);
          }
        };
#ifdef NB_ABL_NODEC
        if constexpr (false)
#else
        if constexpr (SPLITDEC_CT)
#endif
        if (do_dec && split && !skipc) {
          // (probe chunks run both halves: hp = 0 the other edge's half, hp = 1 mine, whose totals stay in md5)
          uint32_t pnib = 0, pweak = 0;
#pragma unroll 1
          for (int hp = probe ? 0 : 1; hp < 2; ++hp) {
            const bool ka = (hp == 1) == kind_a;
            // my half: Sum_k Pm[k] Tm[k ^ s], s = 0, 1, 2, 4, 8 over my register index k, where (is_a) Pm = raw in
            // phase B and Tm = W_e moved to phase B, or (!is_a) Pm = W_e in phase A and Tm = raw moved to phase A.
            // The move: register k of lane t -> row k, position t of my stage row; then lane t reads row t.  Row
            // layout: 16 rows of 16 words, row r's 16-byte chunks XOR-swizzled by (r >> 1) & 3; the odd team's
            // rows shifted by one (row 15 wraps to row 0) -- scalar writes and 16-byte row reads conflict-free.
            __syncwarp();  // transposition reads of my row done
            const int sh = trow & 1;
            // my staged W_e row (WE rows are q + 16 words apart, so the two teams of a warp sit in opposite bank
            // halves): entry z at mpos(z) = 64 c + 4 (b ^ c) + (z & 3), c = (z >> 2) & 3, b = z >> 4
            const float* wrow = WE + ((size_t)buf * nteams + team) * (Q + 16);
            float Tm[16], dA[16];
            if (ka) {
              // Tm = W_e in phase B: z = t | h << 4 at 64 c + 16 (h >> 2) + 4 ((h & 3) ^ c) + (t & 3), c = t >> 2: four
              // pointers (by h & 3), then [pointer + 64 (h >> 2) bytes]
              const float* pk[4];
#pragma unroll
              for (int hl = 0; hl < 4; ++hl) pk[hl] = wrow + 64 * (t >> 2) + 4 * (hl ^ (t >> 2)) + (t & 3);
#pragma unroll
              for (int h = 0; h < 16; ++h) Tm[h] = pk[h & 3][16 * (h >> 2)];
            } else {
              // dA = W_e in phase A: z = 16 t + 4 ch + (0..3), one 16-byte chunk each
#pragma unroll
              for (int ch = 0; ch < 4; ++ch) {
                const float4 v4 = *reinterpret_cast<const float4*>(wrow + 64 * ch + 4 * (t ^ ch));
                dA[4 * ch] = v4.x; dA[4 * ch + 1] = v4.y; dA[4 * ch + 2] = v4.z; dA[4 * ch + 3] = v4.w;
              }
              // Tm = raw in phase A: register k of lane t -> row k, position t of my work row (row r's 16-byte chunks
              // XOR-swizzled by (r >> 1) & 3, the odd team's rows shifted by one); then lane t reads its row t
              float* pw[4];
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) pw[c4] = st + 16 * sh + ((((t >> 2) ^ c4) & 3) << 2) + (t & 3);
              if (active) {
#pragma unroll
                for (int k = 0; k < 16; ++k) (k == 15 ? pw[3][sh ? -16 : 240] : pw[(k >> 1) & 3][16 * k]) = x[k];
              }
              __syncwarp(__activemask());
              const float* rq = st + 16 * ((t + sh) & 15);
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const float4 v4 = *reinterpret_cast<const float4*>(rq + ((((t >> 1) ^ c4) & 3) << 2));
                Tm[4 * c4] = v4.x; Tm[4 * c4 + 1] = v4.y; Tm[4 * c4 + 2] = v4.z; Tm[4 * c4 + 3] = v4.w;
              }
            }
            auto half_dots = [&](const float (&Pm)[16]) {
              float2 acc[5];
#pragma unroll
              for (int b = 0; b < 5; ++b) acc[b] = make_float2(0.0f, 0.0f);
#pragma unroll
              for (int p2 = 0; p2 < 8; ++p2) {
                const int k = 2 * p2;
                const float2 pp = make_float2(Pm[k], Pm[k + 1]);
                acc[0] = __ffma2_rn(pp, make_float2(Tm[k], Tm[k + 1]), acc[0]);
                acc[1] = __ffma2_rn(pp, make_float2(Tm[k + 1], Tm[k]), acc[1]);
                acc[2] = __ffma2_rn(pp, make_float2(Tm[k ^ 2], Tm[(k ^ 2) + 1]), acc[2]);
                acc[3] = __ffma2_rn(pp, make_float2(Tm[k ^ 4], Tm[(k ^ 4) + 1]), acc[3]);
                acc[4] = __ffma2_rn(pp, make_float2(Tm[k ^ 8], Tm[(k ^ 8) + 1]), acc[4]);
              }
#pragma unroll
              for (int b = 0; b < 5; ++b) md5[b] = acc[b].x + acc[b].y;
            };
#ifdef NB_ABL_NODOTS
            for (int b = 0; b < 5; ++b) md5[b] = Tm[b] + dA[b] + x[b];
#else
            if (ka) half_dots(x); else half_dots(dA);
#endif
            if (probe) {
              float mdp[5];  // (the reduction works in place: my half's totals stay in md5 for split_finish)
#pragma unroll
              for (int b = 0; b < 5; ++b) mdp[b] = md5[b];
              const uint32_t sbp = split_sign_bits(mdp, lane);
              // a probe must never contradict the whole decision, whose two halves come from the variable's two
              // edges: a total that is not clearly away from zero (|M(alpha^i)| < 2^-6 |M(0)|, or M(0) zero or not
              // finite -- the totals are left in mdp[0] of team lanes 0, 2, 4, 8, 10) voids the probe
              {
                const float t0 = fabsf(__shfl_sync(0xffffffffu, mdp[0], lane & 16));
                const bool wk = !(fabsf(mdp[0]) >= 0.015625f * t0) || !(t0 > 0.0f) || !(t0 < 3.0e38f);
                pweak |= (__ballot_sync(0xffffffffu, wk) >> (lane & 16)) & 0x0515u;
              }
              const uint32_t nibp = ((sbp >> 1) ^ ((sbp & 1u) ? 0xFu : 0u)) & 0xFu;
              pnib |= ka ? nibp << 4 : nibp;
            }
          }
          if (probe && in_check && t == 0) {  // h_e x_v of my edge, for the probe check's syndrome
            uint32_t cb = 0;
            if (active && pnib != 0) cb = GE[GL[rr.var_h & 0xFFu] + GL[pnib]];
            sh_pc[team & 63] = ((pweak ? ptag ^ 0x800000u : ptag) << 8) | cb;
          }
          if (!do_cn) split_finish();
        }

        // ---- TENTATIVE DECISION at v's first edge: M_v(z) = sum_y raw(y) W_e(z ^ y)
        if (do_dec && !split) {
          // D = Gamma^-1(W_e) in the row layout word(z) = 16 tB(z) + rB(z), over the consumed Wp
#ifdef NB_WO_LATE
          load_wo();
#endif
          float* DB = st;
          // two teams per warp (q = 256): their rows are 1 KB apart (the same banks), so the odd team's D words
          // are XOR-ed by 16 (the other half of the banks) -- the scalar D stores no longer collide
          // (q = 64: XOR 24 -- the writes need the other half of the bank quads (^16), the row reads the
          // complementary quads within a half (^8))
          const int dbx = (trow & 1) ? (TT == 16 ? 16 : TT == 4 ? 24 : 0) : 0;
          if constexpr (TT > 1) __syncwarp();  // transposition reads done
          if constexpr (F16) {
            if (is_a) {
#pragma unroll
              for (int u = 0; u < R / 8; ++u) {
                const float2 a = h2f2(woh[u].x), b = h2f2(woh[u].y), cc = h2f2(woh[u].z), d = h2f2(woh[u].w);
                wo4[2 * u] = make_float4(a.x, a.y, b.x, b.y);
                wo4[2 * u + 1] = make_float4(cc.x, cc.y, d.x, d.y);
              }
            }
          }
          if (is_a) {
            if constexpr (TT > 1) {
              // LJ == 0: the even / odd D rows of my team (dbx = 16 for the odd team of the warp swaps them)
              float* const dbe = DB + (dbx & 16) + (t & 3);
              float* const dbo = DB + (16 ^ (dbx & 16)) + (t & 3);
#pragma unroll
              for (int ch = 0; ch < 4; ++ch) {
                const float4 v = wo4[ch];
                const float d4[4] = {LIN ? v.x : to_lin(v.x), LIN ? v.y : to_lin(v.y), LIN ? v.z : to_lin(v.z),
                                     LIN ? v.w : to_lin(v.w)};
                // z = 16 t + w: tB = w >> LJ, rB = (w & (2^LJ - 1)) | t << LJ; runs of 2^LJ entries stay
                // contiguous in a D row, so store them as one vector
                if constexpr (LJ >= 2) {
                  *reinterpret_cast<float4*>(DB + (dbx ^ db_word(ch >> (LJ - 2), ((4 * ch) & ((1 << LJ) - 1)) | (t << LJ)))) =
                      make_float4(d4[0], d4[1], d4[2], d4[3]);
                } else if constexpr (LJ == 1) {
                  *reinterpret_cast<float2*>(DB + (dbx ^ db_word(2 * ch, t << 1))) = make_float2(d4[0], d4[1]);
                  *reinterpret_cast<float2*>(DB + (dbx ^ db_word(2 * ch + 1, t << 1))) = make_float2(d4[2], d4[3]);
                } else {
                  // DB[dbx ^ db_word(tb, t)], tb = 4 ch + k4: the XOR 16 flips tb's bit 0, so the word is
                  // 32 (tb >> 1) + 16 ((tb & 1) ^ odd) + (((a ^ (tb >> 1)) & 3) << 2) + (t & 3), a = (t >> 2) & 3
#pragma unroll
                  for (int k4 = 0; k4 < 4; ++k4) {
                    const int tb = 4 * ch + k4;
                    float* const rowp = ((tb & 1) ? dbo : dbe) + 32 * (tb >> 1);
                    rowp[((((t >> 2) ^ (tb >> 1)) & 3) << 2)] = d4[k4];
                  }
                }
              }
            } else if (mode == 1 || SYM) {
              // one-thread teams hold all of D themselves (the dot products below read registers); the
              // row is written only for the paper syndrome's points and the symbol outputs (ncu, C5: these
              // stores were 16-way bank-conflicted, 2.0e9 wavefronts per 4,096-frame launch)
              if constexpr (R >= 4) {
#pragma unroll
                for (int ch = 0; ch < CH; ++ch) {
                  const float4 v = wo4[ch];
                  if constexpr (LIN) {
                    *reinterpret_cast<float4*>(DB + 4 * ch) = v;
                  } else {
                    DB[4 * ch] = to_lin(v.x); DB[4 * ch + 1] = to_lin(v.y); DB[4 * ch + 2] = to_lin(v.z); DB[4 * ch + 3] = to_lin(v.w);
                  }
                }
              } else {
                DB[0] = LIN ? wo4[0].x : to_lin(wo4[0].x);
                if constexpr (R > 1) DB[1] = LIN ? wo4[0].y : to_lin(wo4[0].y);
              }
            }
          }
          if constexpr (TT > 1) __syncwarp();
          // q = 256 (two teams per warp, WARPDEC): the decision of a deciding team is computed by the whole
          // warp -- the other team's lanes take the upper half of its entries (x by one shuffle each, D
          // from the deciding team's row) -- so a warp pays half a decision per deciding team; the host
          // orients the warp graph so that every warp has exactly one deciding team
          // measured slower (C4 3,592 -> 3,882, C3 853 -> 935 ns/frame-iter: every warp then runs a decision
          // round, and the other CTA on the SM hid most of the imbalance it removes); NB_WARPDEC=1 builds it
#ifdef NB_WARPDEC
          constexpr bool WARPDEC = TT == 16 && !SYM && !SOFT;
#else
          constexpr bool WARPDEC = false;
#endif
          uint32_t wd_bits = 0;
          if constexpr (WARPDEC) {
            if (mode == 0) {
              const bool dec0 = __shfl_sync(0xffffffffu, (int)is_a, 0) != 0;
              const bool dec1 = __shfl_sync(0xffffffffu, (int)is_a, 16) != 0;
#pragma unroll 1
              for (int T = 0; T < 2; ++T) {
                if (!(T == 0 ? dec0 : dec1)) continue;  // warp-uniform
                const bool inT = (lane >> 4) == T;
                const int hh = inT ? 0 : 1;  // the half of team T's 16 phase-B entries this lane takes
                float xs[8];
#pragma unroll
                for (int hp = 0; hp < 8; ++hp) {
                  const float o = __shfl_xor_sync(0xffffffffu, x[8 + hp], 16);
                  xs[hp] = inT ? x[hp] : o;
                }
                const int trT = (trow & ~1) | T;
                const float* DT = F16 ? GST + NS * GBLKH + trT * C::QS : GST + (WROW ? NS * GBLK : buf * GBLK) + trT * C::QS;
                const int dxT = T ? 16 : 0;
                float dh[8], dq[8];
#pragma unroll
                for (int c4 = 0; c4 < 2; ++c4) {
                  const float4 a4 = *reinterpret_cast<const float4*>(DT + (dxT ^ db_word(t, 8 * hh + 4 * c4)));
                  const float4 b4 = *reinterpret_cast<const float4*>(DT + (dxT ^ db_word(t, 8 * (1 - hh) + 4 * c4)));
                  dh[4 * c4] = a4.x; dh[4 * c4 + 1] = a4.y; dh[4 * c4 + 2] = a4.z; dh[4 * c4 + 3] = a4.w;
                  dq[4 * c4] = b4.x; dq[4 * c4 + 1] = b4.y; dq[4 * c4 + 2] = b4.z; dq[4 * c4 + 3] = b4.w;
                }
                float2 acc[MB + 1];
#pragma unroll
                for (int b = 0; b <= MB; ++b) acc[b] = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                  const float2 xp = make_float2(xs[2 * p], xs[2 * p + 1]);
                  acc[0] = __ffma2_rn(xp, make_float2(dh[2 * p], dh[2 * p + 1]), acc[0]);
                  acc[5] = __ffma2_rn(xp, make_float2(dh[2 * p + 1], dh[2 * p]), acc[5]);                    // z bit 4
                  acc[6] = __ffma2_rn(xp, make_float2(dh[(2 * p) ^ 2], dh[((2 * p) ^ 2) + 1]), acc[6]);      // z bit 5
                  acc[7] = __ffma2_rn(xp, make_float2(dh[(2 * p) ^ 4], dh[((2 * p) ^ 4) + 1]), acc[7]);      // z bit 6
                  acc[8] = __ffma2_rn(xp, make_float2(dq[2 * p], dq[2 * p + 1]), acc[8]);                    // z bit 7
                }
#pragma unroll
                for (int b = 0; b < 4; ++b) {  // z bits 0..3: the partner rows t ^ 2^b
                  const int tp = t ^ (1 << b);
#pragma unroll
                  for (int c4 = 0; c4 < 2; ++c4) {
                    const float4 v4 = *reinterpret_cast<const float4*>(DT + (dxT ^ db_word(tp, 8 * hh + 4 * c4)));
                    acc[b + 1] = __ffma2_rn(make_float2(xs[4 * c4], xs[4 * c4 + 1]), make_float2(v4.x, v4.y), acc[b + 1]);
                    acc[b + 1] = __ffma2_rn(make_float2(xs[4 * c4 + 2], xs[4 * c4 + 3]), make_float2(v4.z, v4.w), acc[b + 1]);
                  }
                }
                float mw[MB + 1];
#pragma unroll
                for (int b = 0; b <= MB; ++b) mw[b] = acc[b].x + acc[b].y;
                int so = 0, sn = MB + 1;
                const uint32_t bits = team_sign_bits<MB + 1, 32>(mw, lane, so, sn);
                if (inT) wd_bits = bits;
              }
            }
          }
          float mf[MB + 1];
#pragma unroll
          for (int b = 0; b <= MB; ++b) mf[b] = 0.0f;
          if (is_a && !(WARPDEC && mode == 0)) {
            // pairwise FFMA2 dot products: M(0) and the register-bit points in-thread, the
            // thread-bit points against the partner thread's row
            float d[R];
            // dbx ^ db_word(t ^ m, 4 ch) = Lt ^ 16 m ^ 4 ((m >> 1) & 3) ^ 4 ch (the fields are disjoint, the map
            // XOR-linear): one XOR with a constant per 16-byte read
            const int Lt = dbx ^ (16 * t) ^ (((t >> 1) & 3) << 2);
            if constexpr (TT > 1) {
#pragma unroll
              for (int ch = 0; ch < 4; ++ch) {
                const float4 v4 = *reinterpret_cast<const float4*>(DB + (Lt ^ (4 * ch)));
                d[4 * ch] = v4.x; d[4 * ch + 1] = v4.y; d[4 * ch + 2] = v4.z; d[4 * ch + 3] = v4.w;
              }
            } else {
#pragma unroll
              for (int r = 0; r < R; ++r) {
                const float v = R >= 4 ? (&wo4[r >> 2].x)[r & 3] : (r == 0 ? wo4[0].x : wo4[0].y);
                d[r] = LIN ? v : to_lin(v);
              }
            }
            if constexpr (R >= 2) {
              float2 acc[MB + 1];
#pragma unroll
              for (int b = 0; b <= MB; ++b) acc[b] = make_float2(0.0f, 0.0f);
#pragma unroll
              for (int p = 0; p < R / 2; ++p) {
                const float2 xp = make_float2(x[2 * p], x[2 * p + 1]);
                acc[0] = __ffma2_rn(xp, make_float2(d[2 * p], d[2 * p + 1]), acc[0]);
#pragma unroll
                for (int rb = 0; rb < LR; ++rb) {
                  const int zb = (TT > 1) ? (rb < LJ ? rb : 4 + rb - LJ) : rb;
                  const int w = (2 * p) ^ (1 << rb);
                  const float2 dp = rb == 0 ? make_float2(d[w], d[w - 1]) : make_float2(d[w], d[w + 1]);
                  acc[zb + 1] = __ffma2_rn(xp, dp, acc[zb + 1]);
                }
              }
              if constexpr (TT > 1) {
#pragma unroll
                for (int b = 0; b < MB - 4; ++b) {
                  const int cm = (16 << b) ^ ((((1 << b) >> 1) & 3) << 2);  // the row t ^ 2^b
#pragma unroll
                  for (int ch = 0; ch < 4; ++ch) {
                    const float4 v4 = *reinterpret_cast<const float4*>(DB + (Lt ^ cm ^ (4 * ch)));
                    acc[LJ + b + 1] = __ffma2_rn(make_float2(x[4 * ch], x[4 * ch + 1]), make_float2(v4.x, v4.y),
                                                 acc[LJ + b + 1]);
                    acc[LJ + b + 1] = __ffma2_rn(make_float2(x[4 * ch + 2], x[4 * ch + 3]), make_float2(v4.z, v4.w),
                                                 acc[LJ + b + 1]);
                  }
                }
              }
#pragma unroll
              for (int b = 0; b <= MB; ++b) mf[b] = acc[b].x + acc[b].y;
            } else {
              mf[0] = x[0] * d[0];
            }
          }
          if constexpr (SYM) {
            // symbol posterior and MAP: every lane runs the transforms (full-warp shuffles)
            float a[R], bq[R];
#pragma unroll
            for (int r = 0; r < R; ++r) a[r] = is_a ? x[r] : 0.0f;
            if constexpr (TT > 1) {
#pragma unroll
              for (int ch = 0; ch < 4; ++ch) {
                const float4 v4 = is_a ? *reinterpret_cast<const float4*>(DB + (dbx ^ db_word(t, 4 * ch))) : make_float4(0.f, 0.f, 0.f, 0.f);
                bq[4 * ch] = v4.x; bq[4 * ch + 1] = v4.y; bq[4 * ch + 2] = v4.z; bq[4 * ch + 3] = v4.w;
              }
            } else {
#pragma unroll
              for (int r = 0; r < R; ++r) bq[r] = is_a ? DB[r] : 0.0f;
            }
            wht_phase_b<MB, R, LR, LJ, TT>(a, t);
            wht_phase_b<MB, R, LR, LJ, TT>(bq, t);
            float tot = 0.0f, best = 0.0f;
            int bx = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              a[r] = fmaxf(a[r] * bq[r], 0.0f);  // mu >= 0; rounding residues clamp to 0
              tot += a[r];
              if (r == 0 || a[r] > best || (a[r] == best && zr[r] < bx)) { best = a[r]; bx = zr[r]; }
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
            if (is_a) {
              const float inv = tot > 0.0f ? 1.0f / tot : 0.0f;
              if (call->post_out) {
                float* dst = call->post_out + ((size_t)f * cd.N + var) * Q;
#pragma unroll
                for (int r = 0; r < R; ++r) dst[zr[r]] = a[r] * inv;
              }
              if (call->map_out && t == 0) call->map_out[(size_t)f * cd.N + var] = (uint8_t)bx;
            }
          }
          // soft outputs requested (grid-uniform): the decision again in fp64 from the edge's linear
          // spectra (decision_f64, reading R22) -- its signs and ratios replace the fp32 ones
          double md[MB + 1];
          if constexpr (SOFT) {
            float bl[R], dl[R], pl[PMF ? R : 1];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int z = t * R + r;
              float bv = 1000.0f;  // packed entries (Gamma^-1 in fp64 inside); 1000: a zero
              if (is_a) {
                if constexpr (F16) bv = __half2float(__ldcg(WinH + (size_t)e * Q + mposh<MB>(z, e)));
                else bv = __ldcg(Win + (size_t)e * Q + mpos<MB>(z, e));
              }
              bl[r] = bv;
              const float dv = R >= 4 ? (&wo4[r >> 2].x)[r & 3] : (r == 0 ? wo4[0].x : wo4[0].y);
              dl[r] = is_a ? dv : 1000.0f;
              if constexpr (PMF) pl[r] = is_a ? __ldcg(Pp + (size_t)var * Q + ppos<MB>(z)) : 0.0f;
            }
            decision_f64<MB, LR, PMF>(bl, dl, pl, th, t, md);
          }
          // signs of M(0) and M(alpha^i) over the team (bit i of sbits = [M(.) < 0], index 0 = M(0))
          uint32_t sbits;
          int s_off = 0, s_n = MB + 1;
#ifndef NB_RS_MIN_TT
#define NB_RS_MIN_TT 8
#endif
          if constexpr (SOFT) {
            sbits = 0;
#pragma unroll
            for (int b = 0; b <= MB; ++b) sbits |= (md[b] < 0.0 ? 1u : 0u) << b;
          } else if (WARPDEC && mode == 0) {
            sbits = wd_bits;
          } else if constexpr (TT >= NB_RS_MIN_TT) {
            sbits = team_sign_bits<MB + 1, TT>(mf, lane, s_off, s_n);
          } else if constexpr (TT > 1) {  // small teams: full butterfly all-reduce, every lane holds all totals
#pragma unroll
            for (int off = TT / 2; off >= 1; off >>= 1)
#pragma unroll
              for (int b = 0; b <= MB; ++b) mf[b] += __shfl_xor_sync(0xffffffffu, mf[b], off);
            sbits = 0;
#pragma unroll
            for (int b = 0; b <= MB; ++b) sbits |= (mf[b] < 0.0f ? 1u : 0u) << b;
          } else {
            sbits = 0;
#pragma unroll
            for (int b = 0; b <= MB; ++b) sbits |= (mf[b] < 0.0f ? 1u : 0u) << b;
          }
          const uint32_t s0z = sbits & 1u;  // sgn_GF2 M(0); an exact zero has sign 0
          if (want_soft && is_a && t == 0) {
#pragma unroll
            for (int b = 0; b < MB; ++b) sout[(size_t)var * MB + b] = soft_ratio(md[b + 1], md[0]);
          }
          if (is_a && t == 0) {
            const int xv = (int)(((sbits >> 1) ^ (s0z ? 0xFFu : 0u)) & ((1u << MB) - 1u));
            xout[var] = (uint8_t)xv;
            if (mode == 0) {  // syndrome contributions h_cv xhat_v to both checks of v
              int ca = 0, cbv = 0;
              if (xv != 0) {  // shared-memory GF tables: no global round trip on the decision's tail
                const int lx = GL[xv];
                ca = GE[GL[rr.var_h & 0xFFu] + lx];
                cbv = GE[GL[(rr.partner_a >> 1) & 0xFF] + lx];
              }
              con[e] = (uint8_t)ca;
              con[rr.partner_a >> 9] = (uint8_t)cbv;
            }
          }
          if (mode == 1) {
            // paper-mode fast syndrome: sign bits of M_v(H_cv alpha^i), both checks
            uint64_t pa = 0, pbv = 0;
            if (is_a) {
              const uint32_t* ea = reinterpret_cast<const uint32_t*>(cd.edges + e) + 3;
              const uint32_t* eb = reinterpret_cast<const uint32_t*>(cd.edges + (rr.partner_a >> 9)) + 3;
              pa = (uint64_t)__ldg(ea) | ((uint64_t)__ldg(ea + 1) << 32);
              pbv = (uint64_t)__ldg(eb) | ((uint64_t)__ldg(eb + 1) << 32);
            }
            int ma = 0, mbb = 0;
#pragma unroll 1
            for (int i = 0; i < 2 * MB; ++i) {
              const int z = (int)(((i < MB ? pa : pbv) >> (8 * (i < MB ? i : i - MB))) & 0xFF);
              float acc = 0.0f;
              if (is_a) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                  const int yy = zr[r] ^ z;
                  int w;
                  if constexpr (TT > 1) {
                    w = dbx ^ db_word((yy >> LJ) & (TT - 1), (yy & ((1 << LJ) - 1)) | ((yy >> 4) << LJ));
                  } else {
                    w = yy;
                  }
                  acc = fmaf(x[r], DB[w], acc);
                }
              }
              if constexpr (TT > 1) {
#pragma unroll
                for (int off = TT / 2; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
              }
              const int bit = (int)(((acc < 0.0f) ? 1u : 0u) ^ s0z);
              if (i < MB) ma |= bit << i; else mbb |= bit << (i - MB);
            }
            if (is_a && t == 0) {
              con[e] = (uint8_t)ma;
              con[rr.partner_a >> 9] = (uint8_t)mbb;
            }
          }
        }

        // ---- CHECK TO VARIABLE
        if (do_cn) {
          // pi_e^-1 of my z's (linear: XOR of basis images)
          int oidx[R];
          // LIN: the byte addresses in my (row-aligned) scatter row directly, st_s ^ 4 pi_e^-1(z) -- the same XOR
          // chain on pre-shifted images; the read-back uses the same addresses (padding edges take h = 1, the
          // identity, so they keep the natural order)
          uint32_t sa[LIN && !PAIRIL ? R : 1];
          if constexpr (LIN && !PAIRIL) {
            const uint64_t pv = PT[active ? (rr.var_h & 0xFFu) : 1u];
            uint32_t base = smem_u32(st);
            NB_CHECK((base & (Q * 4 - 1)) == 0);
            if constexpr (TT > 1) {
#pragma unroll
              for (int b = 0; b < MB - 4; ++b)
                if ((t >> b) & 1) base ^= (uint32_t)((pv >> (8 * (LJ + b))) & 0xFFu) << 2;
            }
            sa[0] = base;
#pragma unroll
            for (int rb = 0; rb < LR; ++rb) {
              const int zb = (TT > 1) ? (rb < LJ ? rb : 4 + rb - LJ) : rb;
              const uint32_t img = (uint32_t)((pv >> (8 * zb)) & 0xFFu) << 2;
#pragma unroll
              for (int jj = 0; jj < (1 << rb); ++jj) sa[(1 << rb) + jj] = sa[jj] ^ img;
            }
          } else {
            const uint64_t pv = PT[rr.var_h & 0xFFu];
            int base = 0;
            if constexpr (TT > 1) {
#pragma unroll
              for (int b = 0; b < MB - 4; ++b)
                if ((t >> b) & 1) base ^= (int)((pv >> (8 * (LJ + b))) & 0xFFu);
            }
            oidx[0] = base;
#pragma unroll
            for (int rb = 0; rb < LR; ++rb) {
              const int zb = (TT > 1) ? (rb < LJ ? rb : 4 + rb - LJ) : rb;
              const int img = (int)((pv >> (8 * zb)) & 0xFFu);
#pragma unroll
              for (int jj = 0; jj < (1 << rb); ++jj) oidx[(1 << rb) + jj] = oidx[jj] ^ img;
            }
            if (!active) {
#pragma unroll
              for (int r = 0; r < R; ++r) oidx[r] = zr[r];
            }
          }
          (void)oidx;
          (void)sa;
          // transposition / DB reads of X done (LANEMAJOR: the scatter writes into the whole warp's buffer)
          if constexpr (TT > 1 || LANEMAJOR) __syncwarp();
          if (cvalid) {
            // scatter: X_e(pi_e^-1 z) = U_e(z) = T_e(.); padding teams hold the neutral message
            // 32-bit shared-window addresses: one LEA per entry instead of an IMAD + IADD3 pair
            if constexpr (PAIRIL) {
              const uint32_t il_s = smem_u32(GST + NS * GBLK + (trow & ~1) * C::QS) + ((uint32_t)(trow & 1) << 2);
#pragma unroll
              for (int r = 0; r < R; ++r) {
                NB_CHECK(oidx[r] >= 0 && oidx[r] < Q);
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(il_s + ((uint32_t)oidx[r] << 3)), "r"(up[r]) : "memory");
              }
            } else if constexpr (LANEMAJOR) {
              // the group's consumed stage buffer (F16: its float work rows), 32 q floats
              const uint32_t xs_s = smem_u32(F16 ? GST + NS * GBLKH : GST + buf * GBLK) + ((uint32_t)(tid - grp * GT) << 2);
#pragma unroll
              for (int r = 0; r < R; ++r) {
                NB_CHECK(oidx[r] >= 0 && oidx[r] < Q && 32 * Q <= GBLK && tid - grp * GT < 32);
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(xs_s + ((uint32_t)oidx[r] << 7)), "r"(up[r]) : "memory");
              }
            } else if constexpr (LIN) {
#pragma unroll
              for (int r = 0; r < R; ++r) {
                NB_CHECK((sa[r] ^ smem_u32(st)) < (uint32_t)Q * 4);
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(sa[r]), "r"(up[r]) : "memory");
              }
            } else {
              const uint32_t st_s = smem_u32(st);
#pragma unroll
              for (int r = 0; r < R; ++r) {
                NB_CHECK(oidx[r] >= 0 && oidx[r] < Q);
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(st_s + ((uint32_t)oidx[r] << 2)), "r"(up[r]) : "memory");
              }
            }
          }
          if (SPLITDEC_CT && split && do_dec) {
            // arrive on the group's scatter barrier (one arrival per warp, after the warp's scatter: __syncwarp orders
            // the lanes' stores before lane 0's release), finish the decision, then wait for the other warps
            __syncwarp();
            if (lane == 0)
              asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(&sh_cbar[grp]))
                           : "memory");
#ifndef NB_ABL_NODEC
            if (!skipc) split_finish();
#endif
            mbar_wait(&sh_cbar[grp], cb_parity);
            cb_parity ^= 1u;
            if (probe && cvalid && pck == 0) {
              // the probe check's syndrome from its teams' words of this chunk; a word with another
              // tag (a team that did not probe) voids the probe
              uint32_t syn = 0;
              bool valid = KT <= 64;
              for (int jj = 0; jj < KT && jj < 64; ++jj) {
                const uint32_t w = *reinterpret_cast<volatile uint32_t*>(&sh_pc[(team + jj) & 63]);
                valid = valid && (w >> 8) == ptag;
                syn ^= w & 0xFFu;
              }
              if (valid && syn != 0) {
                *reinterpret_cast<volatile int*>(&sh_skip) = ps;
                for (uint32_t r = 0; r < csz; ++r)
                  if (r != rank) dsmem_st(dsmem_addr(&sh_skip, r), ps);
              }
            }
          } else {
            check_sync(lc, TPC);
          }
          if constexpr (PAIRIL) {
            float* rows = GST + NS * GBLK + (lc - grp * CPG) * KT * C::QS;
            const int flip = SPLIT == 1 ? ((lane >> 4) & 1) : (pck & 1);
            switch (JPT) {
              case 2: tot_prod_il<R, 2, TT, C::QS>(rows, wgrp, jbase, flip, SPLIT, cvalid); break;
              case 4: tot_prod_il<R, 4, TT, C::QS>(rows, wgrp, jbase, flip, SPLIT, cvalid); break;
              case 8: tot_prod_il<R, 8, TT, C::QS>(rows, wgrp, jbase, flip, SPLIT, cvalid); break;
              default: tot_prod_il<R, R, TT, C::QS>(rows, wgrp, jbase, flip, SPLIT, cvalid); break;
            }
          } else if constexpr (LIN) {
            switch (JPT) {
              case 1: tot_prod<R, 1, TT, C::QS>(smem, gbase + NS * GBLK, SPLIT, cvalid); break;
              case 2: tot_prod<R, (R >= 2 ? 2 : 1), TT, C::QS>(smem, gbase + NS * GBLK, SPLIT, cvalid); break;
              case 4: tot_prod<R, (R >= 4 ? 4 : 1), TT, C::QS>(smem, gbase + NS * GBLK, SPLIT, cvalid); break;
              case 8: tot_prod<R, (R >= 8 ? 8 : 1), TT, C::QS>(smem, gbase + NS * GBLK, SPLIT, cvalid); break;
              default:
#ifndef NB_ABL_NOTOT
                tot_prod<R, R, TT, C::QS>(smem, gbase + NS * GBLK, SPLIT, cvalid);
#endif
                break;
            }
          } else if constexpr (LANEMAJOR) {
            const float* xs = F16 ? GST + NS * GBLKH : GST + buf * GBLK;
            const int c0 = (lc - grp * CPG) * KT;
            switch (JPT) {
              case 1: tot_sum_lm<R, 1>(xs, c0, TOT, wgrp, SPLIT, pck, cvalid); break;
              case 2: tot_sum_lm<R, (R >= 2 ? 2 : 1)>(xs, c0, TOT, wgrp, SPLIT, pck, cvalid); break;
              case 4: tot_sum_lm<R, (R >= 4 ? 4 : 1)>(xs, c0, TOT, wgrp, SPLIT, pck, cvalid); break;
              case 8: tot_sum_lm<R, (R >= 8 ? 8 : 1)>(xs, c0, TOT, wgrp, SPLIT, pck, cvalid); break;
              default: tot_sum_lm<R, R>(xs, c0, TOT, wgrp, SPLIT, pck, cvalid); break;
            }
          } else switch (JPT) {  // tix: two checks per warp -> the odd one rotates its w groups
            case 1: tot_sum<R, 1, TT, C::QS>(smem, gbase + (F16 ? 0 : WROW ? NS * GBLK : buf * GBLK), TOT, wgrp, SPLIT, pck, cvalid, tix); break;
            case 2: tot_sum<R, (R >= 2 ? 2 : 1), TT, C::QS>(smem, gbase + (F16 ? 0 : WROW ? NS * GBLK : buf * GBLK), TOT, wgrp, SPLIT, pck, cvalid, tix); break;
            case 4: tot_sum<R, (R >= 4 ? 4 : 1), TT, C::QS>(smem, gbase + (F16 ? 0 : WROW ? NS * GBLK : buf * GBLK), TOT, wgrp, SPLIT, pck, cvalid, tix); break;
            case 8: tot_sum<R, (R >= 8 ? 8 : 1), TT, C::QS>(smem, gbase + (F16 ? 0 : WROW ? NS * GBLK : buf * GBLK), TOT, wgrp, SPLIT, pck, cvalid, tix); break;
            default: tot_sum<R, R, TT, C::QS>(smem, gbase + (F16 ? 0 : WROW ? NS * GBLK : buf * GBLK), TOT, wgrp, SPLIT, pck, cvalid, tix); break;
          }
          check_sync(lc, TPC);
          // q = 256 (LIN): read W_e back in the phase-A coordinates z = 16 t + r (my own XOR chain of pi_e^-1 images,
          // base from the high nibble t), so that each thread holds 16 consecutive entries: four 16-byte global
          // stores instead of sixteen words, and the scatter addresses are dead after the scatter
          constexpr bool RBA = LIN && TT == 16 && !PAIRIL;
          if (RBA && active) {
            const uint64_t pv = PT[rr.var_h & 0xFFu];
            uint32_t ra[16];
            uint32_t base = smem_u32(st);
#pragma unroll
            for (int b = 0; b < 4; ++b)
              if ((t >> b) & 1) base ^= (uint32_t)((pv >> (8 * (4 + b))) & 0xFFu) << 2;
            ra[0] = base;
#pragma unroll
            for (int rb = 0; rb < 4; ++rb) {
              const uint32_t img = (uint32_t)((pv >> (8 * rb)) & 0xFFu) << 2;
#pragma unroll
              for (int jj = 0; jj < (1 << rb); ++jj) ra[(1 << rb) + jj] = ra[jj] ^ img;
            }
            float out[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(out[r]) : "r"(ra[r]) : "memory");
            const int prow = rr.partner_a >> 9;
            NB_CHECK(prow >= 0 && prow < cd.E);
            float* dst = Wout + (size_t)prow * Q;
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4)
              st_w4(dst + mpos<MB>(16 * t + 4 * c4, prow), make_float4(out[4 * c4], out[4 * c4 + 1], out[4 * c4 + 2], out[4 * c4 + 3]));
          } else if (active) {
            float out[R];
            const uint32_t tot_s = PAIRIL ? smem_u32(GST + NS * GBLK + (trow & ~1) * C::QS) + ((uint32_t)(trow & 1) << 2)
                                          : smem_u32(LIN ? st : TOT);
            constexpr int osh = PAIRIL ? 3 : 2;  // PAIRIL: my entries sit at 2 w + (trow & 1) of the pair
#pragma unroll
            for (int r = 0; r < R; ++r) {
              float xt;
              if constexpr (LIN && !PAIRIL) {
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xt) : "r"(sa[r]) : "memory");
              } else {
                NB_CHECK(oidx[r] >= 0 && oidx[r] < Q);
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xt) : "r"(tot_s + ((uint32_t)oidx[r] << osh)) : "memory");
              }
              if constexpr (LIN) {
                out[r] = xt;  // W_e(z) = prod_{j != e} X_j(pi_e^-1 z), written back into my own scatter row
              } else {
                const float mg = fabsf(xt) - __uint_as_float(up[r] & ~kSign);  // >= 0 up to rounding
                out[r] = __uint_as_float((__float_as_uint(mg) & ~kSign) | ((__float_as_uint(xt) ^ up[r]) & kSign));
              }
            }
            // my last generic access to this chunk's stage buffer: order it before the buffer's next bulk fill
            // here, so that the fence does not wait for the global stores below (LIN: the generic writes go to the
            // work rows, the staged rows are only read -- no fence)

            const int prow = rr.partner_a >> 9;  // stored where the partner edge will read it
            NB_CHECK(prow >= 0 && prow < cd.E);
            float* dst = Wout + (size_t)prow * Q;
            if constexpr (F16) {
              __half* dh = WoutH + (size_t)prow * Q;
              if constexpr (TT > 1) {
                constexpr int V = C::V;  // runs of V = 2^LJ entries, contiguous within a 16-byte unit
#pragma unroll
                for (int h = 0; h < TT; ++h) {
                  const int z0 = (t << LJ) | (h << 4);
                  __half* p = dh + mposh<MB>(z0, prow);
                  if constexpr (V == 1) {
                    *p = NB_F2H1(out[h]);
                  } else if constexpr (V == 2) {
                    *reinterpret_cast<uint32_t*>(p) = f22h(out[2 * h], out[2 * h + 1]);
                  } else if constexpr (V == 4) {
                    *reinterpret_cast<uint2*>(p) = make_uint2(f22h(out[4 * h], out[4 * h + 1]), f22h(out[4 * h + 2], out[4 * h + 3]));
                  } else {
                    *reinterpret_cast<uint4*>(p) = make_uint4(f22h(out[8 * h], out[8 * h + 1]), f22h(out[8 * h + 2], out[8 * h + 3]),
                                                              f22h(out[8 * h + 4], out[8 * h + 5]), f22h(out[8 * h + 6], out[8 * h + 7]));
                  }
                }
              } else {
#pragma unroll
                for (int u = 0; u < R / 8; ++u)
                  *reinterpret_cast<uint4*>(dh + mposh<MB>(8 * u, prow)) =
                      make_uint4(f22h(out[8 * u], out[8 * u + 1]), f22h(out[8 * u + 2], out[8 * u + 3]),
                                 f22h(out[8 * u + 4], out[8 * u + 5]), f22h(out[8 * u + 6], out[8 * u + 7]));
              }
            } else if constexpr (TT > 1) {
              constexpr int V = C::V;
#pragma unroll
              for (int h = 0; h < TT; ++h) {
                const int z0 = (t << LJ) | (h << 4);
                if constexpr (V == 1) {
                  dst[mpos<MB>(z0, prow)] = out[h];
                } else if constexpr (V == 2) {
                  *reinterpret_cast<float2*>(dst + mpos<MB>(z0, prow)) = make_float2(out[2 * h], out[2 * h + 1]);
                } else {
#pragma unroll
                  for (int q4 = 0; q4 < V / 4; ++q4)
                    st_w4(dst + mpos<MB>(z0 + 4 * q4, prow), make_float4(out[h * V + 4 * q4], out[h * V + 4 * q4 + 1],
                                                                         out[h * V + 4 * q4 + 2], out[h * V + 4 * q4 + 3]));
                }
              }
            } else if constexpr (R >= 4) {
#pragma unroll
              for (int ch = 0; ch < CH; ++ch)
                st_w4(dst + mpos<MB>(4 * ch, prow), make_float4(out[4 * ch], out[4 * ch + 1], out[4 * ch + 2], out[4 * ch + 3]));
            } else {
#pragma unroll
              for (int r = 0; r < R; ++r) dst[r] = out[r];
            }
          }
        }
        // generic-proxy writes to this stage buffer (DB) are ordered before its next bulk fill (active teams of a
        // check-node pass fenced before their global stores)
        // LIN: no generic writes to the staged rows; the buffer refilled at the next chunk's start was last read
        // before this chunk's first check barrier, and a work row is rewritten only by its own team after the
        // other threads' check-node accesses to it (second check barrier) -- no end-of-chunk barrier either
        if constexpr (!WROW) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          group_sync();  // the group's buffers of this chunk are free
        }
        buf = buf + 1 == NS ? 0 : buf + 1;
      }
      cp_async_wait<0>();
      // SPLITDEC: x_v = the nibbles of v's two edges (con); the CTA whose check holds v's is_a edge writes x_v,
      // and (decode) each CTA XORs h_e x_v(e) over its checks' edges (exact syndrome) -- one
      // thread per edge slot, the check's KT slots reduced by shuffles (KT divides 32)
      auto split_pass_end = [&](bool want_syn) -> int {
        int badc = 0;
        const int tot_e = nch * CPC * KT;
        constexpr int UB = 8;  // edge slots per thread whose byte loads are in flight together
        for (int i0 = 0; i0 < tot_e; i0 += UB * nthr) {
          uint32_t xa[UB], vh[UB];
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int i = i0 + u * nthr + tid;
            xa[u] = 0;
            vh[u] = 0;
            if (i < tot_e) {
              const int kc = i / (CPC * KT), rem = i - kc * (CPC * KT);
              const int l = rem / KT, jj = rem - l * KT;
              const int c = ((int)rank + kc * (int)csz) * CPC + l;
              const EdgeRec er = recs[i];
              if (c < cd.M && er.partner_a >= 0) {
                xa[u] = (uint32_t)__ldcg(con + c * KPAD + jj) | (uint32_t)__ldcg(con + (er.partner_a >> 9)) | 0x100u;
                vh[u] = er.var_h;
              }
            }
          }
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            uint32_t contrib = 0;
            if (xa[u] & 0x100u) {  // a real edge
              const uint32_t xv = xa[u] & 0xFFu;
              if (vh[u] >> 31) xout[vh[u] >> 8 & 0x7FFFFFu] = (uint8_t)xv;
              if (xv != 0) contrib = GE[GL[vh[u] & 0xFFu] + GL[xv]];
            }
            if (want_syn) {
#pragma unroll
              for (int o = 1; o < 32; o <<= 1)
                if (o < KT) contrib ^= __shfl_xor_sync(0xffffffffu, contrib, o);
              badc |= (int)contrib;
            }
          }
        }
        return badc;
      };
      if (step) {
        if (SPLITDEC_CT && split && do_dec) {
          cluster_sync_all();  // every nibble of the frame is written
          (void)split_pass_end(false);
        }
        break;
      }

      // ---- end of the pass: stopping rule, cluster-uniform
      asm volatile("fence.proxy.async.global;" ::: "memory");  // W_out is read next by bulk copies
      cluster_sync_all();  // every message, estimate and syndrome byte of the pass is written
      if (tid == 0) sh_bad = 0;
      __syncthreads();
      if (SPLITDEC_CT && split && ell >= 1) {
        // lazy decision: a pass with an unsatisfied probe check (or without a stopping rule) does not stop the frame;
        // sh_skip is final here (local and remote writes precede the cluster barrier above)
        const bool skipped = lazy && (lazy_all || *reinterpret_cast<volatile int*>(&sh_skip) == ps);
        if (skipped) {
          if (tid == 0) dsmem_or((ell & 1) ? flag1 : flag0, 1);
        } else {
          const int bad = split_pass_end(true);
          if (__syncthreads_or(bad != 0) && tid == 0) dsmem_or((ell & 1) ? flag1 : flag0, 1);
        }
      } else if (ell >= 1) {
        // my checks' syndromes s_c = XOR of the contribution bytes on their kpad edge slots
        int bad = 0;
        const int kp = KPAD;
        for (int i = tid; i < nch * CPC; i += nthr) {
          const int kc = i / CPC, l = i - kc * CPC;
          const int c = ((int)rank + kc * (int)csz) * CPC + l;
          if (c >= cd.M) continue;
          const uint32_t* cs = reinterpret_cast<const uint32_t*>(con + (size_t)c * kp);
          uint32_t acc = 0;
          for (int w = 0; w < kp / 4; ++w) acc ^= __ldcg(cs + w);
          acc ^= acc >> 16;
          acc ^= acc >> 8;
          bad |= (int)(acc & 0xFFu);
        }
        if (__syncthreads_or(bad != 0) && tid == 0) dsmem_or((ell & 1) ? flag1 : flag0, 1);
      }
      if (rank == 0 && tid == 0) sh_flag[(ell + 1) & 1] = 0;  // read before this pass by everyone
      cluster_sync_all();
      int ok = 0;
      if (ell >= 1) ok = dsmem_ld((ell & 1) ? flag1 : flag0) == 0;
      const bool done = (ell >= 1 && call->early_stop && ok) || ell >= max_iters;
      if (done) {
        if (rank == 0 && tid == 0) {
          call->ok[f] = (uint8_t)ok;
          call->iters[f] = ell;
          if (call->events_out) call->events_out[f] = ws.slot_events[slot];
          ws.slot_events[slot] = 0;
        }
        break;
      }
    }
    if (step) continue;
  }
  cp_async_wait<0>();
  // no CTA may exit while others can still address its shared memory
  if (!step) cluster_sync_all();
}

// message layout conversion for nbldpc_step: natural order (message of edge e in slot e) <-> the
// cluster kernel's reader-ordered rows (message of edge e in row partner(e), entries at mpos)
// lin = 1: the kernel's messages are linear (LIN instantiations), the step format packed log
template <int MB>
__global__ void nb_msg_layout_kernel(const float* src, float* dst, int frames, CodeDev cd, int to_kernel, int lin) {
  constexpr int Q = 1 << MB;
  const size_t n = (size_t)frames * cd.E * Q;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t fe = i / Q;
    const int z = (int)(i % Q);
    const int e = (int)(fe % cd.E);
    const size_t f = fe / cd.E;
    const EdgeDev& ed = cd.edges[e];
    if (ed.var < 0) continue;
    const size_t k = (f * cd.E + ed.partner) * Q + mpos<MB>(z, ed.partner);
    if (to_kernel) dst[k] = lin ? to_lin(src[i]) : src[i];
    else dst[i] = lin ? lin_to_packed(src[k]) : src[k];
  }
}

}  // namespace nb
