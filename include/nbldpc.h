/*
 * nbldpc.h -- C-ABI of the B200-native (sm_100a) batched Log-Fourier SP decoder
 * for (j=2,k)-regular non-binary LDPC codes over GF(2^m), arXiv:1008.4370 (and, beyond the
 * paper's (2,k) codes, any column weight 1..16; plus the conventional Log-SP it compares with).
 *
 * The decoder runs the paper's Log-Fourier sum-product iteration
 * (section 3.2): messages are 2^m-point Walsh-Hadamard spectra
 * held as (sign, log-magnitude); the check node is a leave-one-out sum of
 * log-magnitudes with a sign XOR after the index permutation z -> H_cv z
 * (Appendix A :672); the degree-2 variable node is the signed
 * log-convolution with the channel spectrum; the tentative
 * decision uses the paper's fast bit rule and the decoder
 * stops on a zero syndrome.
 *
 * All functions are plain C; no C++ exception crosses the ABI.  Every entry
 * point returns a status; on error nothing is written to any output buffer and
 * no kernel has been launched (validation precedes all launches), except
 * NBLDPC_ERR_CUDA which reports a failed CUDA call (sticky device errors
 * included).  Symbols: bit r of a symbol is the coefficient of alpha^r
 * (PAPER.md:105-108).  Edges are numbered in "canonical order": the nonzeros of
 * H sorted by (row, col).
 */
#ifndef NBLDPC_H
#define NBLDPC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nbldpc_code_s* nbldpc_code_t;

typedef enum {
  NBLDPC_OK = 0,
  NBLDPC_ERR_INVALID_ARGUMENT = -1, /* NULL pointer, m not in [1,8], M/N/nnz <= 0, index out of range,
                                       coefficient not in [1, 2^m-1], frames < 1, max_iters < 1,
                                       host pointer where a device pointer is required (or vice versa) */
  NBLDPC_ERR_NOT_PRIMITIVE = -2,    /* prim_poly not of degree m, or alpha's period != 2^m - 1 */
  NBLDPC_ERR_UNSUPPORTED = -3,      /* a column weight outside 1..16, duplicate (row, col), a row degree
                                       < 2, a row degree too large for one thread block, or an option
                                       combination a code does not support (see the options) */
  NBLDPC_ERR_CUDA = -4,             /* a CUDA runtime call failed */
  NBLDPC_ERR_OUT_OF_MEMORY = -5     /* device or pinned host allocation failed */
} nbldpc_status_t;

typedef enum {
  NBLDPC_SYNDROME_EXACT = 0, /* s_c = sum_v h_cv xhat_v over GF(2^m); the default */
  NBLDPC_SYNDROME_PAPER = 1  /* the paper's fast Fourier-domain syndrome */
} nbldpc_syndrome_mode_t;

/* How the variable node evaluates the signed log-convolution U = Lambda^0 [+] W.
 * Both compute the same result up to rounding. */
typedef enum {
  NBLDPC_VN_SEPARABLE = 0, /* default: the binary-image channel spectrum is the tensor product
                              P^0 = (x)_i (1, tanh(L_i/2)), so the XOR-
                              convolution factors into m butterfly stages x(z) += t_i x(z ^ alpha^i):
                              m 2^m FMAs per edge */
  NBLDPC_VN_DIRECT = 1,    /* the paper's CONV (Table 1): 2^{2m} FMAs per edge */
  NBLDPC_VN_GENERAL = 2    /* any column weight: the (d-1)-fold convolution in the probability
                              domain, U_i = WHT(p^0 prod_{i' != i} WHT(W_i') / 2^m), one CTA per frame; always
                              used when some column weight is not 2 (the paper syndrome mode is then
                              unavailable) */
} nbldpc_vn_algorithm_t;

/* Decoding algorithm (nbldpc_decode_opts_t::algorithm). */
typedef enum {
  NBLDPC_ALG_LOG_FOURIER = 0, /* the paper's Log-Fourier SP: the hot path */
  NBLDPC_ALG_LOG_SP = 1       /* the conventional Log-SP it is compared with: log-domain
                                 messages, check node = leave-one-out log-convolutions (forward-backward,
                                 3(k-2) q^2-term log-convolutions per check), symbol-MAP decisions
                                 argmax_x mu_v(x) (:271-276), exact-syndrome stop.  Same outputs as SP
                                 (:279); soft_out, events_out, the symbol outputs and the paper syndrome
                                 mode are not available (NBLDPC_ERR_INVALID_ARGUMENT) */
} nbldpc_algorithm_t;

/* Storage format of the messages in HBM / L2 (nbldpc_decode_opts_t::message_format). */
typedef enum {
  NBLDPC_MSG_F32 = 0, /* float32 (sign bit | -log2|x|): the reference precision */
  NBLDPC_MSG_F16 = 1  /* IEEE half, same packing: half the message bytes (the paper's reduced-precision
                         motivation); arithmetic stays fp32.  Only the Log-Fourier cluster
                         kernel (NBLDPC_VN_SEPARABLE, LLR input, column weight 2, m >= 3; else
                         NBLDPC_ERR_INVALID_ARGUMENT / NBLDPC_ERR_UNSUPPORTED).  Results are not
                         bit-identical to F32: evaluated by frame error rate */
} nbldpc_message_format_t;

/* Options of nbldpc_decode_ex / nbldpc_decode_host.  Zero-initialise, then set
 * struct_size = sizeof(nbldpc_decode_opts_t).  NULL opts = all defaults. */
typedef struct {
  size_t struct_size;
  int syndrome_mode; /* nbldpc_syndrome_mode_t, default EXACT */
  int no_early_stop; /* 0 (default): stop a frame at its first zero syndrome;
                        1: always run max_iters iterations (diagnostic timing only) */
  float* soft_out;   /* device, [frames][N*m] or NULL: ln|M_v(alpha^i)/M_v(0)| at the stopping
                        iteration (posterior bit log-magnitudes) */
  int32_t* events_out; /* device, [frames] or NULL: numerical events (variable-node DC term <= 0) */
  int slots;         /* frames resident on the device at once (0 = library default, sized to L2) */
  int use_graph;     /* 0 = default (CUDA graph with a device-side WHILE loop), 1 = force graph,
                        -1 = host-driven launch loop */
  int vn_algorithm;  /* nbldpc_vn_algorithm_t, default NBLDPC_VN_SEPARABLE */
  float* symbol_post_out;   /* device, 16-byte aligned, [frames][N][2^m] or NULL: the symbol posterior
                               mu_v(x) / sum_x mu_v(x), mu_v(x) = sum_z M_v(z) (-1)^{z.x}, at the
                               stopping iteration */
  uint8_t* symbol_map_out;  /* device, [frames][N] or NULL: argmax_x mu_v(x), ties -> lowest x
                               (the paper's symbol-level TENTATIVE DECISION) */
  /* The symbol decision is evaluated at every iteration (the stopping one is not known in advance;
   * 2 WHTs of size 2^m per variable) and written to the frame's output rows each time, so the last
   * write is the stopping iteration's; the rows hold intermediate values until the decode completes.
   * With LLR input it runs inside the cluster kernel (its symbol-output variant, NBLDPC_VN_SEPARABLE);
   * with symbol-pmf input (nbldpc_decode_pmf) it selects the slot-pass kernel (NBLDPC_VN_DIRECT). */
  int algorithm;     /* nbldpc_algorithm_t, default NBLDPC_ALG_LOG_FOURIER */
  int message_format; /* nbldpc_message_format_t, default NBLDPC_MSG_F32 */
  /* --- since round 2 (callers built against the older, shorter struct keep working: fields past
   *     their struct_size read as zero) --- */
  void* workspace;        /* DEVICE, 256-byte aligned, or NULL (default: the handle's own workspace).
                             Caller-provided workspace of at least nbldpc_workspace_bytes(code, frames)
                             bytes for nbldpc_decode_ex with LLR input on the cluster kernel
                             (NBLDPC_VN_SEPARABLE, column weight 2); other entry points / paths return
                             NBLDPC_ERR_UNSUPPORTED.  The caller owns it; it must not be used by another
                             decode until this one completes on `stream`.  A decode with its own
                             workspace writes nothing of the handle and takes no handle lock, so decodes
                             with distinct workspaces may run concurrently on distinct streams. */
  size_t workspace_bytes; /* size of `workspace` (NBLDPC_ERR_INVALID_ARGUMENT if too small) */
} nbldpc_decode_opts_t;

/* Builds a code from H given as nnz (row, col, coefficient) triplets in any order.
 *   m         : field GF(2^m), 1 <= m <= 8
 *   prim_poly : primitive polynomial as a full mask including x^m (e.g. 0x7, 0x13, 0x43, 0x11D)
 *   M, N      : H is M x N
 *   rows, cols, coeffs : HOST arrays of length nnz, 0-based indices, coefficients in [1, 2^m-1]
 *   out       : receives the handle (caller owns it; release with nbldpc_destroy)
 * Every column must have 1..16 nonzeros in distinct rows and every row at least two; row degree times
 * max(1, 2^m/16) must not exceed 512 (one check per thread block).  Column weight 2
 * everywhere (the (2,k) codes of PAPER.md:36-41) runs the Log-Fourier cluster kernel; any other column
 * weight ("the extension ... is straightforward") runs NBLDPC_VN_GENERAL, for which
 * nbldpc_step and NBLDPC_ALG_LOG_SP are unavailable (NBLDPC_ERR_UNSUPPORTED).  The handle copies H, builds its device tables (GF tables, canonical edge list,
 * Fourier permutation bases) on the CUDA device current at the call, and is
 * immutable afterwards.  Decoding must happen on that device.
 * Length: each CTA of the cluster kernel keeps 8-byte records of its share of the edge slots in shared
 * memory; long codes get larger clusters (up to 16 CTAs per frame).  A code whose share still exceeds
 * the 227 KB of shared memory (about E * 2^m > 16 * 227 KB * 2^m / 8 bytes of edge records, i.e. tens
 * of thousands of symbols) is accepted and decoded by the general-column-weight kernel (same results
 * up to rounding); nbldpc_step with NBLDPC_VN_SEPARABLE, NBLDPC_MSG_F16 and caller workspaces are then
 * NBLDPC_ERR_UNSUPPORTED.  Edge slots must fit 22 bits (M * kpad < 2^22, kpad = the next power of two
 * >= max(4, largest row degree)). */
nbldpc_status_t nbldpc_code_create(int m, uint32_t prim_poly, int M, int N, int nnz, const int32_t* rows,
                                   const int32_t* cols, const uint16_t* coeffs, nbldpc_code_t* out);

/* Releases the handle and everything it allocated.  NULL is a no-op.  Waits (host side) for the last
 * decode that used the handle's own workspace to complete before releasing it; decodes that ran with a
 * caller-provided workspace must have completed (synchronise their streams first). */
void nbldpc_destroy(nbldpc_code_t code);

/* Human-readable text of a status (static storage). */
const char* nbldpc_status_string(nbldpc_status_t s);

/* Name and text of the last CUDA error that made a call on this thread return NBLDPC_ERR_CUDA or
 * NBLDPC_ERR_OUT_OF_MEMORY ("" if none).  Thread-local storage, valid until the next call. */
const char* nbldpc_last_cuda_error(void);

/* Code dimensions (any pointer may be NULL): field degree m, rows M, columns N, edges E = nnz (2N for column weight 2),
 * largest row degree k_max. */
nbldpc_status_t nbldpc_code_info(nbldpc_code_t code, int* m, int* M, int* N, int* E, int* k_max);

/* Device bytes the decoder keeps per resident frame slot (messages, channel terms, estimates). */
size_t nbldpc_slot_bytes(nbldpc_code_t code);

/* Device bytes of the workspace a default nbldpc_decode of `frames` frames keeps on this handle
 * (min(frames, resident clusters) slots of about nbldpc_slot_bytes each, plus the per-call control
 * block) -- also the size a caller-provided nbldpc_decode_opts_t::workspace needs; 0 for a NULL code,
 * frames < 1, or a code the cluster kernel does not run (column weight other than 2, or too long, see
 * nbldpc_code_create: the general kernel sizes a workspace per call from the occupancy).  The handle's
 * workspace is allocated by the first decode and re-carved when the slot count changes, stream-ordered
 * on the decode's stream (cudaFreeAsync / cudaMallocAsync after the handle's previous decode, wherever
 * it ran -- no device-wide synchronisation); it is released by nbldpc_destroy. */
size_t nbldpc_workspace_bytes(nbldpc_code_t code, int frames);

/* Number of kernels the most recent decode on this handle launched (setup, pass and control
 * kernels).  Synchronises the stream of that decode.  0 before the first decode. */
nbldpc_status_t nbldpc_last_decode_launches(nbldpc_code_t code, long long* launches);

/* Decodes `frames` independent frames (the hot path).
 *   llr          : DEVICE, float32 [frames][N*m]; LLR = ln Pr(b=0|y)/Pr(b=1|y) of bit i of symbol v at
 *                  index v*m + i (binary image of the codeword)
 *   max_iters    : >= 1, the iteration limit l_max of PAPER.md:144
 *   hard_symbols : DEVICE, uint8 [frames][N]; the fast-rule estimate at the stopping iteration
 *   syndrome_ok  : DEVICE, uint8 [frames]; 1 iff the syndrome of that estimate is zero
 *   iters_used   : DEVICE, int32 [frames]; the stopping iteration, in [1, max_iters]
 *   stream       : cudaStream_t (NULL = legacy default stream)
 * Stream-ordered: returns after enqueueing; outputs are valid when `stream` reaches that point.
 * Results depend only on (code, llr row, max_iters, options), not on frames, batching or slots.
 * Calls sharing one handle's workspace are serialised by a lock and by stream order (a decode whose
 * slot count differs re-carves the workspace after the previous one completes, stream-ordered); give
 * each concurrent stream its own nbldpc_decode_opts_t::workspace to overlap decodes of one handle. */
nbldpc_status_t nbldpc_decode(nbldpc_code_t code, const float* llr, int frames, int max_iters,
                              uint8_t* hard_symbols, uint8_t* syndrome_ok, int32_t* iters_used, void* stream);

/* nbldpc_decode with options (opts may be NULL). */
nbldpc_status_t nbldpc_decode_ex(nbldpc_code_t code, const float* llr, int frames, int max_iters,
                                 uint8_t* hard_symbols, uint8_t* syndrome_ok, int32_t* iters_used, void* stream,
                                 const nbldpc_decode_opts_t* opts);

/* End-to-end variant with HOST buffers: copies llr_host (float32 [frames][N*m], pinned memory
 * recommended) to the device, decodes, copies the results back to the host arrays
 * (hard_host [frames][N], ok_host [frames], iters_host [frames]) and synchronises `stream`
 * before returning.  opts->soft_out / events_out are ignored here.  On the cluster-kernel path the
 * host-to-device copy runs in up to 16 chunks on an internal copy stream, overlapped with the decode
 * (the kernel starts after the first chunk; a frame of a later chunk is taken only after its chunk's
 * arrival flag is raised by a stream memory write).  NBLDPC_NO_OVERLAP=1 in the environment disables it. */
nbldpc_status_t nbldpc_decode_host(nbldpc_code_t code, const float* llr_host, int frames, int max_iters,
                                   uint8_t* hard_host, uint8_t* ok_host, int32_t* iters_host, void* stream,
                                   const nbldpc_decode_opts_t* opts);

/* Decodes `frames` frames from a general symbol-level channel pmf (the
 * initialisation P_v^(0)(z) = sum_x p_v^(0)(x) (-1)^{z.x}, for channels whose prior does not factor
 * over the bits -- q-ary modulations, symbol erasures, soft symbol demappers).
 *   pmf : DEVICE, float32 [frames][N][2^m]; entry x of row (frame, v) is a nonnegative weight of
 *         Pr(X_v = x | Y_v).  Any positive scale per row is allowed: the row is scaled to sum to one
 *         (reading R23).  A row whose sum is not positive is treated as uniform and counted as a
 *         numerical event (opts->events_out), as are the iterations it stays degenerate in.
 *   the other arguments as nbldpc_decode_ex; soft_out holds the same posterior bit log-magnitudes.
 * The channel spectrum of a general pmf is not a tensor product, so the variable node runs in the
 * probability domain (XOR-convolution theorem): raw = WHT(p_v . WHT(W_e')) / 2^m, 2m butterfly stages
 * per entry.  opts->vn_algorithm picks the kernel: NBLDPC_VN_SEPARABLE (default) the cluster-per-frame
 * kernel of nbldpc_decode, NBLDPC_VN_DIRECT the slot-pass kernel (also selected by the symbol outputs).
 * The scaled rows are kept in a per-slot buffer of N*2^m floats (allocated on first use, released
 * with the handle).
 * pmf must be 16-byte aligned (NBLDPC_ERR_INVALID_ARGUMENT otherwise).
 * Stream-ordered; same results-independence and stream rules as nbldpc_decode. */
nbldpc_status_t nbldpc_decode_pmf(nbldpc_code_t code, const float* pmf, int frames, int max_iters,
                                  uint8_t* hard_symbols, uint8_t* syndrome_ok, int32_t* iters_used, void* stream,
                                  const nbldpc_decode_opts_t* opts);

/* nbldpc_decode_pmf with HOST buffers, as nbldpc_decode_host: pmf_host float32 [frames][N][2^m] (pinned
 * recommended), results to the host arrays; the copy overlaps the decode on the cluster-kernel path. */
nbldpc_status_t nbldpc_decode_pmf_host(nbldpc_code_t code, const float* pmf_host, int frames, int max_iters,
                                       uint8_t* hard_host, uint8_t* ok_host, int32_t* iters_host, void* stream,
                                       const nbldpc_decode_opts_t* opts);

/* One Log-Fourier iteration from a given state (step-parity tests; not on the hot path).
 * Requires every row of H to have the same degree k, a power of two >= 4 (else
 * NBLDPC_ERR_UNSUPPORTED): then the decoder's internal edge slots coincide with canonical order.
 * Message format (w_in, w_out, u_out): float32 [frames][E][2^m], edge e in canonical order; entry z
 * holds |Gamma| as the non-negative value -log2|x| (0 = magnitude 1, >= 126 = zero) and the message
 * sign in the IEEE sign bit.
 *   iter == 0 : computes W^(1) = CHECK-TO-VARIABLE(Lambda^(0)); w_in, u_out,
 *               hard, soft are not used.
 *   iter >= 1 : given W^(iter) in w_in, computes U^(iter) = VARIABLE-TO-CHECK (u_out, optional),
 *               the tentative decision (hard [frames][N], soft [frames][N*m] optional) and
 *               W^(iter+1) = CHECK-TO-VARIABLE(U^(iter)) in w_out.
 * vn_algorithm: nbldpc_vn_algorithm_t.  All pointers are DEVICE pointers; llr as for
 * nbldpc_decode.  Stream-ordered. */
nbldpc_status_t nbldpc_step(nbldpc_code_t code, const float* llr, int frames, int iter, const float* w_in,
                            float* w_out, float* u_out, uint8_t* hard, float* soft, int vn_algorithm, void* stream);

/* nbldpc_step for symbol-pmf input (the Log-Fourier cluster kernel's pmf variant, NBLDPC_VN_SEPARABLE):
 * pmf as for nbldpc_decode_pmf (DEVICE, float32 [frames][N][2^m], 16-byte aligned, rows scaled to
 * probabilities); the other arguments as nbldpc_step.  Same code requirements;
 * NBLDPC_ERR_UNSUPPORTED where the cluster kernel does not run the code. */
nbldpc_status_t nbldpc_step_pmf(nbldpc_code_t code, const float* pmf, int frames, int iter, const float* w_in,
                                float* w_out, float* u_out, uint8_t* hard, float* soft, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NBLDPC_H */
