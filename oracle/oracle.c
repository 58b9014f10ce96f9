/*
 * oracle/oracle.c -- CPU ORACLE for arXiv:1008.4370, "Log-SP in the Fourier
 * domain" decoding of (j=2,k)-regular non-binary LDPC codes over GF(2^m).
 *
 * ===================== TEST INFRASTRUCTURE ONLY =====================
 * This file is the correctness reference. It is NOT part of the product.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load it (through oracle/__init__.py).
 * It shares no code, header, table or constant generator with the CUDA
 * path in paper_1008_4370_b200/ and neither side includes the other.
 * =====================================================================
 *
 * Style: plain, slow, obviously correct.  Every function follows one passage
 * of /root/reference/PAPER.md (cited as PAPER.md:<line>, with the section) in
 * the paper's order and notation.  No blocking, fusion or reordering beyond
 * what the cited definition states.  Floating point is double (fp64) unless a
 * function name ends in _f32 (the float32 diagnostic twin of the Log-Fourier
 * decoder, used only to classify "stable frames", reading R20).
 *
 * Conventions (readings of the paper, listed in DESIGN.md section 3):
 *  - symbols are integers 0..q-1, bit r = coefficient of alpha^r
 *    (the GF(8) listing; alpha^{i-1} = 1 << (i-1)).
 *  - LLR convention L = ln Pr(b=0|y)/Pr(b=1|y); bit i of symbol v is llr[v*m+i].
 *  - Gamma(x) = (sgn, ln|x|) with sgn(0) = 0 and ln 0 encoded as the floor
 *    OR_FLOOR = -745 (reading R6, R7).
 *  - edges are numbered in canonical order: nonzeros of H sorted by
 *    (row, col); a variable's edges are taken in that order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_FLOOR (-745.0)
#define OR_MAXM 10

/* ------------------------------------------------------------------ */
/* GF(2^m): PAPER.md:100-108 (section 2, m-bit representation)         */
/* ------------------------------------------------------------------ */
typedef struct {
  int m, q;
  unsigned poly;             /* full mask including x^m, e.g. 0xB for x^3+x+1 */
  int exp_t[1 << OR_MAXM];   /* exp_t[i] = alpha^i as an m-bit integer, i < q-1 */
  int log_t[1 << OR_MAXM];   /* log_t[x] = i with alpha^i = x, x != 0 */
  /* perm[h][z] = H_cv z with H_cv = (A^i)^T, h = alpha^i (Appendix A) */
  int* perm;                 /* q*q entries; row 0 unused */
  int* perm_inv;             /* perm_inv[h][perm[h][z]] = z (inverse permutation) */
} or_field;

/* alpha^{i+1} = alpha * alpha^i: shift the polynomial and reduce by the
 * primitive polynomial pi(x).  Returns 0 on success, -1 if the
 * polynomial is not of degree m or alpha has period != 2^m - 1 (not primitive). */
static int field_tables(or_field* f) {
  int q = f->q, m = f->m;
  if (m < 1 || m > OR_MAXM) return -1;
  if ((f->poly >> m) != 1u) return -1;
  for (int x = 0; x < q; ++x) f->log_t[x] = -1;
  int a = 1;
  for (int i = 0; i < q - 1; ++i) {
    if (i > 0 && a == 1) return -1; /* period shorter than 2^m-1 */
    if (f->log_t[a] != -1) return -1;
    f->exp_t[i] = a;
    f->log_t[a] = i;
    a <<= 1;
    if (a & q) a ^= (int)f->poly;
  }
  if (a != 1) return -1;
  return 0;
}

int or_gf_mul(const or_field* f, int a, int b) {
  if (a == 0 || b == 0) return 0;
  return f->exp_t[(f->log_t[a] + f->log_t[b]) % (f->q - 1)];
}
int or_gf_inv(const or_field* f, int a) {
  if (a == 0) return -1;
  return f->exp_t[(f->q - 1 - f->log_t[a]) % (f->q - 1)];
}
int or_gf_add(int a, int b) { return a ^ b; }
int or_field_exp(const or_field* f, int i) { return f->exp_t[((i % (f->q - 1)) + (f->q - 1)) % (f->q - 1)]; }
int or_field_log(const or_field* f, int x) { return x ? f->log_t[x] : -1; }

/* Companion matrix of alpha, PAPER.md:662-666 (Appendix A):
 *   A = [[0,...,0,pi_0],[1,0,...,0,pi_1],...,[0,...,1,pi_{m-1}]],
 * i.e. A[r][c] = 1 if r == c+1, and A[r][m-1] = pi_r.  A^i alpha^j = alpha^{i+j}
 * (PAPER.md:669). */
static void companion(const or_field* f, unsigned char A[OR_MAXM][OR_MAXM]) {
  int m = f->m;
  memset(A, 0, sizeof(unsigned char) * OR_MAXM * OR_MAXM);
  for (int r = 1; r < m; ++r) A[r][r - 1] = 1;
  for (int r = 0; r < m; ++r) A[r][m - 1] ^= (unsigned char)((f->poly >> r) & 1u);
}
static void matmul2(int m, unsigned char X[OR_MAXM][OR_MAXM], unsigned char Y[OR_MAXM][OR_MAXM],
                    unsigned char Z[OR_MAXM][OR_MAXM]) {
  unsigned char T[OR_MAXM][OR_MAXM];
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < m; ++c) {
      int s = 0;
      for (int t = 0; t < m; ++t) s ^= X[r][t] & Y[t][c];
      T[r][c] = (unsigned char)s;
    }
  memcpy(Z, T, sizeof(T));
}
/* (A^i)^T as an m x m 0/1 matrix, row-major into out[m*m]. */
void or_companion_pow_T(const or_field* f, int i, unsigned char* out) {
  unsigned char A[OR_MAXM][OR_MAXM], P[OR_MAXM][OR_MAXM];
  int m = f->m;
  companion(f, A);
  memset(P, 0, sizeof(P));
  for (int r = 0; r < m; ++r) P[r][r] = 1;
  for (int s = 0; s < i; ++s) matmul2(m, P, A, P);
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < m; ++c) out[r * m + c] = P[c][r];
}
/* apply an m x m binary matrix (row-major) to the bit vector of z over GF(2) */
int or_apply_binary_matrix(int m, const unsigned char* Mx, int z) {
  int y = 0;
  for (int r = 0; r < m; ++r) {
    int s = 0;
    for (int c = 0; c < m; ++c) s ^= Mx[r * m + c] & ((z >> c) & 1);
    y |= s << r;
  }
  return y;
}

or_field* or_field_new(int m, unsigned poly) {
  if (m < 1 || m > OR_MAXM) return NULL;
  or_field* f = (or_field*)calloc(1, sizeof(or_field));
  f->m = m;
  f->q = 1 << m;
  f->poly = poly;
  if (field_tables(f) != 0) { free(f); return NULL; }
  int q = f->q;
  f->perm = (int*)calloc((size_t)q * q, sizeof(int));
  f->perm_inv = (int*)calloc((size_t)q * q, sizeof(int));
  unsigned char HT[OR_MAXM * OR_MAXM];
  for (int h = 1; h < q; ++h) {
    or_companion_pow_T(f, f->log_t[h], HT); /* H_cv = (A^i)^T for h = alpha^i */
    for (int z = 0; z < q; ++z) f->perm[h * q + z] = or_apply_binary_matrix(m, HT, z);
    for (int z = 0; z < q; ++z) f->perm_inv[h * q + f->perm[h * q + z]] = z;
  }
  return f;
}
void or_field_free(or_field* f) {
  if (!f) return;
  free(f->perm);
  free(f->perm_inv);
  free(f);
}
int or_field_q(const or_field* f) { return f->q; }
/* z -> H_cv z for h_cv = h */
int or_fourier_perm(const or_field* f, int h, int z) { return f->perm[h * f->q + z]; }
int or_fourier_perm_inv(const or_field* f, int h, int z) { return f->perm_inv[h * f->q + z]; }

/* dot product parity of the binary representations */
int or_dot_parity(int z, int x) {
  int s = 0;
  for (int b = z & x; b; b >>= 1) s ^= b & 1;
  return s;
}

/* ------------------------------------------------------------------ */
/* Transforms: PAPER.md:174-177 (convolution), :209-219 (Fourier pair),*/
/* :450-463 (Gamma), :489-494 (signed log-convolution)                 */
/* ------------------------------------------------------------------ */
/* P(z) = sum_x p(x) (-1)^{z.x}, direct O(q^2) sum */
void or_wht(int m, const double* p, double* P) {
  int q = 1 << m;
  for (int z = 0; z < q; ++z) {
    double s = 0.0;
    for (int x = 0; x < q; ++x) s += or_dot_parity(z, x) ? -p[x] : p[x];
    P[z] = s;
  }
}
/* q(x) = 2^{-m} sum_z Q(z) (-1)^{z.x}   (sum read over z) */
void or_iwht(int m, const double* Q, double* p) {
  int q = 1 << m;
  for (int x = 0; x < q; ++x) {
    double s = 0.0;
    for (int z = 0; z < q; ++z) s += or_dot_parity(z, x) ? -Q[z] : Q[z];
    p[x] = s / (double)q;
  }
}
/* (p1 (x) p2)(x) = sum_{x1 + x2 = x} p1(x1) p2(x2) */
void or_convolve(int m, const double* p1, const double* p2, double* out) {
  int q = 1 << m;
  for (int x = 0; x < q; ++x) out[x] = 0.0;
  for (int x1 = 0; x1 < q; ++x1)
    for (int x2 = 0; x2 < q; ++x2) out[x1 ^ x2] += p1[x1] * p2[x2];
}
/* Gamma(x) = (sgn_GF2(x), ln|x|); sgn(0) = 0, ln 0 = floor */
void or_gamma(double x, int* s, double* l) {
  *s = x < 0.0 ? 1 : 0;
  if (x == 0.0) {
    *l = OR_FLOOR;
  } else {
    double v = log(fabs(x));
    *l = v < OR_FLOOR ? OR_FLOOR : v;
  }
}
double or_gamma_inv(int s, double l) {
  if (l <= OR_FLOOR) return 0.0;
  double v = exp(l);
  return s ? -v : v;
}
/* Signed log-convolution:
 *   (L1 [+] L2)(x) = Gamma( sum_{x1+x2=x} Gamma^{-1}( L1(x1) + L2(x2) ) ),
 * where + on (GF(2) x R) adds the sign bits in GF(2) and the log-magnitudes
 * in R.  Evaluated literally, one signed exp per term, positive and negative
 * mass accumulated separately. */
void or_boxplus(int m, const int* s1, const double* l1, const int* s2, const double* l2, int* so, double* lo) {
  int q = 1 << m;
  for (int x = 0; x < q; ++x) {
    double pos = 0.0, neg = 0.0;
    for (int x1 = 0; x1 < q; ++x1) {
      int x2 = x ^ x1;
      if (l1[x1] <= OR_FLOOR || l2[x2] <= OR_FLOOR) continue; /* Gamma^{-1}(s, floor) = 0 */
      double t = exp(l1[x1] + l2[x2]);
      if (s1[x1] ^ s2[x2]) neg += t; else pos += t;
    }
    or_gamma(pos - neg, &so[x], &lo[x]);
  }
}

/* ------------------------------------------------------------------ */
/* Code: H over GF(2^m), Tanner graph V_c / C_v    */
/* ------------------------------------------------------------------ */
typedef struct {
  const or_field* f;
  int M, N, E;
  int* e_row;     /* edge -> check c */
  int* e_col;     /* edge -> variable v */
  int* e_h;       /* edge -> h_cv */
  int* c_ptr;     /* check c owns edges c_ptr[c] .. c_ptr[c+1]-1 (canonical order) */
  int* v_ptr;     /* variable v owns v_edges[v_ptr[v] .. v_ptr[v+1]-1] */
  int* v_edges;
} or_code;

static int cmp_rc(const void* a, const void* b) {
  const int* x = (const int*)a;
  const int* y = (const int*)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
  return 0;
}

/* Builds the Tanner graph.  Returns NULL on invalid input (index out of range,
 * coefficient not in 1..q-1, duplicate (row, col)).  Column weights >= 1 are
 * allowed here (the tree pin of tests/ uses weight-1 leaves). */
or_code* or_code_new(const or_field* f, int M, int N, int nnz, const int* rows, const int* cols, const int* coeffs) {
  if (!f || M <= 0 || N <= 0 || nnz <= 0) return NULL;
  int* trip = (int*)malloc(sizeof(int) * 3 * (size_t)nnz);
  for (int i = 0; i < nnz; ++i) {
    if (rows[i] < 0 || rows[i] >= M || cols[i] < 0 || cols[i] >= N || coeffs[i] < 1 || coeffs[i] >= f->q) {
      free(trip);
      return NULL;
    }
    trip[3 * i] = rows[i];
    trip[3 * i + 1] = cols[i];
    trip[3 * i + 2] = coeffs[i];
  }
  qsort(trip, (size_t)nnz, 3 * sizeof(int), cmp_rc);
  for (int i = 1; i < nnz; ++i)
    if (trip[3 * i] == trip[3 * i - 3] && trip[3 * i + 1] == trip[3 * i - 2]) { free(trip); return NULL; }
  or_code* c = (or_code*)calloc(1, sizeof(or_code));
  c->f = f;
  c->M = M;
  c->N = N;
  c->E = nnz;
  c->e_row = (int*)malloc(sizeof(int) * nnz);
  c->e_col = (int*)malloc(sizeof(int) * nnz);
  c->e_h = (int*)malloc(sizeof(int) * nnz);
  c->c_ptr = (int*)calloc((size_t)M + 1, sizeof(int));
  c->v_ptr = (int*)calloc((size_t)N + 1, sizeof(int));
  c->v_edges = (int*)malloc(sizeof(int) * nnz);
  for (int e = 0; e < nnz; ++e) {
    c->e_row[e] = trip[3 * e];
    c->e_col[e] = trip[3 * e + 1];
    c->e_h[e] = trip[3 * e + 2];
    c->c_ptr[c->e_row[e] + 1]++;
    c->v_ptr[c->e_col[e] + 1]++;
  }
  free(trip);
  for (int i = 0; i < M; ++i) c->c_ptr[i + 1] += c->c_ptr[i];
  for (int i = 0; i < N; ++i) c->v_ptr[i + 1] += c->v_ptr[i];
  int* fill = (int*)calloc((size_t)N, sizeof(int));
  for (int e = 0; e < nnz; ++e) {
    int v = c->e_col[e];
    c->v_edges[c->v_ptr[v] + fill[v]++] = e;
  }
  free(fill);
  return c;
}
void or_code_free(or_code* c) {
  if (!c) return;
  free(c->e_row); free(c->e_col); free(c->e_h); free(c->c_ptr); free(c->v_ptr); free(c->v_edges);
  free(c);
}
int or_code_E(const or_code* c) { return c->E; }
/* canonical edge list export (for tests): rows, cols, coeffs in canonical order */
void or_code_edges(const or_code* c, int* rows, int* cols, int* coeffs) {
  for (int e = 0; e < c->E; ++e) { rows[e] = c->e_row[e]; cols[e] = c->e_col[e]; coeffs[e] = c->e_h[e]; }
}

/* syndrome s_c = sum_{v in V_c} h_cv x_v over GF(2^m).
 * Returns 1 iff all s_c = 0, i.e. x is a codeword. */
int or_code_syndrome(const or_code* c, const int* x, int* s) {
  int ok = 1;
  for (int r = 0; r < c->M; ++r) {
    int acc = 0;
    for (int e = c->c_ptr[r]; e < c->c_ptr[r + 1]; ++e) acc = or_gf_add(acc, or_gf_mul(c->f, c->e_h[e], x[c->e_col[e]]));
    if (s) s[r] = acc;
    if (acc) ok = 0;
  }
  return ok;
}

/* Gaussian-elimination encoder (BASELINE.json north_star: "Gaussian-elimination
 * encoder").  Reduces the dense M x N H to reduced row echelon form over
 * GF(2^m); pivot columns P, free columns F.  The codeword takes x_f = draws[f]
 * for f in F (random symbols drawn by the caller) and, from row i of the RREF
 * x_{p_i} + sum_{f in F} R[i][f] x_f = 0, x_{p_i} = sum_f R[i][f] x_f.
 * Returns rank(H). */
int or_code_encode(const or_code* c, const int* draws, int* x) {
  int M = c->M, N = c->N;
  const or_field* f = c->f;
  int* H = (int*)calloc((size_t)M * N, sizeof(int));
  for (int e = 0; e < c->E; ++e) H[(size_t)c->e_row[e] * N + c->e_col[e]] = c->e_h[e];
  int* pivcol = (int*)malloc(sizeof(int) * M);
  int* is_piv = (int*)calloc((size_t)N, sizeof(int));
  int rank = 0;
  for (int col = 0; col < N && rank < M; ++col) {
    int pr = -1;
    for (int r = rank; r < M; ++r) if (H[(size_t)r * N + col]) { pr = r; break; }
    if (pr < 0) continue;
    if (pr != rank)
      for (int j = 0; j < N; ++j) { int t = H[(size_t)pr * N + j]; H[(size_t)pr * N + j] = H[(size_t)rank * N + j]; H[(size_t)rank * N + j] = t; }
    int inv = or_gf_inv(f, H[(size_t)rank * N + col]);
    for (int j = 0; j < N; ++j) H[(size_t)rank * N + j] = or_gf_mul(f, inv, H[(size_t)rank * N + j]);
    for (int r = 0; r < M; ++r) {
      if (r == rank) continue;
      int g = H[(size_t)r * N + col];
      if (!g) continue;
      for (int j = 0; j < N; ++j) H[(size_t)r * N + j] = or_gf_add(H[(size_t)r * N + j], or_gf_mul(f, g, H[(size_t)rank * N + j]));
    }
    pivcol[rank] = col;
    is_piv[col] = 1;
    rank++;
  }
  for (int v = 0; v < N; ++v) x[v] = is_piv[v] ? 0 : draws[v];
  for (int i = 0; i < rank; ++i) {
    int acc = 0;
    for (int v = 0; v < N; ++v)
      if (!is_piv[v]) acc = or_gf_add(acc, or_gf_mul(f, H[(size_t)i * N + v], x[v]));
    x[pivcol[i]] = acc;
  }
  free(H); free(pivcol); free(is_piv);
  return rank;
}

/* ------------------------------------------------------------------ */
/* Channel prior p_v^(0)(x) = Pr(X_v = x | Y_v = y_v). */
/* For the binary image over BPSK/AWGN the bits are independent given  */
/* y, so p(x) = prod_i Pr(b_i = x_i | L_i) with Pr(b=0|L) = 1/(1+e^-L).*/
/* ------------------------------------------------------------------ */
void or_channel_prior(int m, const double* llr, double* p) {
  int q = 1 << m;
  for (int x = 0; x < q; ++x) {
    double v = 1.0;
    for (int i = 0; i < m; ++i) {
      double L = llr[i];
      v *= ((x >> i) & 1) ? 1.0 / (1.0 + exp(L)) : 1.0 / (1.0 + exp(-L));
    }
    p[x] = v;
  }
}

/* ------------------------------------------------------------------ */
/* O-SP: conventional SP in the probability domain  */
/* Messages: u[e][x] = p_vc (variable->check), w[e][x] = p_cv.         */
/* ------------------------------------------------------------------ */
void or_sp_init(const or_code* c, const double* llr, double* p0) {
  int m = c->f->m, q = c->f->q;
  for (int v = 0; v < c->N; ++v) or_channel_prior(m, llr + (size_t)v * m, p0 + (size_t)v * q);
}
/* CHECK TO VARIABLE:
 *   p~_vc(x) = p_vc(h_cv^{-1} x);  p~_cv = (x)_{v' in V_c \ v} p~_v'c;  p_cv(x) = p~_cv(h_cv x) */
void or_sp_check_to_variable(const or_code* c, const double* u, double* w) {
  const or_field* f = c->f;
  int m = f->m, q = f->q;
  double* tl = (double*)malloc(sizeof(double) * q);
  double* acc = (double*)malloc(sizeof(double) * q);
  double* tmp = (double*)malloc(sizeof(double) * q);
  for (int r = 0; r < c->M; ++r) {
    for (int ej = c->c_ptr[r]; ej < c->c_ptr[r + 1]; ++ej) {
      for (int x = 0; x < q; ++x) acc[x] = x == 0 ? 1.0 : 0.0; /* identity of (x) */
      for (int ek = c->c_ptr[r]; ek < c->c_ptr[r + 1]; ++ek) {
        if (ek == ej) continue;
        int hinv = or_gf_inv(f, c->e_h[ek]);
        for (int x = 0; x < q; ++x) tl[x] = u[(size_t)ek * q + or_gf_mul(f, hinv, x)];
        or_convolve(m, acc, tl, tmp);
        memcpy(acc, tmp, sizeof(double) * q);
      }
      for (int x = 0; x < q; ++x) w[(size_t)ej * q + x] = acc[or_gf_mul(f, c->e_h[ej], x)];
    }
  }
  free(tl); free(acc); free(tmp);
}
/* VARIABLE TO CHECK: p_vc(x) = p0(x) prod_{c' in C_v \ c} p_c'v(x),
 * normalised to sum 1 (norm_mode 0) or to value-at-0 = 1 (norm_mode 1, :190-193). */
void or_sp_variable_to_check(const or_code* c, const double* p0, const double* w, double* u, int norm_mode) {
  int q = c->f->q;
  for (int v = 0; v < c->N; ++v)
    for (int i = c->v_ptr[v]; i < c->v_ptr[v + 1]; ++i) {
      int e = c->v_edges[i];
      double s = 0.0;
      for (int x = 0; x < q; ++x) {
        double val = p0[(size_t)v * q + x];
        for (int j = c->v_ptr[v]; j < c->v_ptr[v + 1]; ++j)
          if (c->v_edges[j] != e) val *= w[(size_t)c->v_edges[j] * q + x];
        u[(size_t)e * q + x] = val;
        s += val;
      }
      double nrm = norm_mode == 0 ? s : u[(size_t)e * q + 0];
      for (int x = 0; x < q; ++x) u[(size_t)e * q + x] /= nrm;
    }
}
/* TENTATIVE DECISION posterior: q_v(x) = p0(x) prod_{c' in C_v} p_c'v(x),
 * normalised to sum 1 for reporting. */
void or_sp_posterior(const or_code* c, const double* p0, const double* w, double* qv) {
  int q = c->f->q;
  for (int v = 0; v < c->N; ++v) {
    double s = 0.0;
    for (int x = 0; x < q; ++x) {
      double val = p0[(size_t)v * q + x];
      for (int j = c->v_ptr[v]; j < c->v_ptr[v + 1]; ++j) val *= w[(size_t)c->v_edges[j] * q + x];
      qv[(size_t)v * q + x] = val;
      s += val;
    }
    for (int x = 0; x < q; ++x) qv[(size_t)v * q + x] /= s;
  }
}

/* ------------------------------------------------------------------ */
/* IEEE 754 binary16 rounding, written out from the format's           */
/* definition: 1 sign bit, 5 exponent bits (bias 15), 10 fraction bits; */
/* normal numbers 2^-14 .. 65504, subnormals with the quantum 2^-24;   */
/* round to nearest, ties to even; overflow to infinity.  It is the    */
/* storage rule of the half-precision message format (O-LF-half,       */
/* SURVEY 8(f) row 4, the quantisation motivation of PAPER.md:57-71;   */
/* reading R26): not part of the paper's arithmetic.                   */
/* ------------------------------------------------------------------ */
/* mode 1: round to nearest, ties to even (the format's default rounding, the storage rule); mode 2:
 * round toward zero -- used only as a second, equally valid rounding of the same format, to tell
 * frames whose outcome depends on how stored values round (tests/test_gpu_f16.py) */
double or_round_half_mode(double v, int mode) {
  if (v != v || v == 0.0 || isinf(v)) return v;
  double a = fabs(v);
  int e;
  frexp(a, &e);          /* a = f 2^e, f in [0.5, 1): the leading bit weighs 2^(e-1) */
  int lead = e - 1;
  if (lead < -14) lead = -14;             /* subnormals: all share the quantum 2^-24 */
  double quantum = ldexp(1.0, lead - 10); /* 10 fraction bits below the leading bit */
  double r = (mode == 2 ? floor(a / quantum) : nearbyint(a / quantum)) * quantum; /* nearbyint: ties to even */
  if (r > 65504.0) r = mode == 2 ? 65504.0 : INFINITY;
  return v < 0 ? -r : r;
}
double or_round_half(double v) { return or_round_half_mode(v, 1); }

/* ------------------------------------------------------------------ */
/* O-LF: the paper's Log-Fourier SP, double and a   */
/* float32 diagnostic twin generated from lf_body.inc.                 */
/* ------------------------------------------------------------------ */
#define LF_REAL double
#define LF_SFX(name) name
#define LF_EXP exp
#define LF_LOG log
#define LF_FABS fabs
#include "lf_body.inc"
#undef LF_REAL
#undef LF_SFX
#undef LF_EXP
#undef LF_LOG
#undef LF_FABS

#define LF_REAL float
#define LF_SFX(name) name##_f32
#define LF_EXP expf
#define LF_LOG logf
#define LF_FABS fabsf
#include "lf_body.inc"

/* ------------------------------------------------------------------ */
/* O-LS: the conventional Log-SP, the paper's       */
/* comparison algorithm; double and a float32 diagnostic twin.         */
/* ------------------------------------------------------------------ */
#define LS_REAL double
#define LS_SFX(name) name
#define LS_EXP exp
#define LS_LOG log
#include "logsp_body.inc"
#undef LS_REAL
#undef LS_SFX
#undef LS_EXP
#undef LS_LOG

#define LS_REAL float
#define LS_SFX(name) name##_f32
#define LS_EXP expf
#define LS_LOG logf
#include "logsp_body.inc"
