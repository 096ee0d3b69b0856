/*
 * tileqr_oracle.c -- plain, slow, obviously-correct CPU oracle of the tile
 * Householder QR factorization (flat "TS" tree) studied in arxiv 1102.5328
 * (INRIA RR-7526).
 *
 *   *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke()
 *   and bench.py's cpu_baseline / --impl reference legs may load this file's
 *   library.  The product path (paper_1102_5328_b200/) never links, imports
 *   or executes it, and shares no source, header, table or helper with it.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n,
 * S:n = /root/reference/SPEC.md line n, SURVEY §8(c) = the adopted readings):
 *   - The matrix of order N is split into NT x NT tiles of order NB
 *     ("split the initial matrix of order N into NT x NT smaller
 *     square pieces of order NB, called tiles"); non-dividing sizes are padded
 *     (reading R5).
 *   - Four serial kernels: GEQRT and TSQRT factor the panel,
 *     LARFB and SSRFB apply its reflectors to the trailing tiles.  Kernel
 *     internals follow the standard compact-WY formulation with inner
 *     blocking IB, which the paper delegates to
 *     [tileplasma].
 *   - Every step is written as plain nested loops in fp64, in the order the
 *     algorithm states it; no blocking, fusion or reordering beyond the
 *     algorithm itself.  No BLAS.
 *
 * Parity pins (tests/test_oracle_*.py): LAPACK dgeqrt/dtpqrt/dgemqrt/dtpmqrt
 * via scipy, numpy.linalg.qr, a textbook unblocked Householder QR written in
 * the test, 50-digit Gram-Schmidt, closed forms ([3 1;4 2], [I;I]),
 * compact-WY identities, R^T R = A^T A, thread-count bitwise invariance.
 *
 * Layouts: every matrix is column-major; a tile is an
 * NB x NB block addressed inside a larger column-major array with leading
 * dimension ld; T of one tile is IB x NB (ld = ldt): panel p's IB x IB
 * upper-triangular factor occupies columns [p*IB, (p+1)*IB).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EL(a, ld, i, j) ((a)[(size_t)(i) + (size_t)(j) * (size_t)(ld)])

/* ------------------------------------------------------------------------ *
 * Reflector rule (reading R1; LAPACK larfg convention, S:142 says
 * the paper is silent).  x = [alpha; x2] of length 1 + n2 (x2 stride incx).
 *   sigma = sum x2_i^2
 *   sigma == 0  ->  tau = 0, beta = alpha, v2 = 0          (no reflection)
 *   else        ->  beta = -sgn(alpha) sqrt(alpha^2 + sigma), sgn(+-0) = +1
 *                   tau  = (beta - alpha) / beta
 *                   v2   = x2 / (alpha - beta)
 * H = I - tau v v^T with v = [1; v2] satisfies H x = beta e1.
 * On return *alpha = beta and x2 is overwritten by v2.
 * ------------------------------------------------------------------------ */
double oracle_larfg(int n2, double *alpha, double *x2, int incx) {
  double sigma = 0.0;
  for (int i = 0; i < n2; ++i) sigma += x2[(size_t)i * incx] * x2[(size_t)i * incx];
  if (sigma == 0.0) return 0.0;
  double a = *alpha;
  double norm = sqrt(a * a + sigma);
  double beta = (a >= 0.0) ? -norm : norm; /* -0.0 >= 0.0 is true: sgn(-0) = +1 */
  double tau = (beta - a) / beta;
  double scal = 1.0 / (a - beta);
  for (int i = 0; i < n2; ++i) x2[(size_t)i * incx] *= scal;
  *alpha = beta;
  return tau;
}

/* ------------------------------------------------------------------------ *
 * T of one panel (compact WY, forward, columnwise):
 *   T[i,i] = tau_i,  T[0:i, i] = -tau_i * T[0:i,0:i] * z,  z_l = v_l^T v_i.
 * dots[l + i*ib] must hold v_l^T v_i for l < i.  T is written at t (ld ldt).
 * ------------------------------------------------------------------------ */
static void build_t(int ib, const double *tau, const double *dots, double *t, int ldt) {
  for (int i = 0; i < ib; ++i) {
    for (int l = 0; l < ib; ++l) EL(t, ldt, l, i) = 0.0;
    EL(t, ldt, i, i) = tau[i];
    for (int r = 0; r < i; ++r) {
      /* (T[0:i,0:i] z)_r = sum_{l=r}^{i-1} T[r,l] z_l   (T upper triangular) */
      double s = 0.0;
      for (int l = r; l < i; ++l) s += EL(t, ldt, r, l) * dots[l + (size_t)i * ib];
      EL(t, ldt, r, i) = -tau[i] * s;
    }
  }
}

/* ------------------------------------------------------------------------ *
 * GEQRT: QR of one NB x NB tile with inner blocking IB (
 * SURVEY §8(c) step 2a).  On return: R in the upper triangle, V strictly
 * below (unit diagonal implicit), T (IB x NB, ld ldt) with the strictly-lower
 * part of every IB x IB block zero.
 * ------------------------------------------------------------------------ */
void oracle_geqrt(int nb, int ib, double *a, int lda, double *t, int ldt) {
  double *tau = (double *)malloc(sizeof(double) * ib);
  double *dots = (double *)malloc(sizeof(double) * ib * ib);
  double *w = (double *)malloc(sizeof(double) * ib * nb);
  for (int c0 = 0; c0 < nb; c0 += ib) {
    /* 1. factor the panel column by column */
    for (int j = c0; j < c0 + ib; ++j) {
      tau[j - c0] = oracle_larfg(nb - j - 1, &EL(a, lda, j, j), &EL(a, lda, j + 1, j), 1);
      for (int c = j + 1; c < c0 + ib; ++c) {
        double s = EL(a, lda, j, c);
        for (int i = j + 1; i < nb; ++i) s += EL(a, lda, i, j) * EL(a, lda, i, c);
        EL(a, lda, j, c) -= tau[j - c0] * s;
        for (int i = j + 1; i < nb; ++i) EL(a, lda, i, c) -= tau[j - c0] * EL(a, lda, i, j) * s;
      }
    }
    /* 2. T_p: z_l = v_l^T v_i over rows >= c0+i (v_i is 0 above, 1 at c0+i) */
    for (int i = 0; i < ib; ++i)
      for (int l = 0; l < i; ++l) {
        int ri = c0 + i;
        double s = EL(a, lda, ri, c0 + l); /* v_l[ri] * 1 */
        for (int r = ri + 1; r < nb; ++r) s += EL(a, lda, r, c0 + l) * EL(a, lda, r, ri);
        dots[l + (size_t)i * ib] = s;
      }
    build_t(ib, tau, dots, &EL(t, ldt, 0, c0), ldt);
    /* 3. apply Q_p^T to the trailing columns c >= c0+ib, rows >= c0:
     *    W = V_p^T C;  W = T_p^T W;  C -= V_p W                           */
    int nc = nb - (c0 + ib);
    for (int c = 0; c < nc; ++c)
      for (int i = 0; i < ib; ++i) {
        int vi = c0 + i; /* v_i: 1 at row vi, A[r, vi] below */
        double s = EL(a, lda, vi, c0 + ib + c);
        for (int r = vi + 1; r < nb; ++r) s += EL(a, lda, r, vi) * EL(a, lda, r, c0 + ib + c);
        w[i + (size_t)c * ib] = s;
      }
    for (int c = 0; c < nc; ++c)
      for (int i = ib - 1; i >= 0; --i) { /* W[i] = sum_{l<=i} T[l,i] W[l] */
        double s = 0.0;
        for (int l = 0; l <= i; ++l) s += EL(t, ldt, l, c0 + i) * w[l + (size_t)c * ib];
        w[i + (size_t)c * ib] = s;
      }
    for (int c = 0; c < nc; ++c)
      for (int r = c0; r < nb; ++r) {
        double s = 0.0;
        for (int i = 0; i < ib; ++i) {
          int vi = c0 + i;
          double v = (r == vi) ? 1.0 : (r > vi ? EL(a, lda, r, vi) : 0.0);
          s += v * w[i + (size_t)c * ib];
        }
        EL(a, lda, r, c0 + ib + c) -= s;
      }
  }
  free(tau);
  free(dots);
  free(w);
}

/* ------------------------------------------------------------------------ *
 * TSQRT: QR of [R; B] (R upper triangular NB x NB, B full NB x NB) with inner
 * blocking IB.  Reflector j is
 * v_j = [e_j; V2[:, j]]; V2 overwrites B; R's upper triangle is updated; the
 * strict lower part of R is never read or written.
 * ------------------------------------------------------------------------ */
void oracle_tsqrt(int nb, int ib, double *r, int ldr, double *b, int ldb, double *t, int ldt) {
  double *tau = (double *)malloc(sizeof(double) * ib);
  double *dots = (double *)malloc(sizeof(double) * ib * ib);
  double *w = (double *)malloc(sizeof(double) * ib * nb);
  for (int c0 = 0; c0 < nb; c0 += ib) {
    for (int j = c0; j < c0 + ib; ++j) {
      tau[j - c0] = oracle_larfg(nb, &EL(r, ldr, j, j), &EL(b, ldb, 0, j), 1);
      for (int c = j + 1; c < c0 + ib; ++c) {
        double s = EL(r, ldr, j, c);
        for (int i = 0; i < nb; ++i) s += EL(b, ldb, i, j) * EL(b, ldb, i, c);
        EL(r, ldr, j, c) -= tau[j - c0] * s;
        for (int i = 0; i < nb; ++i) EL(b, ldb, i, c) -= tau[j - c0] * EL(b, ldb, i, j) * s;
      }
    }
    /* the top parts e_j are distinct unit vectors: v_l^T v_i = V2_l^T V2_i */
    for (int i = 0; i < ib; ++i)
      for (int l = 0; l < i; ++l) {
        double s = 0.0;
        for (int q = 0; q < nb; ++q) s += EL(b, ldb, q, c0 + l) * EL(b, ldb, q, c0 + i);
        dots[l + (size_t)i * ib] = s;
      }
    build_t(ib, tau, dots, &EL(t, ldt, 0, c0), ldt);
    /* trailing columns c >= c0+ib:  W = R[c0:c0+ib, c] + V2_p^T B[:, c];
     * W = T_p^T W;  R[c0:c0+ib, c] -= W;  B[:, c] -= V2_p W              */
    int nc = nb - (c0 + ib);
    for (int c = 0; c < nc; ++c)
      for (int i = 0; i < ib; ++i) {
        double s = EL(r, ldr, c0 + i, c0 + ib + c);
        for (int q = 0; q < nb; ++q) s += EL(b, ldb, q, c0 + i) * EL(b, ldb, q, c0 + ib + c);
        w[i + (size_t)c * ib] = s;
      }
    for (int c = 0; c < nc; ++c)
      for (int i = ib - 1; i >= 0; --i) {
        double s = 0.0;
        for (int l = 0; l <= i; ++l) s += EL(t, ldt, l, c0 + i) * w[l + (size_t)c * ib];
        w[i + (size_t)c * ib] = s;
      }
    for (int c = 0; c < nc; ++c) {
      for (int i = 0; i < ib; ++i) EL(r, ldr, c0 + i, c0 + ib + c) -= w[i + (size_t)c * ib];
      for (int q = 0; q < nb; ++q) {
        double s = 0.0;
        for (int i = 0; i < ib; ++i) s += EL(b, ldb, q, c0 + i) * w[i + (size_t)c * ib];
        EL(b, ldb, q, c0 + ib + c) -= s;
      }
    }
  }
  free(tau);
  free(dots);
  free(w);
}

/* W := op(T_p) W for one panel, W ib x nc (ld ib).  trans='T': W = T^T W
 * (T upper => T^T lower, rows computed bottom-up in place); 'N': W = T W. */
static void apply_tp(char trans, int ib, const double *tp, int ldt, double *w, int nc) {
  for (int c = 0; c < nc; ++c) {
    double *wc = w + (size_t)c * ib;
    if (trans == 'T') {
      for (int i = ib - 1; i >= 0; --i) {
        double s = 0.0;
        for (int l = 0; l <= i; ++l) s += EL(tp, ldt, l, i) * wc[l];
        wc[i] = s;
      }
    } else {
      for (int i = 0; i < ib; ++i) {
        double s = 0.0;
        for (int l = i; l < ib; ++l) s += EL(tp, ldt, i, l) * wc[l];
        wc[i] = s;
      }
    }
  }
}

/* ------------------------------------------------------------------------ *
 * LARFB: C <- Q^T C (trans='T') or Q C ('N') for the tile reflectors of a
 * GEQRT.  V is the GEQRT output tile (unit lower, strict
 * lower part read), C is NB x ncols.  Q = Q_0 Q_1 ... Q_{P-1}, Q_p = I -
 * V_p T_p V_p^T, so Q^T applies panels p = 0..P-1 with T_p^T and Q applies
 * p = P-1..0 with T_p.
 * ------------------------------------------------------------------------ */
void oracle_larfb(char trans, int nb, int ib, const double *v, int ldv, const double *t, int ldt,
                  double *c, int ldc, int ncols) {
  double *w = (double *)malloc(sizeof(double) * ib * (ncols > 0 ? ncols : 1));
  int np = nb / ib;
  for (int pp = 0; pp < np; ++pp) {
    int p = (trans == 'T') ? pp : np - 1 - pp;
    int c0 = p * ib;
    for (int cc = 0; cc < ncols; ++cc)
      for (int i = 0; i < ib; ++i) {
        int vi = c0 + i;
        double s = EL(c, ldc, vi, cc);
        for (int r = vi + 1; r < nb; ++r) s += EL(v, ldv, r, vi) * EL(c, ldc, r, cc);
        w[i + (size_t)cc * ib] = s;
      }
    apply_tp(trans, ib, &EL(t, ldt, 0, c0), ldt, w, ncols);
    for (int cc = 0; cc < ncols; ++cc)
      for (int r = c0; r < nb; ++r) {
        double s = 0.0;
        for (int i = 0; i < ib; ++i) {
          int vi = c0 + i;
          double vv = (r == vi) ? 1.0 : (r > vi ? EL(v, ldv, r, vi) : 0.0);
          s += vv * w[i + (size_t)cc * ib];
        }
        EL(c, ldc, r, cc) -= s;
      }
  }
  free(w);
}

/* ------------------------------------------------------------------------ *
 * SSRFB: [C1; C2] <- Q^T [C1; C2] (trans='T') or Q [C1; C2] ('N') for the
 * reflectors of a TSQRT, v_j = [e_j; V2[:, j]] (
 * S:88-96).  For each panel p (ascending for 'T'):
 *   W = C1[p rows, :] + V2_p^T C2;  W = op(T_p) W;
 *   C1[p rows, :] -= W;  C2 -= V2_p W.
 * ------------------------------------------------------------------------ */
void oracle_ssrfb(char trans, int nb, int ib, const double *v2, int ldv, const double *t, int ldt,
                  double *c1, int ldc1, double *c2, int ldc2, int ncols) {
  double *w = (double *)malloc(sizeof(double) * ib * (ncols > 0 ? ncols : 1));
  int np = nb / ib;
  for (int pp = 0; pp < np; ++pp) {
    int p = (trans == 'T') ? pp : np - 1 - pp;
    int c0 = p * ib;
    for (int cc = 0; cc < ncols; ++cc)
      for (int i = 0; i < ib; ++i) {
        double s = EL(c1, ldc1, c0 + i, cc);
        for (int q = 0; q < nb; ++q) s += EL(v2, ldv, q, c0 + i) * EL(c2, ldc2, q, cc);
        w[i + (size_t)cc * ib] = s;
      }
    apply_tp(trans, ib, &EL(t, ldt, 0, c0), ldt, w, ncols);
    for (int cc = 0; cc < ncols; ++cc) {
      for (int i = 0; i < ib; ++i) EL(c1, ldc1, c0 + i, cc) -= w[i + (size_t)cc * ib];
      for (int q = 0; q < nb; ++q) {
        double s = 0.0;
        for (int i = 0; i < ib; ++i) s += EL(v2, ldv, q, c0 + i) * w[i + (size_t)cc * ib];
        EL(c2, ldc2, q, cc) -= s;
      }
    }
  }
  free(w);
}

/* ------------------------------------------------------------------------ *
 * Whole tile QR.
 *
 *   M x N matrix A (ld lda) -> padded At of order (MT*NB) x (NT*NB):
 *     At = A on [0,M) x [0,N); rows >= M are 0; a padded column j >= N is
 *     e_j when M <= j < MT*NB, else 0 (reading R5).
 *   for k = 0 .. min(MT,NT)-1:
 *     GEQRT(k,k); LARFB(k,n) for n > k; TSQRT(k,m) for m = k+1..MT-1 in
 *     order (flat tree, reading R6); SSRFB(k,m,n) for m > k, n > k.
 *   Threads own tile columns n ("1-D cyclic assignment of tile
 *   columns"); for fixed n the m loop is sequential, so every tile sees the
 *   same sequence of operations for any thread count.
 *
 *   kmax limits the outer loop (k < kmax; kmax <= 0 means all): the first
 *   kmax block rows of R and the first kmax panels of V/T are then final.
 *   Used to check sampled outputs of very large factorizations.
 *
 * On return A[0:M,0:N] holds R (upper triangle) and the V tiles below; T is
 * MT*NT*IB*NB doubles, tile (m,k) at offset (m + k*MT)*IB*NB with ld IB.
 * Returns 0, or 1 if A holds a non-finite entry (A and T then untouched),
 * or -1 on allocation failure.
 * ------------------------------------------------------------------------ */
int oracle_tileqr_factor(int64_t M, int64_t N, double *A, int64_t lda, int NB, int IB, double *T,
                         int nthreads, int kmax) {
  if (M == 0 || N == 0) return 0;
  for (int64_t j = 0; j < N; ++j)
    for (int64_t i = 0; i < M; ++i)
      if (!isfinite(EL(A, lda, i, j))) return 1;
  int64_t MT = (M + NB - 1) / NB, NT = (N + NB - 1) / NB;
  int64_t ldp = MT * NB, np = NT * NB;
  double *P = (double *)calloc((size_t)ldp * (size_t)np, sizeof(double));
  if (!P) return -1;
  for (int64_t j = 0; j < N; ++j)
    for (int64_t i = 0; i < M; ++i) EL(P, ldp, i, j) = EL(A, lda, i, j);
  for (int64_t j = N; j < np; ++j)
    if (j >= M && j < ldp) EL(P, ldp, j, j) = 1.0;
  memset(T, 0, sizeof(double) * (size_t)(MT * NT) * IB * NB);
#define TILE(m, n) (&EL(P, ldp, (m) * NB, (n) * NB))
#define TT(m, k) (T + ((size_t)(m) + (size_t)(k) * MT) * IB * NB)
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int64_t KT = MT < NT ? MT : NT;
  if (kmax > 0 && kmax < KT) KT = kmax;
  for (int64_t k = 0; k < KT; ++k) {
    oracle_geqrt(NB, IB, TILE(k, k), (int)ldp, TT(k, k), IB);
#pragma omp parallel for schedule(static, 1)
    for (int64_t n = k + 1; n < NT; ++n)
      oracle_larfb('T', NB, IB, TILE(k, k), (int)ldp, TT(k, k), IB, TILE(k, n), (int)ldp, NB);
    for (int64_t m = k + 1; m < MT; ++m)
      oracle_tsqrt(NB, IB, TILE(k, k), (int)ldp, TILE(m, k), (int)ldp, TT(m, k), IB);
#pragma omp parallel for schedule(static, 1)
    for (int64_t n = k + 1; n < NT; ++n)
      for (int64_t m = k + 1; m < MT; ++m)
        oracle_ssrfb('T', NB, IB, TILE(m, k), (int)ldp, TT(m, k), IB, TILE(k, n), (int)ldp,
                     TILE(m, n), (int)ldp, NB);
  }
  for (int64_t j = 0; j < N; ++j)
    for (int64_t i = 0; i < M; ++i) EL(A, lda, i, j) = EL(P, ldp, i, j);
  free(P);
#undef TILE
#undef TT
  return 0;
}

/* ------------------------------------------------------------------------ *
 * Apply the Q of a tile QR to B (M x NRHS, ld ldb):
 *   trans='T': B <- Q^T B: k ascending, LARFB(k) then SSRFB(k,m) m ascending;
 *   trans='N': B <- Q B:   k descending, SSRFB(k,m) m descending, then LARFB.
 * A (M x K, ld lda) and T are a tileqr factor output with the same NB, IB.
 * Returns 0 (or -1 on allocation failure).
 * ------------------------------------------------------------------------ */
int oracle_tileqr_apply(char trans, int64_t M, int64_t NRHS, int64_t K, const double *A, int64_t lda,
                        const double *T, int NB, int IB, double *B, int64_t ldb, int nthreads) {
  if (M == 0 || NRHS == 0 || K == 0) return 0;
  int64_t MT = (M + NB - 1) / NB, KTt = (K + NB - 1) / NB;
  int64_t KT = MT < KTt ? MT : KTt;
  int64_t ldp = MT * NB;
  /* padded copies: V tiles of A (column tiles 0..KT-1), B with zero rows */
  double *V = (double *)calloc((size_t)ldp * (size_t)(KT * NB), sizeof(double));
  double *Bp = (double *)calloc((size_t)ldp * (size_t)NRHS, sizeof(double));
  if (!V || !Bp) { free(V); free(Bp); return -1; }
  for (int64_t j = 0; j < K && j < KT * NB; ++j)
    for (int64_t i = 0; i < M; ++i) EL(V, ldp, i, j) = EL(A, lda, i, j);
  for (int64_t j = 0; j < NRHS; ++j)
    for (int64_t i = 0; i < M; ++i) EL(Bp, ldp, i, j) = EL(B, ldb, i, j);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  for (int64_t kk = 0; kk < KT; ++kk) {
    int64_t k = (trans == 'T') ? kk : KT - 1 - kk;
    const double *Vkk = &EL(V, ldp, k * NB, k * NB);
    const double *Tkk = T + ((size_t)k + (size_t)k * MT) * IB * NB;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < NRHS; ++c) {
      double *Bk = &EL(Bp, ldp, k * NB, c);
      if (trans == 'T') oracle_larfb('T', NB, IB, Vkk, (int)ldp, Tkk, IB, Bk, (int)ldp, 1);
      for (int64_t mm = k + 1; mm < MT; ++mm) {
        int64_t m = (trans == 'T') ? mm : MT - 1 - (mm - (k + 1));
        const double *Vmk = &EL(V, ldp, m * NB, k * NB);
        const double *Tmk = T + ((size_t)m + (size_t)k * MT) * IB * NB;
        oracle_ssrfb(trans, NB, IB, Vmk, (int)ldp, Tmk, IB, Bk, (int)ldp, &EL(Bp, ldp, m * NB, c),
                     (int)ldp, 1);
      }
      if (trans == 'N') oracle_larfb('N', NB, IB, Vkk, (int)ldp, Tkk, IB, Bk, (int)ldp, 1);
    }
  }
  for (int64_t j = 0; j < NRHS; ++j)
    for (int64_t i = 0; i < M; ++i) EL(B, ldb, i, j) = EL(Bp, ldp, i, j);
  free(V);
  free(Bp);
  return 0;
}

/* ======================================================================== *
 * Tall-skinny / communication-avoiding variant (PAPER.md
 * P:840-850 names "tall and skinny" matrices and communication-avoiding QR
 * with p domains as the next tunable): the TSQRT chain of a panel is
 * replaced by a reduction TREE -- domain heads factored by GEQRT, merged
 * pairwise by TTQRT ("triangle on triangle"), whose reflectors are applied
 * by TTMQRT.  Readings (R20): domains of BS consecutive tile rows
 * [d*BS, (d+1)*BS) in absolute tile-row numbers (the head of a domain at
 * panel k is its first row >= k); flat TS chain inside a domain; binary
 * tree over the heads (distance 1, 2, 4, ...: head i absorbs head i + s for
 * i a multiple of 2s).  BS >= MT is the flat tree of oracle_tileqr_factor.
 * ======================================================================== */

/* ------------------------------------------------------------------------ *
 * TTQRT: QR of [R1; R2], R1 and R2 both NB x NB upper triangular, with inner
 * blocking IB (LAPACK dtpqrt with L = NB computes the same kernel).
 * Reflector j is v_j = [e_j; V2[0:j, j]] (rows 0..j of column j of R2):
 * x = [R1(j,j); R2(0:j, j)].  V2 overwrites the upper triangle (diagonal
 * included) of R2; the strict lower parts of R1 and R2 are neither read nor
 * written.  T (IB x NB, ld ldt) as for TSQRT.
 * ------------------------------------------------------------------------ */
void oracle_ttqrt(int nb, int ib, double *r, int ldr, double *b, int ldb, double *t, int ldt) {
  double *tau = (double *)malloc(sizeof(double) * ib);
  double *dots = (double *)malloc(sizeof(double) * ib * ib);
  double *w = (double *)malloc(sizeof(double) * ib * nb);
  for (int c0 = 0; c0 < nb; c0 += ib) {
    for (int j = c0; j < c0 + ib; ++j) {
      tau[j - c0] = oracle_larfg(j + 1, &EL(r, ldr, j, j), &EL(b, ldb, 0, j), 1);
      for (int c = j + 1; c < c0 + ib; ++c) {
        double s = EL(r, ldr, j, c);
        for (int i = 0; i <= j; ++i) s += EL(b, ldb, i, j) * EL(b, ldb, i, c);
        EL(r, ldr, j, c) -= tau[j - c0] * s;
        for (int i = 0; i <= j; ++i) EL(b, ldb, i, c) -= tau[j - c0] * EL(b, ldb, i, j) * s;
      }
    }
    /* v_l^T v_i = V2_l^T V2_i over rows 0..c0+l (V2_l is zero below row c0+l) */
    for (int i = 0; i < ib; ++i)
      for (int l = 0; l < i; ++l) {
        double s = 0.0;
        for (int q = 0; q <= c0 + l; ++q) s += EL(b, ldb, q, c0 + l) * EL(b, ldb, q, c0 + i);
        dots[l + (size_t)i * ib] = s;
      }
    build_t(ib, tau, dots, &EL(t, ldt, 0, c0), ldt);
    /* trailing columns c >= c0+ib:  W = R1[c0:c0+ib, c] + V2_p^T R2[:, c];
     * W = T_p^T W;  R1[c0:c0+ib, c] -= W;  R2[0:c0+ib, c] -= V2_p W       */
    int nc = nb - (c0 + ib);
    for (int c = 0; c < nc; ++c)
      for (int i = 0; i < ib; ++i) {
        double s = EL(r, ldr, c0 + i, c0 + ib + c);
        for (int q = 0; q <= c0 + i; ++q) s += EL(b, ldb, q, c0 + i) * EL(b, ldb, q, c0 + ib + c);
        w[i + (size_t)c * ib] = s;
      }
    for (int c = 0; c < nc; ++c)
      for (int i = ib - 1; i >= 0; --i) {
        double s = 0.0;
        for (int l = 0; l <= i; ++l) s += EL(t, ldt, l, c0 + i) * w[l + (size_t)c * ib];
        w[i + (size_t)c * ib] = s;
      }
    for (int c = 0; c < nc; ++c) {
      for (int i = 0; i < ib; ++i) EL(r, ldr, c0 + i, c0 + ib + c) -= w[i + (size_t)c * ib];
      for (int q = 0; q < c0 + ib; ++q) {
        double s = 0.0;
        for (int i = 0; i < ib; ++i)
          if (q <= c0 + i) s += EL(b, ldb, q, c0 + i) * w[i + (size_t)c * ib];
        EL(b, ldb, q, c0 + ib + c) -= s;
      }
    }
  }
  free(tau);
  free(dots);
  free(w);
}

/* ------------------------------------------------------------------------ *
 * TTMQRT: [C1; C2] <- Q^T [C1; C2] ('T') or Q [C1; C2] ('N') for the
 * reflectors of a TTQRT (V2 = the upper triangle, diagonal included, of its
 * second tile; the strict lower part of that tile is not read).  LAPACK
 * dtpmqrt with L = NB computes the same kernel.  As SSRFB with the V2 sums
 * restricted to rows q <= c0+i.
 * ------------------------------------------------------------------------ */
void oracle_ttmqrt(char trans, int nb, int ib, const double *v2, int ldv, const double *t, int ldt,
                   double *c1, int ldc1, double *c2, int ldc2, int ncols) {
  double *w = (double *)malloc(sizeof(double) * ib * (ncols > 0 ? ncols : 1));
  int np = nb / ib;
  for (int pp = 0; pp < np; ++pp) {
    int p = (trans == 'T') ? pp : np - 1 - pp;
    int c0 = p * ib;
    for (int cc = 0; cc < ncols; ++cc)
      for (int i = 0; i < ib; ++i) {
        double s = EL(c1, ldc1, c0 + i, cc);
        for (int q = 0; q <= c0 + i; ++q) s += EL(v2, ldv, q, c0 + i) * EL(c2, ldc2, q, cc);
        w[i + (size_t)cc * ib] = s;
      }
    apply_tp(trans, ib, &EL(t, ldt, 0, c0), ldt, w, ncols);
    for (int cc = 0; cc < ncols; ++cc) {
      for (int i = 0; i < ib; ++i) EL(c1, ldc1, c0 + i, cc) -= w[i + (size_t)cc * ib];
      for (int q = 0; q < c0 + ib; ++q) {
        double s = 0.0;
        for (int i = 0; i < ib; ++i)
          if (q <= c0 + i) s += EL(v2, ldv, q, c0 + i) * w[i + (size_t)cc * ib];
        EL(c2, ldc2, q, cc) -= s;
      }
    }
  }
  free(w);
}

/* Heads of panel k's domains (R20): h_d = max(d*BS, k) for every
 * domain d with rows >= k; returns their count. */
static int64_t tree_heads(int64_t MT, int64_t k, int64_t BS, int64_t *heads) {
  int64_t nh = 0;
  for (int64_t d = k / BS; d * BS < MT; ++d) heads[nh++] = d * BS > k ? d * BS : k;
  return nh;
}

/* ------------------------------------------------------------------------ *
 * Whole tile QR with the reduction tree (f3).  As oracle_tileqr_factor
 * (padding, layouts) with, for each panel k:
 *   for every domain (heads h ascending):
 *     GEQRT(h,k); LARFB(h,k;n) for n > k;
 *     for m in the domain, m > h, ascending: TSQRT(h,m;k); SSRFB(h,m,k;n);
 *   for s = 1, 2, 4, ...: for i = 0, 2s, 4s, ... with i + s < #heads:
 *     a = head[i], b = head[i+s]: TTQRT(a,b;k) (R_b merged into R_a, V2 in the
 *     upper triangle of tile (b,k), T2(b,k)); TTMQRT(a,b,k;n) for n > k.
 *   (The panel operations only touch column k and the V / T they leave are
 *   never rewritten, so all of them run before the updates, which run in the
 *   same order per tile column; threads own tile columns.)
 * T holds 2 * MT*NT*IB*NB doubles: T (GEQRT / TSQRT, tile (m,k) at
 * (m + k*MT)*IB*NB) followed by T2 (TTQRT, same offsets).  BS >= MT gives
 * oracle_tileqr_factor's result with T2 = 0.
 * Returns 0, 1 for a non-finite input, -1 on allocation failure.
 * ------------------------------------------------------------------------ */
int oracle_tileqr_factor_tree(int64_t M, int64_t N, double *A, int64_t lda, int NB, int IB, int64_t BS,
                              double *T, int nthreads) {
  if (M == 0 || N == 0) return 0;
  if (BS < 1) BS = 1;
  for (int64_t j = 0; j < N; ++j)
    for (int64_t i = 0; i < M; ++i)
      if (!isfinite(EL(A, lda, i, j))) return 1;
  int64_t MT = (M + NB - 1) / NB, NT = (N + NB - 1) / NB;
  int64_t ldp = MT * NB, np = NT * NB;
  double *P = (double *)calloc((size_t)ldp * (size_t)np, sizeof(double));
  int64_t *heads = (int64_t *)malloc(sizeof(int64_t) * (size_t)(MT + 1));
  if (!P || !heads) { free(P); free(heads); return -1; }
  for (int64_t j = 0; j < N; ++j)
    for (int64_t i = 0; i < M; ++i) EL(P, ldp, i, j) = EL(A, lda, i, j);
  for (int64_t j = N; j < np; ++j)
    if (j >= M && j < ldp) EL(P, ldp, j, j) = 1.0;
  const size_t tsz = (size_t)(MT * NT) * IB * NB;
  memset(T, 0, sizeof(double) * 2 * tsz);
#define TILE(m, n) (&EL(P, ldp, (m) * NB, (n) * NB))
#define TT(m, k) (T + ((size_t)(m) + (size_t)(k) * MT) * IB * NB)
#define TT2(m, k) (T + tsz + ((size_t)(m) + (size_t)(k) * MT) * IB * NB)
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int64_t KT = MT < NT ? MT : NT;
  for (int64_t k = 0; k < KT; ++k) {
    int64_t nh = tree_heads(MT, k, BS, heads);
    /* panel operations (column k) */
    for (int64_t d = 0; d < nh; ++d) {
      int64_t h = heads[d], end = (h / BS + 1) * BS < MT ? (h / BS + 1) * BS : MT;
      oracle_geqrt(NB, IB, TILE(h, k), (int)ldp, TT(h, k), IB);
      for (int64_t m = h + 1; m < end; ++m)
        oracle_tsqrt(NB, IB, TILE(h, k), (int)ldp, TILE(m, k), (int)ldp, TT(m, k), IB);
    }
    for (int64_t s = 1; s < nh; s *= 2)
      for (int64_t i = 0; i + s < nh; i += 2 * s)
        oracle_ttqrt(NB, IB, TILE(heads[i], k), (int)ldp, TILE(heads[i + s], k), (int)ldp,
                     TT2(heads[i + s], k), IB);
    /* the same operations on every tile column n > k */
#pragma omp parallel for schedule(static, 1)
    for (int64_t n = k + 1; n < NT; ++n) {
      for (int64_t d = 0; d < nh; ++d) {
        int64_t h = heads[d], end = (h / BS + 1) * BS < MT ? (h / BS + 1) * BS : MT;
        oracle_larfb('T', NB, IB, TILE(h, k), (int)ldp, TT(h, k), IB, TILE(h, n), (int)ldp, NB);
        for (int64_t m = h + 1; m < end; ++m)
          oracle_ssrfb('T', NB, IB, TILE(m, k), (int)ldp, TT(m, k), IB, TILE(h, n), (int)ldp,
                       TILE(m, n), (int)ldp, NB);
      }
      for (int64_t s = 1; s < nh; s *= 2)
        for (int64_t i = 0; i + s < nh; i += 2 * s)
          oracle_ttmqrt('T', NB, IB, TILE(heads[i + s], k), (int)ldp, TT2(heads[i + s], k), IB,
                        TILE(heads[i], n), (int)ldp, TILE(heads[i + s], n), (int)ldp, NB);
    }
  }
  for (int64_t j = 0; j < N; ++j)
    for (int64_t i = 0; i < M; ++i) EL(A, lda, i, j) = EL(P, ldp, i, j);
  free(P);
  free(heads);
#undef TILE
#undef TT
#undef TT2
  return 0;
}

/* ------------------------------------------------------------------------ *
 * Apply the Q of a tree tile QR (oracle_tileqr_factor_tree, same NB, IB, BS)
 * to B (M x NRHS): 'T' replays the factorization's operations (k ascending;
 * domains, then the merges in tree order); 'N' runs them backwards (k
 * descending; merges in reverse order, then domains in reverse with the TS
 * chain descending, each kernel with trans 'N').
 * ------------------------------------------------------------------------ */
int oracle_tileqr_apply_tree(char trans, int64_t M, int64_t NRHS, int64_t K, const double *A, int64_t lda,
                             const double *T, int NB, int IB, int64_t BS, double *B, int64_t ldb,
                             int nthreads) {
  if (M == 0 || NRHS == 0 || K == 0) return 0;
  if (BS < 1) BS = 1;
  int64_t MT = (M + NB - 1) / NB, KTt = (K + NB - 1) / NB;
  int64_t KT = MT < KTt ? MT : KTt;
  int64_t ldp = MT * NB;
  const size_t tsz = (size_t)(MT * KTt) * IB * NB;
  double *V = (double *)calloc((size_t)ldp * (size_t)(KT * NB), sizeof(double));
  double *Bp = (double *)calloc((size_t)ldp * (size_t)NRHS, sizeof(double));
  int64_t *heads = (int64_t *)malloc(sizeof(int64_t) * (size_t)(MT + 1));
  if (!V || !Bp || !heads) { free(V); free(Bp); free(heads); return -1; }
  for (int64_t j = 0; j < K && j < KT * NB; ++j)
    for (int64_t i = 0; i < M; ++i) EL(V, ldp, i, j) = EL(A, lda, i, j);
  for (int64_t j = 0; j < NRHS; ++j)
    for (int64_t i = 0; i < M; ++i) EL(Bp, ldp, i, j) = EL(B, ldb, i, j);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#define VT(m, k) (&EL(V, ldp, (m) * NB, (k) * NB))
#define T1(m, k) (T + ((size_t)(m) + (size_t)(k) * MT) * IB * NB)
#define T2(m, k) (T + tsz + ((size_t)(m) + (size_t)(k) * MT) * IB * NB)
  for (int64_t kk = 0; kk < KT; ++kk) {
    int64_t k = (trans == 'T') ? kk : KT - 1 - kk;
    int64_t nh = tree_heads(MT, k, BS, heads);
    int64_t top = 1;
    while (top < nh) top *= 2;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < NRHS; ++c) {
      double *bc = &EL(Bp, ldp, 0, c);
      if (trans == 'T') {
        for (int64_t d = 0; d < nh; ++d) {
          int64_t h = heads[d], end = (h / BS + 1) * BS < MT ? (h / BS + 1) * BS : MT;
          oracle_larfb('T', NB, IB, VT(h, k), (int)ldp, T1(h, k), IB, bc + h * NB, (int)ldp, 1);
          for (int64_t m = h + 1; m < end; ++m)
            oracle_ssrfb('T', NB, IB, VT(m, k), (int)ldp, T1(m, k), IB, bc + h * NB, (int)ldp, bc + m * NB,
                         (int)ldp, 1);
        }
        for (int64_t s = 1; s < nh; s *= 2)
          for (int64_t i = 0; i + s < nh; i += 2 * s)
            oracle_ttmqrt('T', NB, IB, VT(heads[i + s], k), (int)ldp, T2(heads[i + s], k), IB,
                          bc + heads[i] * NB, (int)ldp, bc + heads[i + s] * NB, (int)ldp, 1);
      } else {
        for (int64_t s = top / 2; s >= 1; s /= 2) {
          int64_t last = -1;
          for (int64_t i = 0; i + s < nh; i += 2 * s) last = i;
          for (int64_t i = last; i >= 0; i -= 2 * s)
            oracle_ttmqrt('N', NB, IB, VT(heads[i + s], k), (int)ldp, T2(heads[i + s], k), IB,
                          bc + heads[i] * NB, (int)ldp, bc + heads[i + s] * NB, (int)ldp, 1);
        }
        for (int64_t d = nh - 1; d >= 0; --d) {
          int64_t h = heads[d], end = (h / BS + 1) * BS < MT ? (h / BS + 1) * BS : MT;
          for (int64_t m = end - 1; m > h; --m)
            oracle_ssrfb('N', NB, IB, VT(m, k), (int)ldp, T1(m, k), IB, bc + h * NB, (int)ldp, bc + m * NB,
                         (int)ldp, 1);
          oracle_larfb('N', NB, IB, VT(h, k), (int)ldp, T1(h, k), IB, bc + h * NB, (int)ldp, 1);
        }
      }
    }
  }
  for (int64_t j = 0; j < NRHS; ++j)
    for (int64_t i = 0; i < M; ++i) EL(B, ldb, i, j) = EL(Bp, ldp, i, j);
  free(V);
  free(Bp);
  free(heads);
#undef VT
#undef T1
#undef T2
  return 0;
}
