/*
 * oracle/hqr_oracle.c -- plain, slow CPU oracle for ONE small-bulge multishift QR sweep.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or helper with
 * the CUDA product path (paper_2007_03576_b200/csrc); neither includes or links the other.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, cited as P:<line>):
 *   One QR iteration is a product of orthogonal similarities H <- Q^T H Q, Z <- Z Q
 *   (Eq. "H <- Q_k^T ... Q_1^T H Q_1 ... Q_k").  For the multishift sweep the method
 *   reaches exactly (up to rounding order) the result of nshifts/2 textbook double-implicit-shift
 *   (Francis) steps, one per shift pair, pair 0 first (P:198-206 the double-shift step, P:206
 *   implicit-Q theorem, P:227-233 tightly-coupled bulges "chased ... as a single unit").  This
 *   file writes that plain definition out: every 3x3 (final: 2x2) Householder reflector is applied
 *   directly to the full matrix H (rows 0..n-1, the "wantt" convention) and to all n rows of Z.
 *
 * Readings of the paper (listed in DESIGN.md "Readings"):
 *   R1 bulge vector: first column of (H - s I)(H - s' I) in real form.
 *   R2 Householder: beta = -sign(x0)*||x||, sign(0)=+1, tau = (beta-x0)/beta,
 *      v = [1, x1/(x0-beta), ...]; zero tail => tau = 0, beta = x0 (identity).
 *   R3 shift pairs: consecutive (2j, 2j+1); sigma = s+s', pi = s*s' (= re*re' - im*im').
 *   R6 no vigilant deflation during the sweep.  R9 annihilated entries stored as exact 0.0.
 *   R15 the reflector and bulge vectors are computed on inputs scaled by a power of two (exact:
 *      bit-identical where the unscaled formulas stay finite, finite where they would not).
 *
 * Layout: column-major doubles, leading dimension n (element (i,j) at i + j*n).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EL(A, i, j, ld) (A)[(size_t)(i) + (size_t)(j) * (size_t)(ld)]

/* Scaling by a power of two (reading R15): for amax = m 2^e with m in [0.5, 1),
 * returns e; x * 2^-e is exact (no rounding) whenever it is a normal number, so the scaled
 * formulas below give bit-identical results to the unscaled ones wherever those do not overflow or
 * underflow, and stay finite where they would (|H| up to ~1e300, down to ~1e-300).  Any nonzero
 * scaling of x gives the same reflector (SURVEY §8(c) reading 1). */
static int pow2_exponent(double amax) {
  int e;
  (void)frexp(amax, &e);
  return e;
}

/* R2: Householder reflector of length m (2 or 3) mapping x to beta*e1 ("generate a 3-by-3
 * Householder reflector Q1 such that Q1^T v is a multiple of e1").  P = I - tau v v^T.
 * Computed on x scaled by 2^-e (R15); beta is scaled back. */
void oracle_house(int m, const double* x, double* v, double* tau, double* beta) {
  double amax = 0.0;
  for (int i = 0; i < m; ++i) amax = fmax(amax, fabs(x[i]));
  v[0] = 1.0;
  for (int i = 1; i < m; ++i) v[i] = 0.0;
  *tau = 0.0;
  *beta = x[0];
  if (amax == 0.0) return;
  const int e = pow2_exponent(amax);
  double xs[3];
  for (int i = 0; i < m; ++i) xs[i] = ldexp(x[i], -e);
  double alpha = xs[0];
  double tail2 = 0.0;
  for (int i = 1; i < m; ++i) tail2 += xs[i] * xs[i];
  if (tail2 == 0.0) return; /* zero tail: P = I, beta = x0 */
  double norm = sqrt(alpha * alpha + tail2);
  double b = (alpha >= 0.0) ? -norm : norm; /* sign(0) = +1 */
  *tau = (b - alpha) / b;
  for (int i = 1; i < m; ++i) v[i] = xs[i] / (alpha - b);
  *beta = ldexp(b, e);
}

/* R1: x = (H - s I)(H - s' I) e_ilo restricted to rows ilo..ilo+2, in real arithmetic
 * ("v = (H - l1 I)(H - l2 I) e1"), with sigma = s + s' and pi = s s' = re re' - im im'
 * (R3).  Returned scaled (R15): the true vector is x * 2^(*e2); every input is multiplied by the
 * same 2^-e first, so x = 2^-2e times the unscaled expression, rounding for rounding. */
void oracle_first_column(const double* H, int64_t n, int64_t ilo, double re0, double re1,
                         double im0, double im1, double* x, int* e2) {
  double h00 = EL(H, ilo, ilo, n), h01 = EL(H, ilo, ilo + 1, n);
  double h10 = EL(H, ilo + 1, ilo, n), h11 = EL(H, ilo + 1, ilo + 1, n);
  double h21 = EL(H, ilo + 2, ilo + 1, n);
  const double all[9] = {h00, h01, h10, h11, h21, re0, re1, im0, im1};
  double amax = 0.0;
  for (int i = 0; i < 9; ++i) amax = fmax(amax, fabs(all[i]));
  const int e = amax == 0.0 ? 0 : pow2_exponent(amax);
  h00 = ldexp(h00, -e); h01 = ldexp(h01, -e); h10 = ldexp(h10, -e);
  h11 = ldexp(h11, -e); h21 = ldexp(h21, -e);
  re0 = ldexp(re0, -e); re1 = ldexp(re1, -e); im0 = ldexp(im0, -e); im1 = ldexp(im1, -e);
  const double sigma = re0 + re1;
  const double pi = re0 * re1 - im0 * im1;
  x[0] = h00 * (h00 - sigma) + h01 * h10 + pi;
  x[1] = h10 * (h00 + h11 - sigma);
  x[2] = h10 * h21;
  *e2 = 2 * e;
}

/* Apply the reflector of bulge j at position p (acting on rows/cols p+1..p+m) to the full H and Z,
 * exactly as one step of the textbook chase: compute the vector, apply from the left to
 * rows p+1..p+m (all columns to the right), store beta / exact zeros in column p, apply from the
 * right to columns p+1..p+m (all rows above the bulge), and accumulate into Z (all n rows). */
static void apply_one(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, int64_t p,
                      const double* sr, const double* si, int j) {
  int m = (p <= ihi - 3) ? 3 : 2;
  double x[3], v[3], tau, beta;
  if (p == ilo - 1) { /* bulge j: shifts (2j, 2j+1), R3 */
    int e2;
    oracle_first_column(H, n, ilo, sr[2 * j], sr[2 * j + 1], si[2 * j], si[2 * j + 1], x, &e2);
  } else {
    for (int i = 0; i < m; ++i) x[i] = EL(H, p + 1 + i, p, n);
  }
  oracle_house(m, x, v, &tau, &beta);

  /* left: H(p+1..p+m, c) -= tau v (v^T H(p+1..p+m, c)) for c = first..n-1 */
  int64_t c0 = (p == ilo - 1) ? ilo : p + 1;
#pragma omp parallel for schedule(static) if (n - c0 > 2048)
  for (int64_t c = c0; c < n; ++c) {
    double w = 0.0;
    for (int i = 0; i < m; ++i) w += v[i] * EL(H, p + 1 + i, c, n);
    for (int i = 0; i < m; ++i) EL(H, p + 1 + i, c, n) -= tau * v[i] * w;
  }
  if (p >= ilo) { /* R9: annihilated column stored exactly */
    EL(H, p + 1, p, n) = beta;
    for (int i = 1; i < m; ++i) EL(H, p + 1 + i, p, n) = 0.0;
  }
  /* right: H(r, p+1..p+m) -= tau (H(r, p+1..p+m) v) v^T for r = 0..min(p+m+1, ihi) */
  int64_t r1 = (p + m + 1 < ihi) ? p + m + 1 : ihi;
#pragma omp parallel for schedule(static) if (r1 > 2048)
  for (int64_t r = 0; r <= r1; ++r) {
    double w = 0.0;
    for (int i = 0; i < m; ++i) w += EL(H, r, p + 1 + i, n) * v[i];
    for (int i = 0; i < m; ++i) EL(H, r, p + 1 + i, n) -= tau * w * v[i];
  }
  /* Z <- Z P ("Q <- Q Q_1 ... Q_k"), all rows */
  if (Z) {
#pragma omp parallel for schedule(static) if (n > 2048)
    for (int64_t r = 0; r < n; ++r) {
      double w = 0.0;
      for (int i = 0; i < m; ++i) w += EL(Z, r, p + 1 + i, n) * v[i];
      for (int i = 0; i < m; ++i) EL(Z, r, p + 1 + i, n) -= tau * w * v[i];
    }
  }
}

/*
 * The oracle: one multishift sweep as nshifts/2 sequential Francis double-shift steps (SURVEY §8(c)
 * algorithm).  order = 0: sequential (bulge 0 sweeps the whole block, then
 * bulge 1, ...).  order = 1: pipelined (step t: bulge j at p = ilo-1+t-3j, lowest bulge first;
 * P:228 "chasing them down the diagonal just enough so that the next bulge can be introduced").
 * Order 1 is used only to measure the rounding noise floor between two valid orders.
 * Bulges j0 .. j1-1 only (j0 = 0, j1 = nshifts/2 is the whole sweep; a sub-range is the bounded
 * CPU-baseline sample).  Returns 0.  No argument validation: callers pass valid input.
 */
int oracle_sweep(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, const double* sr,
                 const double* si, int nshifts, int order, int j0, int j1) {
  (void)nshifts;
  if (order == 0) {
    for (int j = j0; j < j1; ++j)
      for (int64_t p = ilo - 1; p <= ihi - 2; ++p) apply_one(H, Z, n, ilo, ihi, p, sr, si, j);
  } else {
    int nb = j1 - j0;
    int64_t last = (ihi - 2) - (ilo - 1) + 3 * (int64_t)(nb - 1);
    for (int64_t t = 0; t <= last; ++t) {
      for (int jj = 0; jj < nb; ++jj) { /* lowest (earliest introduced) first */
        int64_t p = ilo - 1 + t - 3 * (int64_t)jj;
        if (p < ilo - 1 || p > ihi - 2) continue;
        apply_one(H, Z, n, ilo, ihi, p, sr, si, j0 + jj);
      }
    }
  }
  return 0;
}

/* F_alg: flops of applying every reflector directly, per bulge:
 * 10*[(n - max(p+1, ilo)) + (min(p+4, ihi)+1) + n] per 3-reflector, 6*[...] for the final one. */
double oracle_flops(int64_t n, int64_t ilo, int64_t ihi, int nbulges, int with_z) {
  double f = 0.0;
  for (int64_t p = ilo - 1; p <= ihi - 2; ++p) {
    int m = (p <= ihi - 3) ? 3 : 2;
    int64_t c0 = (p == ilo - 1) ? ilo : p + 1;
    int64_t r1 = (p + m + 1 < ihi) ? p + m + 1 : ihi;
    double per = (m == 3) ? 10.0 : 6.0;
    f += per * ((double)(n - c0) + (double)(r1 + 1) + (with_z ? (double)n : 0.0));
  }
  return f * nbulges;
}

/* Subdiagonal scan (check only; "scanning the sub-diagonal entries in order to identify
 * any unreduced blocks that were decoupled during the bulge chasing step ... stored to a special
 * aftermath vector that has an entry for each row of the matrix"), reading R16: for every row i
 * with ilo-1 <= i <= ihi (and 0 <= i <= n-2), h = H[i+1, i], d = |H[i,i]| + |H[i+1,i+1]|:
 *   flags[i] = 2 if h == 0 (decoupled), 1 if |h| <= 2^-52 d (negligible by the standard
 *   criterion), else 0.  Other entries are left as they are (the caller initialises them). */
void oracle_subdiag_scan(const double* H, int64_t n, int64_t ilo, int64_t ihi, signed char* flags) {
  int64_t i0 = ilo - 1 < 0 ? 0 : ilo - 1;
  int64_t i1 = ihi < n - 2 ? ihi : n - 2;
  for (int64_t i = i0; i <= i1; ++i) {
    double h = EL(H, i + 1, i, n);
    double d = fabs(EL(H, i, i, n)) + fabs(EL(H, i + 1, i + 1, n));
    flags[i] = (h == 0.0) ? 2 : (fabs(h) <= 0x1p-52 * d) ? 1 : 0;
  }
}

/* ===================================================================================================
 * Generalized (QZ) sweep -- SURVEY §8(f) NEXT-4; PAPER.md P:208-213 (the generalized double-shift
 * step) and P:412-439 (push bulges on a Hessenberg-triangular pair).  Test infrastructure like the
 * rest of this file.
 *
 * One multishift QZ sweep on a Hessenberg-triangular pair (H, T): (H, T) <- Q^T (H, T) Z,
 * Qacc <- Qacc Q, Zacc <- Zacc Z, the product of nshifts/2 sequential double-shift QZ steps (pair 0
 * first).  Per step (P:209-211 and the textbook QZ step it cites, Moler-Stewart): the bulge vector
 * v = (H T^-1 - s I)(H T^-1 - s' I) e_ilo (reading R17), a 3x3 Householder reflector from the left,
 * then, at every position p, a left reflector from H's column p (rows p+1..p+m) and two "right-hand
 * side" reflectors from the right that return T to triangular form: the first from T's row p+3
 * (columns p+1..p+3, zeroing T[p+3, p+1..p+2]), the second from T's row p+2 (columns p+1..p+2,
 * zeroing T[p+2, p+1]); at the last position (m = 2) a single 2-element right reflector.
 * =================================================================================================== */

/* Right-hand side reflector (reading R18): for a row vector r of length m (2 or 3) returns u
 * (u[m-1] = 1) and tau with r (I - tau u u^T) = beta e_m^T -- the R2 reflector of the reversed
 * vector (r[m-1], ..., r[0]), reversed. */
void oracle_rhs_house(int m, const double* r, double* u, double* tau, double* beta) {
  double x[3], v[3];
  for (int i = 0; i < m; ++i) x[i] = r[m - 1 - i];
  oracle_house(m, x, v, tau, beta);
  for (int i = 0; i < m; ++i) u[i] = v[m - 1 - i];
}

/* R17: v = (M - s I)(M - s' I) e_1 at rows ilo..ilo+2, M = H T^-1 on the active block, with
 * sigma = s + s', pi = s s' (R3).  M e1 = (h00/t00, h10/t00, 0); y = T^-1 M e1 has y1 = h10/(t00 t11)
 * and y0 = (h00/t00 - t01 y1)/t00; M^2 e1 = H y. */
void oracle_qz_first_column(const double* H, const double* T, int64_t n, int64_t ilo, double re0,
                            double re1, double im0, double im1, double* x) {
  const double h00 = EL(H, ilo, ilo, n), h01 = EL(H, ilo, ilo + 1, n);
  const double h10 = EL(H, ilo + 1, ilo, n), h11 = EL(H, ilo + 1, ilo + 1, n);
  const double h21 = EL(H, ilo + 2, ilo + 1, n);
  const double t00 = EL(T, ilo, ilo, n), t01 = EL(T, ilo, ilo + 1, n), t11 = EL(T, ilo + 1, ilo + 1, n);
  const double sigma = re0 + re1, pi = re0 * re1 - im0 * im1;
  const double a = h00 / t00, b = h10 / t00;
  const double y1 = b / t11;
  const double y0 = (a - t01 * y1) / t00;
  x[0] = h00 * y0 + h01 * y1 - sigma * a + pi;
  x[1] = h10 * y0 + h11 * y1 - sigma * b;
  x[2] = h21 * y1;
}

static void left_rows(double* A, int64_t n, int64_t r0, int m, int64_t c0, int64_t c1, const double* v,
                      double tau) { /* A(r0..r0+m-1, c0..c1-1) -= tau v (v^T A) */
#pragma omp parallel for schedule(static) if (c1 - c0 > 2048)
  for (int64_t c = c0; c < c1; ++c) {
    double w = 0.0;
    for (int i = 0; i < m; ++i) w += v[i] * EL(A, r0 + i, c, n);
    for (int i = 0; i < m; ++i) EL(A, r0 + i, c, n) -= tau * v[i] * w;
  }
}

static void right_cols(double* A, int64_t n, int64_t c0, int m, int64_t r1, const double* u, double tau) {
  /* A(0..r1, c0..c0+m-1) -= tau (A u) u^T */
#pragma omp parallel for schedule(static) if (r1 > 2048)
  for (int64_t r = 0; r <= r1; ++r) {
    double w = 0.0;
    for (int i = 0; i < m; ++i) w += EL(A, r, c0 + i, n) * u[i];
    for (int i = 0; i < m; ++i) EL(A, r, c0 + i, n) -= tau * w * u[i];
  }
}

static void qz_apply_one(double* H, double* T, double* Qa, double* Za, int64_t n, int64_t ilo, int64_t ihi,
                         int64_t p, const double* sr, const double* si, int j) {
  const int m = (p <= ihi - 3) ? 3 : 2;
  double x[3], v[3], tau, beta;
  if (p == ilo - 1)
    oracle_qz_first_column(H, T, n, ilo, sr[2 * j], sr[2 * j + 1], si[2 * j], si[2 * j + 1], x);
  else
    for (int i = 0; i < m; ++i) x[i] = EL(H, p + 1 + i, p, n);
  oracle_house(m, x, v, &tau, &beta);
  /* left: rows p+1..p+m of H (columns from ilo / p+1) and T (columns from p+1), Qacc columns */
  left_rows(H, n, p + 1, m, (p == ilo - 1) ? ilo : p + 1, n, v, tau);
  if (p >= ilo) {
    EL(H, p + 1, p, n) = beta;
    for (int i = 1; i < m; ++i) EL(H, p + 1 + i, p, n) = 0.0;
  }
  left_rows(T, n, p + 1, m, p + 1, n, v, tau);
  if (Qa) right_cols(Qa, n, p + 1, m, n - 1, v, tau);
  /* right: restore T's triangular form, last row of the block first */
  const int64_t hr = (p + 4 < ihi) ? p + 4 : ihi;
  for (int mm = m; mm >= 2; --mm) {
    const int64_t row = p + mm; /* T row whose entries left of the diagonal are zeroed */
    double r[3], u[3], tz, bz;
    for (int i = 0; i < mm; ++i) r[i] = EL(T, row, p + 1 + i, n);
    oracle_rhs_house(mm, r, u, &tz, &bz);
    right_cols(H, n, p + 1, mm, hr, u, tz);
    right_cols(T, n, p + 1, mm, row, u, tz);
    for (int i = 0; i < mm - 1; ++i) EL(T, row, p + 1 + i, n) = 0.0; /* R9: exact zeros */
    EL(T, row, row, n) = bz;
    if (Za) right_cols(Za, n, p + 1, mm, n - 1, u, tz);
  }
}

/* The QZ oracle: nshifts/2 sequential double-shift QZ steps, bulges j0 .. j1-1.  Qa / Za may be
 * NULL.  No argument validation. */
int oracle_qz_sweep(double* H, double* T, double* Qa, double* Za, int64_t n, int64_t ilo, int64_t ihi,
                    const double* sr, const double* si, int j0, int j1) {
  for (int j = j0; j < j1; ++j)
    for (int64_t p = ilo - 1; p <= ihi - 2; ++p) qz_apply_one(H, T, Qa, Za, n, ilo, ihi, p, sr, si, j);
  return 0;
}

/* ===================================================================================================
 * QR iteration (partial; PAPER.md P:270-297 shifts, P:370-381 deflation,
 * P:1142-1189 deflation criteria): repeated sweeps whose shifts are the eigenvalues of the trailing
 * nshifts x nshifts block of the active block, with the small-subdiagonal deflation test after every
 * sweep.  (The paper's AED -- deflating eigenvalues of the trailing window through the spike and
 * reordering -- is not reproduced: reading R21.)  Test infrastructure like the rest of this file.
 * =================================================================================================== */

/* Eigenvalues of a 2x2 block [[a, b], [c, d]] (reading R21): tr/2 +- sqrt((a-d)^2/4 + bc); a
 * real pair is returned larger-magnitude root first computed as tr/2 + sign(tr/2) sqrt(disc) and
 * the other as det / that root (no cancellation); a complex pair as re +- i im. */
static void eig2(double a, double b, double c, double d, double* wr1, double* wi1, double* wr2, double* wi2) {
  const double h = 0.5 * (a + d);
  const double q = 0.5 * (a - d);
  const double disc = q * q + b * c;
  if (disc >= 0.0) {
    const double r = sqrt(disc);
    const double l1 = (h >= 0.0) ? h + r : h - r;
    const double det = a * d - b * c;
    const double l2 = (l1 != 0.0) ? det / l1 : h - (l1 - h);
    *wr1 = l1; *wi1 = 0.0; *wr2 = l2; *wi2 = 0.0;
  } else {
    const double im = sqrt(-disc);
    *wr1 = h; *wi1 = im; *wr2 = h; *wi2 = -im;
  }
}

/* Eigenvalues of the m x m upper-Hessenberg matrix A (column-major, ld lda; overwritten) by the
 * textbook Francis double-shift QR iteration with deflation (Golub & Van Loan Alg. 7.5.2, the
 * paper's small Schur task P:367-372 uses LAPACK's DHSEQR for this), eigenvalues only: reflectors
 * act on the active block [l, i] only.  Deflation test R16 (|h(k,k-1)| <= 2^-52 (|h(k-1,k-1)| +
 * |h(k,k)|) -> 0); exceptional shifts after 10 and 20 iterations without deflation.
 * Returns 0, or the number of eigenvalues not found (iteration limit 30 m). */
int oracle_small_eig(double* A, int64_t m, int64_t lda, double* wr, double* wi) {
#define A_(r, c) A[(size_t)(r) + (size_t)(c) * (size_t)lda]
  int64_t i = m - 1;
  int64_t total = 0;
  while (i >= 0) {
    int its = 0;
    int64_t l = 0;
    for (;;) {
      /* deflation: the lowest negligible subdiagonal of the active part */
      for (l = i; l > 0; --l) {
        const double s = fabs(A_(l - 1, l - 1)) + fabs(A_(l, l));
        if (fabs(A_(l, l - 1)) <= 0x1p-52 * s) {
          A_(l, l - 1) = 0.0;
          break;
        }
      }
      if (l >= i - 1) break;
      if (++total > 30 * m) return (int)(i + 1);
      ++its;
      double sigma, pi;
      if (its == 10 || its == 20) { /* exceptional shift (as LAPACK's dlahqr) */
        const double s = fabs(A_(i, i - 1)) + fabs(A_(i - 1, i - 2));
        const double h11 = 0.75 * s + A_(i, i);
        sigma = 2.0 * h11;
        pi = h11 * h11 + 0.4375 * s * s;
      } else { /* the trailing 2x2 block's eigenvalues (Francis) */
        const double a = A_(i - 1, i - 1), b = A_(i - 1, i), c = A_(i, i - 1), d = A_(i, i);
        sigma = a + d;
        pi = a * d - b * c;
      }
      /* double-shift sweep on [l, i] */
      for (int64_t p = l - 1; p <= i - 2; ++p) {
        const int mm = (p <= i - 3) ? 3 : 2;
        double x[3], v[3], tau, beta;
        if (p == l - 1) {
          const double h00 = A_(l, l), h01 = A_(l, l + 1), h10 = A_(l + 1, l), h11 = A_(l + 1, l + 1);
          const double h21 = A_(l + 2, l + 1);
          x[0] = h00 * (h00 - sigma) + h01 * h10 + pi;
          x[1] = h10 * (h00 + h11 - sigma);
          x[2] = h10 * h21;
        } else {
          for (int k = 0; k < mm; ++k) x[k] = A_(p + 1 + k, p);
        }
        oracle_house(mm, x, v, &tau, &beta);
        const int64_t c0 = (p == l - 1) ? l : p + 1;
        for (int64_t c = c0; c <= i; ++c) {
          double w = 0.0;
          for (int k = 0; k < mm; ++k) w += v[k] * A_(p + 1 + k, c);
          for (int k = 0; k < mm; ++k) A_(p + 1 + k, c) -= tau * v[k] * w;
        }
        if (p >= l) {
          A_(p + 1, p) = beta;
          for (int k = 1; k < mm; ++k) A_(p + 1 + k, p) = 0.0;
        }
        const int64_t r1 = (p + mm + 1 < i) ? p + mm + 1 : i;
        for (int64_t r = l; r <= r1; ++r) {
          double w = 0.0;
          for (int k = 0; k < mm; ++k) w += A_(r, p + 1 + k) * v[k];
          for (int k = 0; k < mm; ++k) A_(r, p + 1 + k) -= tau * w * v[k];
        }
      }
    }
    if (l == i) {
      wr[i] = A_(i, i);
      wi[i] = 0.0;
      i -= 1;
    } else {
      eig2(A_(i - 1, i - 1), A_(i - 1, i), A_(i, i - 1), A_(i, i), &wr[i - 1], &wi[i - 1], &wr[i], &wi[i]);
      i -= 2;
    }
  }
#undef A_
  return 0;
}

/* Shifts from m eigenvalues (R21): the complex pairs in the order found (positive imaginary part
 * first, its exact conjugate next), then the real ones paired in the order found; at most ns
 * (even).  Returns the number of shifts written (even). */
static int make_shifts(const double* wr, const double* wi, int64_t m, int ns, double* sr, double* si) {
  int k = 0;
  /* complex pairs as they appear (wi > 0 followed by its conjugate), then reals in pairs */
  for (int64_t j = 0; j < m && k + 1 < ns; ++j)
    if (wi[j] > 0.0) {
      sr[k] = wr[j]; si[k] = wi[j]; sr[k + 1] = wr[j]; si[k + 1] = -wi[j];
      k += 2;
    }
  int64_t pending = -1;
  for (int64_t j = 0; j < m && k + 1 < ns; ++j)
    if (wi[j] == 0.0) {
      if (pending < 0) {
        pending = j;
      } else {
        sr[k] = wr[pending]; si[k] = 0.0; sr[k + 1] = wr[j]; si[k + 1] = 0.0;
        k += 2;
        pending = -1;
      }
    }
  return k;
}

/* The QR iteration on H (n x n, active block [ilo, ihi]) with Z: until every unreduced block is at
 * most nmin long, sweep the bottom unreduced block [l, hi] with the eigenvalues of its trailing
 * nshifts x nshifts block as shifts (oracle_sweep), then set negligible subdiagonals (R16) to zero;
 * the remaining small blocks in real Schur form (small_block_schur, R24), so H ends quasi-triangular.
 * wr / wi: n entries (rows outside [ilo, ihi] untouched).  Returns 0, or -(sweeps) when max_sweeps
 * was reached. */
int oracle_aed(double* H, double* Z, int64_t n, int64_t ilo, int64_t k0, int nw, double thr, double* wr,
               double* wi, double* swr, double* swi, int* nund);

/* A small unreduced block [l, hi] (N = hi-l+1 rows, h(l, l-1) = 0) at the end of the QR iteration, in
 * real Schur form (reading R24: LAPACK's wantt / wantz): N = 1 is its own eigenvalue; 2 <= N <= 112
 * (the GPU's one-CTA window) goes through oracle_aed on the window [l, hi] with l as the block start,
 * so the spike is zero and every block deflates -- T (real Schur form) written back, its factor
 * applied to the rest of H and to Z; larger blocks: the eigenvalues only (oracle_small_eig). */
static void small_block_schur(double* H, double* Z, int64_t n, int64_t l, int64_t hi, double* B, double* wr,
                              double* wi) {
  const int64_t N = hi - l + 1;
  if (N == 1) {
    wr[l] = EL(H, l, l, n);
    wi[l] = 0.0;
  } else if (N <= 112) {
    double* sw = (double*)malloc(sizeof(double) * 2 * (size_t)N);
    int nund = 0;
    oracle_aed(H, Z, n, l, l, (int)N, 0.0, wr, wi, sw, sw + N, &nund);
    free(sw);
  } else {
    for (int64_t c = 0; c < N; ++c)
      for (int64_t r = 0; r < N; ++r) B[r + c * N] = EL(H, l + r, l + c, n);
    oracle_small_eig(B, N, N, wr + l, wi + l);
  }
}

int oracle_qr_iterate(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, int nshifts, int64_t nmin,
                      int max_sweeps, double* wr, double* wi, int* sweeps_out) {
  int sweeps = 0;
  int64_t hi = ihi;
  double* work = (double*)malloc(sizeof(double) * (size_t)(nshifts * nshifts + 4 * nshifts + nmin * nmin + 8));
  while (hi >= ilo) {
    int64_t l = hi;
    while (l > ilo && EL(H, l, l - 1, n) != 0.0) --l;
    const int64_t N = hi - l + 1;
    if (N <= nmin) {
      small_block_schur(H, Z, n, l, hi, work, wr, wi);
      hi = l - 1;
      continue;
    }
    if (sweeps >= max_sweeps) {
      free(work);
      *sweeps_out = sweeps;
      return -sweeps;
    }
    int ns = nshifts;
    if (ns > N - 2) ns = (int)((N - 2) & ~(int64_t)1);
    if (ns < 2) ns = 2;
    double* B = work;
    double* ewr = B + (size_t)ns * ns;
    double* ewi = ewr + ns;
    double* sr = ewi + ns;
    double* si = sr + ns;
    for (int c = 0; c < ns; ++c)
      for (int r = 0; r < ns; ++r) B[r + c * ns] = EL(H, hi - ns + 1 + r, hi - ns + 1 + c, n);
    oracle_small_eig(B, ns, ns, ewr, ewi);
    const int k = make_shifts(ewr, ewi, ns, ns, sr, si);
    oracle_sweep(H, Z, n, l, hi, sr, si, k, 0, 0, k / 2);
    ++sweeps;
    for (int64_t r = l + 1; r <= hi; ++r) { /* deflation (R16 criterion), after the sweep */
      const double s = fabs(EL(H, r - 1, r - 1, n)) + fabs(EL(H, r, r, n));
      if (fabs(EL(H, r, r - 1, n)) <= 0x1p-52 * s) EL(H, r, r - 1, n) = 0.0;
    }
  }
  free(work);
  *sweeps_out = sweeps;
  return 0;
}

/* ===================================================================================================
 * Aggressive early deflation (deflation conditions
 * P:1142-1189; reading R22): on the trailing nw x nw window of an unreduced block,
 *   (1) reduce the window to real Schur form T = U^T W U (Francis double-shift QR with deflation,
 *       all window columns / rows updated, U accumulated);
 *   (2) the spike v = s U(0, :) (s = the subdiagonal entry left of the window); from the bottom,
 *       a 1x1 / 2x2 block of T is deflated when its spike entries are <= u ||H||_F (the paper's
 *       default "norm-stable" condition); a block that fails is moved above the remaining
 *       unevaluated blocks by swaps of adjacent diagonal blocks (oracle_swap, R23), which
 *       pushes those down; a rejected swap halts the reordering and the blocks not yet
 *       evaluated stay undeflated;
 *   (3) if anything deflated: zero the deflated spike entries, reflect the remaining spike v(0:m)
 *       onto e1 (P = I - tau w w^T, applied to T(0:m,0:m) from both sides and to U(:, 0:m)) and
 *       restore Hessenberg form of T(0:m, 0:m) by Householder reflectors (general length, R2
 *       convention), accumulated into U;
 *   (4) write T into H's window, the spike column (beta, 0, ...) left of it, and propagate U:
 *       H(window, right) <- U^T H(window, right), H(above, window) <- H(above, window) U,
 *       Z(:, window) <- Z(:, window) U.
 * The eigenvalues of T(0:m, 0:m) -- the failed candidates -- are the next sweep's shifts.
 * =================================================================================================== */

/* R2 Householder reflector of general length m (x overwritten by v, v[0] = 1).  Returns tau, beta. */
static void house_n(int m, double* x, double* tau, double* beta) {
  double tail2 = 0.0;
  for (int i = 1; i < m; ++i) tail2 += x[i] * x[i];
  const double alpha = x[0];
  if (tail2 == 0.0) {
    *tau = 0.0;
    *beta = alpha;
    x[0] = 1.0;
    for (int i = 1; i < m; ++i) x[i] = 0.0;
    return;
  }
  const double norm = sqrt(alpha * alpha + tail2);
  const double b = (alpha >= 0.0) ? -norm : norm;
  *tau = (b - alpha) / b;
  for (int i = 1; i < m; ++i) x[i] = x[i] / (alpha - b);
  x[0] = 1.0;
  *beta = b;
}

/* A(r0.., c0..c1) -= tau w (w^T A) for rows r0..r0+m-1 (ld lda) */
static void refl_left(double* A, int64_t lda, int64_t r0, int m, int64_t c0, int64_t c1, const double* w, double tau) {
  for (int64_t c = c0; c < c1; ++c) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += w[i] * A[(r0 + i) + c * lda];
    for (int i = 0; i < m; ++i) A[(r0 + i) + c * lda] -= tau * w[i] * s;
  }
}
/* A(r0..r1-1, c0..c0+m-1) -= tau (A w) w^T */
static void refl_right(double* A, int64_t lda, int64_t r0, int64_t r1, int64_t c0, int m, const double* w, double tau) {
  for (int64_t r = r0; r < r1; ++r) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += A[r + (c0 + i) * lda] * w[i];
    for (int i = 0; i < m; ++i) A[r + (c0 + i) * lda] -= tau * s * w[i];
  }
}

/* Swap of the adjacent diagonal blocks A = T(i:i+p, i:i+p) and B = T(i+p:i+p+q, i+p:i+p+q) of the
 * quasi-triangular T (nw x nw, ld ldt; p, q in {1, 2}) by an orthogonal similarity accumulated into U
 * (nw x nw, ld ldu) -- the eigenvalue reordering of P:289-290 (LAPACK's DTREXC), reading R23:
 *   X solves the Sylvester equation A X - X B = C, C = T(i:i+p, i+p:i+p+q), so that
 *   T [-X; I_q] = [-X; I_q] B: the columns of [-X; I_q] span B's invariant subspace;
 *   Q = P1 (P2) = the Householder (R2) QR factor of [-X; I_q]; T <- Q^T T Q puts B's eigenvalues in
 *   the leading q x q block; U <- U Q; the new lower-left p x q block is set to exact zeros.
 * The Sylvester equation is solved as its pq x pq Kronecker system (I_q (x) A - B^T (x) I_p) vec X =
 * vec C by Gaussian elimination with complete pivoting, a pivot below 2^-52 max|K| replaced by that
 * value (A and B sharing an eigenvalue).  The swap is rejected -- returns 1, T and U unchanged -- when
 * the lower-left block of Q^T D Q (D = the (p+q)^2 diagonal block) exceeds 10 * 2^-52 * max|D| (too
 * ill-conditioned).  Returns 0 on success. */
int oracle_swap(double* T, int64_t ldt, int64_t nw, double* U, int64_t ldu, int64_t i, int p, int q) {
  const int k = p + q;
  double D[16], K[16], x[4], w1[4], w2[4];
  double dnorm = 0.0;
  for (int c = 0; c < k; ++c)
    for (int r = 0; r < k; ++r) {
      D[r + 4 * c] = T[(i + r) + (i + c) * ldt];
      if (fabs(D[r + 4 * c]) > dnorm) dnorm = fabs(D[r + 4 * c]);
    }
  /* Kronecker system, unknown X(r, c) at index r + c p, equation (r, c) at row r + c p */
  const int nk = p * q;
  double kmax = 0.0;
  for (int e = 0; e < nk * nk; ++e) K[e] = 0.0;
  for (int c = 0; c < q; ++c)
    for (int r = 0; r < p; ++r) {
      const int row = r + c * p;
      for (int t = 0; t < p; ++t) K[row + nk * (t + c * p)] += D[r + 4 * t];            /* A(r,t) X(t,c) */
      for (int t = 0; t < q; ++t) K[row + nk * (r + t * p)] -= D[(p + t) + 4 * (p + c)]; /* X(r,t) B(t,c) */
      x[row] = D[r + 4 * (p + c)];                                                       /* C(r,c) */
    }
  for (int e = 0; e < nk * nk; ++e)
    if (fabs(K[e]) > kmax) kmax = fabs(K[e]);
  const double smin = (kmax > 0.0 ? kmax : 1.0) * 0x1p-52;
  int perm[4] = {0, 1, 2, 3}; /* column permutation (complete pivoting) */
  for (int j = 0; j < nk; ++j) {
    int pr = j, pc = j;
    for (int c = j; c < nk; ++c)
      for (int r = j; r < nk; ++r)
        if (fabs(K[r + nk * c]) > fabs(K[pr + nk * pc])) { pr = r; pc = c; }
    for (int c = 0; c < nk; ++c) { /* row swap */
      const double t = K[j + nk * c]; K[j + nk * c] = K[pr + nk * c]; K[pr + nk * c] = t;
    }
    { const double t = x[j]; x[j] = x[pr]; x[pr] = t; }
    for (int r = 0; r < nk; ++r) { /* column swap */
      const double t = K[r + nk * j]; K[r + nk * j] = K[r + nk * pc]; K[r + nk * pc] = t;
    }
    { const int t = perm[j]; perm[j] = perm[pc]; perm[pc] = t; }
    if (fabs(K[j + nk * j]) < smin) K[j + nk * j] = smin;
    for (int r = j + 1; r < nk; ++r) {
      const double f = K[r + nk * j] / K[j + nk * j];
      for (int c = j; c < nk; ++c) K[r + nk * c] -= f * K[j + nk * c];
      x[r] -= f * x[j];
    }
  }
  double y[4];
  for (int j = nk - 1; j >= 0; --j) {
    double a = x[j];
    for (int c = j + 1; c < nk; ++c) a -= K[j + nk * c] * y[c];
    y[j] = a / K[j + nk * j];
  }
  double X[4];
  for (int j = 0; j < nk; ++j) X[perm[j]] = y[j];
  /* Householder QR of M = [-X; I_q] (k x q) */
  double M[8];
  for (int c = 0; c < q; ++c)
    for (int r = 0; r < k; ++r) M[r + 4 * c] = (r < p) ? -X[r + c * p] : ((r - p == c) ? 1.0 : 0.0);
  double tau1, tau2 = 0.0, beta;
  for (int r = 0; r < k; ++r) w1[r] = M[r];
  house_n(k, w1, &tau1, &beta);
  if (q == 2) {
    double s = 0.0;
    for (int r = 0; r < k; ++r) s += w1[r] * M[r + 4];
    for (int r = 0; r < k; ++r) M[r + 4] -= tau1 * w1[r] * s;
    for (int r = 0; r < k - 1; ++r) w2[r] = M[1 + r + 4];
    house_n(k - 1, w2, &tau2, &beta);
  }
  /* the check on D: D' = Q^T D Q */
  refl_left(D, 4, 0, k, 0, k, w1, tau1);
  refl_right(D, 4, 0, k, 0, k, w1, tau1);
  if (q == 2) {
    refl_left(D, 4, 1, k - 1, 0, k, w2, tau2);
    refl_right(D, 4, 0, k, 1, k - 1, w2, tau2);
  }
  double low = 0.0;
  for (int c = 0; c < q; ++c)
    for (int r = q; r < k; ++r)
      if (fabs(D[r + 4 * c]) > low) low = fabs(D[r + 4 * c]);
  if (!(low <= 10.0 * 0x1p-52 * dnorm)) return 1;
  /* accepted: T <- Q^T T Q (rows i..i+k-1 from column i on; columns i..i+k-1 for rows 0..i+k-1),
   * U <- U Q, exact zeros below the new leading q x q block */
  refl_left(T, ldt, i, k, i, nw, w1, tau1);
  refl_right(T, ldt, 0, i + k, i, k, w1, tau1);
  refl_right(U, ldu, 0, nw, i, k, w1, tau1);
  if (q == 2) {
    refl_left(T, ldt, i + 1, k - 1, i, nw, w2, tau2);
    refl_right(T, ldt, 0, i + k, i + 1, k - 1, w2, tau2);
    refl_right(U, ldu, 0, nw, i + 1, k - 1, w2, tau2);
  }
  for (int c = 0; c < q; ++c)
    for (int r = q; r < k; ++r) T[(i + r) + (i + c) * ldt] = 0.0;
  return 0;
}

/* Real Schur form of the m x m Hessenberg matrix A (ld lda) with U (m x m, ld ldu) accumulated:
 * oracle_small_eig's iteration with every reflector applied to all columns right of / rows above the
 * active block (wantt) and to U (wantz).  Eigenvalues to wr / wi.  Returns 0 or the count not found. */
int oracle_schur(double* A, int64_t m, int64_t lda, double* U, int64_t ldu, double* wr, double* wi) {
#define A_(r, c) A[(size_t)(r) + (size_t)(c) * (size_t)lda]
  int64_t i = m - 1;
  int64_t total = 0;
  while (i >= 0) {
    int its = 0;
    int64_t l = 0;
    for (;;) {
      for (l = i; l > 0; --l) {
        const double s = fabs(A_(l - 1, l - 1)) + fabs(A_(l, l));
        if (fabs(A_(l, l - 1)) <= 0x1p-52 * s) {
          A_(l, l - 1) = 0.0;
          break;
        }
      }
      if (l >= i - 1) break;
      if (++total > 30 * m) return (int)(i + 1);
      ++its;
      double sigma, pi;
      if (its == 10 || its == 20) {
        const double s = fabs(A_(i, i - 1)) + fabs(A_(i - 1, i - 2));
        const double h11 = 0.75 * s + A_(i, i);
        sigma = 2.0 * h11;
        pi = h11 * h11 + 0.4375 * s * s;
      } else {
        const double a = A_(i - 1, i - 1), b = A_(i - 1, i), c = A_(i, i - 1), d = A_(i, i);
        sigma = a + d;
        pi = a * d - b * c;
      }
      for (int64_t p = l - 1; p <= i - 2; ++p) {
        const int mm = (p <= i - 3) ? 3 : 2;
        double x[3], v[3], tau, beta;
        if (p == l - 1) {
          const double h00 = A_(l, l), h01 = A_(l, l + 1), h10 = A_(l + 1, l), h11 = A_(l + 1, l + 1);
          const double h21 = A_(l + 2, l + 1);
          x[0] = h00 * (h00 - sigma) + h01 * h10 + pi;
          x[1] = h10 * (h00 + h11 - sigma);
          x[2] = h10 * h21;
        } else {
          for (int k = 0; k < mm; ++k) x[k] = A_(p + 1 + k, p);
        }
        oracle_house(mm, x, v, &tau, &beta);
        refl_left(A, lda, p + 1, mm, (p == l - 1) ? l : p + 1, m, v, tau);   /* wantt: all columns */
        if (p >= l) {
          A_(p + 1, p) = beta;
          for (int k = 1; k < mm; ++k) A_(p + 1 + k, p) = 0.0;
        }
        refl_right(A, lda, 0, ((p + mm + 1 < i) ? p + mm + 1 : i) + 1, p + 1, mm, v, tau);  /* rows 0.. */
        refl_right(U, ldu, 0, m, p + 1, mm, v, tau);
      }
    }
    if (l == i) {
      wr[i] = A_(i, i);
      wi[i] = 0.0;
      i -= 1;
    } else {
      eig2(A_(i - 1, i - 1), A_(i - 1, i), A_(i, i - 1), A_(i, i), &wr[i - 1], &wi[i - 1], &wr[i], &wi[i]);
      i -= 2;
    }
  }
#undef A_
  return 0;
}

/* AED on the window [k0, k0+nw) of H (n x n, column-major) inside the unreduced block [ilo, ihi]
 * (k0 + nw - 1 == ihi).  thr: the deflation threshold (u ||H||_F).  Writes the eigenvalues of the
 * deflated blocks to wr / wi at their rows and the window's undeflated eigenvalues (the shifts, top
 * to bottom) to swr / swi (nw entries; count returned through *nund).  Returns the number of
 * deflated eigenvalues nd (the rows k0+nw-nd .. ihi are then decoupled: H[ihi-nd+1, ihi-nd] = 0).
 * H and Z change only when nd > 0. */
int oracle_aed(double* H, double* Z, int64_t n, int64_t ilo, int64_t k0, int nw, double thr, double* wr,
               double* wi, double* swr, double* swi, int* nund) {
  double* T = (double*)malloc(sizeof(double) * (size_t)nw * nw * 2 + sizeof(double) * (size_t)(4 * nw + 8));
  double* U = T + (size_t)nw * nw;
  double* v = U + (size_t)nw * nw;
  double* ew = v + nw;
  double* ei = ew + nw;
  double* w = ei + nw;
  for (int c = 0; c < nw; ++c)
    for (int r = 0; r < nw; ++r) {
      T[r + c * nw] = EL(H, k0 + r, k0 + c, n);
      U[r + c * nw] = (r == c) ? 1.0 : 0.0;
    }
  oracle_schur(T, nw, nw, U, nw, ew, ei);
  const double s = (k0 > ilo) ? EL(H, k0, k0 - 1, n) : 0.0;
  for (int j = 0; j < nw; ++j) v[j] = s * U[0 + j * nw];
  /* deflation from the bottom (norm-stable condition, R22) with the failed blocks reordered to the
   * top (R23): [0, ntop) the failed blocks, [ntop, m) not yet evaluated, [m, nw) deflated */
  int m = nw, ntop = 0;
  while (m > ntop) {
    const int bs = (m - 2 >= ntop && T[(m - 1) + (m - 2) * nw] != 0.0) ? 2 : 1;
    int ok = 1;
    for (int j = m - bs; j < m; ++j) ok &= fabs(s * U[0 + j * nw]) <= thr;
    if (ok) {
      m -= bs;
      continue;
    }
    int cur = m - bs, moved = 1;
    while (cur > ntop) { /* move the failed block up past each block above it */
      const int p = (cur - 2 >= ntop && T[(cur - 1) + (cur - 2) * nw] != 0.0) ? 2 : 1;
      if (oracle_swap(T, nw, nw, U, nw, cur - p, p, bs) != 0) {
        moved = 0;
        break;
      }
      cur -= p;
    }
    if (!moved) break; /* a rejected swap halts the reordering */
    ntop += bs;
  }
  /* the eigenvalues of the final blocks (the reordered T), the spike of the undeflated part */
  for (int j = 0; j < nw;) {
    if (j + 1 < nw && T[(j + 1) + j * nw] != 0.0) {
      eig2(T[j + j * nw], T[j + (j + 1) * nw], T[(j + 1) + j * nw], T[(j + 1) + (j + 1) * nw], &ew[j], &ei[j],
           &ew[j + 1], &ei[j + 1]);
      j += 2;
    } else {
      ew[j] = T[j + j * nw];
      ei[j] = 0.0;
      j += 1;
    }
  }
  for (int j = 0; j < nw; ++j) v[j] = (j < m) ? s * U[0 + j * nw] : 0.0;
  for (int j = m; j < nw; ++j) {
    wr[k0 + j] = ew[j];
    wi[k0 + j] = ei[j];
  }
  const int nd = nw - m;
  *nund = m;
  for (int j = 0; j < m; ++j) {
    swr[j] = ew[j];
    swi[j] = ei[j];
  }
  if (nd > 0) {
    double beta = 0.0;
    if (m > 1 && s != 0.0) { /* reflect the remaining spike onto e1 */
      double tau;
      for (int j = 0; j < m; ++j) w[j] = v[j];
      house_n(m, w, &tau, &beta);
      refl_left(T, nw, 0, m, 0, nw, w, tau);
      refl_right(T, nw, 0, m, 0, m, w, tau);
      refl_right(U, nw, 0, nw, 0, m, w, tau);
      /* Hessenberg form of T(0:m, 0:m) */
      for (int j = 0; j + 2 < m; ++j) {
        const int len = m - j - 1;
        for (int k = 0; k < len; ++k) w[k] = T[(j + 1 + k) + j * nw];
        double tj, bj;
        house_n(len, w, &tj, &bj);
        refl_left(T, nw, j + 1, len, j + 1, nw, w, tj);
        T[(j + 1) + j * nw] = bj;
        for (int k = 1; k < len; ++k) T[(j + 1 + k) + j * nw] = 0.0;
        refl_right(T, nw, 0, m, j + 1, len, w, tj);
        refl_right(U, nw, 0, nw, j + 1, len, w, tj);
      }
    } else {
      beta = v[0];
    }
    /* write back: the window, the spike column, then U into the rest of H and into Z */
    for (int c = 0; c < nw; ++c)
      for (int r = 0; r < nw; ++r) EL(H, k0 + r, k0 + c, n) = T[r + c * nw];
    if (k0 > ilo) {
      EL(H, k0, k0 - 1, n) = beta;
      for (int r = 1; r < nw; ++r) EL(H, k0 + r, k0 - 1, n) = 0.0;
    }
    /* H(window, k0+nw : n) <- U^T H(window, ...) */
    double* tmp = (double*)malloc(sizeof(double) * (size_t)nw);
    for (int64_t c = k0 + nw; c < n; ++c) {
      for (int i = 0; i < nw; ++i) {
        double a = 0.0;
        for (int k = 0; k < nw; ++k) a += U[k + i * nw] * EL(H, k0 + k, c, n);
        tmp[i] = a;
      }
      for (int i = 0; i < nw; ++i) EL(H, k0 + i, c, n) = tmp[i];
    }
    /* H(0:k0, window) <- H(0:k0, window) U ; Z(:, window) <- Z(:, window) U */
    for (int pass = 0; pass < 2; ++pass) {
      double* M = pass == 0 ? H : Z;
      const int64_t rows = pass == 0 ? k0 : n;
      if (!M) continue;
      for (int64_t r = 0; r < rows; ++r) {
        for (int j = 0; j < nw; ++j) {
          double a = 0.0;
          for (int k = 0; k < nw; ++k) a += EL(M, r, k0 + k, n) * U[k + j * nw];
          tmp[j] = a;
        }
        for (int j = 0; j < nw; ++j) EL(M, r, k0 + j, n) = tmp[j];
      }
    }
    free(tmp);
  }
  free(T);
  return nd;
}

/* The QR iteration with AED (R22): per round on the bottom unreduced block [l, hi] (N rows):
 * N <= nmin -> oracle_small_eig; else AED on the trailing min(nw, N) window; if it deflated more than
 * 14% of the window (LAPACK's nibble rule) the next round starts at once, else the block is swept with
 * the bottom-most (up to nshifts) undeflated candidates as shifts, followed by the small-subdiagonal
 * deflation (R16).  thr = 2^-53 ||H||_F (u = the unit roundoff, R10).  Returns 0, or -(sweeps) when
 * max_sweeps was reached; *naed_out = AED steps, *ndefl_out = eigenvalues deflated by AED. */
int oracle_qr_iterate_aed(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, int nshifts, int nw,
                          int64_t nmin, int max_sweeps, double* wr, double* wi, int* sweeps_out, int* naed_out,
                          int* ndefl_out) {
  double fro = 0.0;
  for (size_t k = 0; k < (size_t)n * (size_t)n; ++k) fro += H[k] * H[k];
  const double thr = 0x1p-53 * sqrt(fro);
  int sweeps = 0, naed = 0, ndefl = 0;
  int64_t hi = ihi;
  double* B = (double*)malloc(sizeof(double) * (size_t)(nmin * nmin + 4 * nw + 4 * nshifts + 8));
  double* swr = B + (size_t)nmin * nmin;
  double* swi = swr + nw;
  double* sr = swi + nw;
  double* si = sr + nshifts;
  int rc = 0;
  while (hi >= ilo) {
    int64_t l = hi;
    while (l > ilo && EL(H, l, l - 1, n) != 0.0) --l;
    const int64_t N = hi - l + 1;
    if (N <= nmin) {
      small_block_schur(H, Z, n, l, hi, B, wr, wi);
      hi = l - 1;
      continue;
    }
    if (sweeps >= max_sweeps) {
      rc = -sweeps;
      break;
    }
    const int nwin = (int)((N < nw) ? N : nw);
    int nund = 0;
    const int nd = oracle_aed(H, Z, n, l, hi - nwin + 1, nwin, thr, wr, wi, swr, swi, &nund);
    ++naed;
    ndefl += nd;
    if (nd > 0) {
      hi -= nd;
      if (100 * nd > 14 * nwin) continue;
      if (hi - l + 1 <= nmin) continue;
    }
    /* shifts: the bottom-most undeflated candidates, paired (make_shifts) */
    const int ns_avail = nund;
    const int want = (nshifts < ns_avail) ? nshifts : ns_avail;
    int k = make_shifts(swr + (ns_avail - want), swi + (ns_avail - want), want, want, sr, si);
    if (k > hi - l + 1) k = (int)((hi - l + 1) & ~(int64_t)1);
    if (k < 2) { /* no usable candidates: the eigenvalues of the trailing block (R21) */
      const int64_t Nb = hi - l + 1;
      int ns = (int)((nshifts < ((Nb - 2) & ~(int64_t)1)) ? nshifts : ((Nb - 2) & ~(int64_t)1));
      if (ns < 2) ns = 2;
      double* Bt = (double*)malloc(sizeof(double) * (size_t)(ns * ns + 2 * ns));
      for (int c = 0; c < ns; ++c)
        for (int r = 0; r < ns; ++r) Bt[r + c * ns] = EL(H, hi - ns + 1 + r, hi - ns + 1 + c, n);
      oracle_small_eig(Bt, ns, ns, Bt + ns * ns, Bt + ns * ns + ns);
      k = make_shifts(Bt + ns * ns, Bt + ns * ns + ns, ns, ns, sr, si);
      free(Bt);
      if (k < 2) {
        rc = -sweeps;
        break;
      }
    }
    oracle_sweep(H, Z, n, l, hi, sr, si, k, 0, 0, k / 2);
    ++sweeps;
    for (int64_t r = l + 1; r <= hi; ++r) {
      const double sd = fabs(EL(H, r - 1, r - 1, n)) + fabs(EL(H, r, r, n));
      if (fabs(EL(H, r, r - 1, n)) <= 0x1p-52 * sd) EL(H, r, r - 1, n) = 0.0;
    }
  }
  free(B);
  *sweeps_out = sweeps;
  *naed_out = naed;
  *ndefl_out = ndefl;
  return rc;
}
