// qriter.cu -- the QR iteration around the sweep (readings R21, R22):
// aggressive early deflation on the trailing window of a block (Schur form of the window
// with its factor U, spike, the norm-stable deflation condition of P:1142-1189, Hessenberg
// re-reduction -- one CTA; U then goes through the DMMA update kernels), the eigenvalues of a small
// Hessenberg block (shifts when AED has none, and the small blocks left at the end -- the role of the
// paper's small Schur task: a Francis double-shift QR iteration in one CTA), the deflation
// step that sets negligible subdiagonal entries to zero after a sweep (criterion R16), and
// ||H||_F for the deflation threshold.
#include <cuda_runtime.h>

#include <algorithm>

#include "device_common.cuh"
#include "kernels.hpp"

namespace hqr {

namespace {

constexpr int kSmallMax = 128;  // largest block the SMEM-resident solver takes

__device__ __forceinline__ void eig2_dev(double a, double b, double c, double d, double* wr1, double* wi1,
                                         double* wr2, double* wi2) {
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

// Eigenvalues of the m x m upper-Hessenberg block H(r0 : r0+m, r0 : r0+m) (global, column-major,
// ld n), m <= kSmallMax: one warp, the block in SMEM (odd leading dimension).  Francis double-shift
// QR with deflation on the active part [l, i] (eigenvalues only), exceptional shifts after 10 and
// 20 iterations, 2x2 blocks by eig2 (the oracle's algorithm and formulas, oracle_small_eig).
__global__ void __launch_bounds__(32, 1) small_eig_kernel(const double* __restrict__ H, int64_t n, int64_t r0,
                                                          int m, double* wr, double* wi, int* info) {
  extern __shared__ double A[];
  const int ld = m | 1;
  const int lane = threadIdx.x;
  for (int c = 0; c < m; ++c)
    for (int r = lane; r < m; r += 32) A[r + c * ld] = H[(r0 + r) + (r0 + c) * n];
  __syncwarp();
#define A_(r, c) A[(r) + (c) * ld]
  int i = m - 1, total = 0;
  while (i >= 0) {
    int its = 0, l = 0;
    for (;;) {
      for (l = i; l > 0; --l) {
        const double s = fabs(A_(l - 1, l - 1)) + fabs(A_(l, l));
        if (fabs(A_(l, l - 1)) <= 0x1p-52 * s) break;
      }
      __syncwarp();
      if (l > 0 && lane == 0) A_(l, l - 1) = 0.0;
      __syncwarp();
      if (l >= i - 1) break;
      if (++total > 30 * m) {
        if (lane == 0) *info = i + 1;
        return;
      }
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
      for (int p = l - 1; p <= i - 2; ++p) {
        const int mm = (p <= i - 3) ? 3 : 2;
        double x0, x1, x2;
        if (p == l - 1) {
          const double h00 = A_(l, l), h01 = A_(l, l + 1), h10 = A_(l + 1, l), h11 = A_(l + 1, l + 1);
          const double h21 = A_(l + 2, l + 1);
          x0 = h00 * (h00 - sigma) + h01 * h10 + pi;
          x1 = h10 * (h00 + h11 - sigma);
          x2 = h10 * h21;
        } else {
          x0 = A_(p + 1, p);
          x1 = A_(p + 2, p);
          x2 = (mm == 3) ? A_(p + 3, p) : 0.0;
        }
        double v1, v2, tau, beta;
        house(x0, x1, x2, v1, v2, tau, beta);
        __syncwarp();
        if (p >= l && lane < mm) A_(p + 1 + lane, p) = (lane == 0) ? beta : 0.0;
        if (tau != 0.0) {
          left_apply(&A_(p + 1, 0), ld, (p == l - 1) ? l : p + 1, i + 1, mm, v1, v2, tau, lane);
          __syncwarp();
          Refl rf;
          rf.v1 = v1; rf.v2 = v2; rf.tau = tau; rf.pl = p; rf.m = mm;
          const int r1 = min(p + mm + 1, i);
          right_apply(&A_(l, p + 1), ld, r1 - l + 1, rf, lane);
        }
        __syncwarp();
      }
    }
    if (lane == 0) {
      if (l == i) {
        wr[i] = A_(i, i);
        wi[i] = 0.0;
      } else {
        eig2_dev(A_(i - 1, i - 1), A_(i - 1, i), A_(i, i - 1), A_(i, i), &wr[i - 1], &wi[i - 1], &wr[i], &wi[i]);
      }
    }
    i -= (l == i) ? 1 : 2;
    __syncwarp();
  }
#undef A_
  if (lane == 0) *info = 0;
}

// Deflation after a sweep: h(k, k-1) = 0 where |h(k,k-1)| <= 2^-52 (|h(k-1,k-1)| + |h(k,k)|),
// k in [lo+1, hi]; *count += the entries zeroed.
__global__ void deflate_kernel(double* H, int64_t n, int64_t lo, int64_t hi, int* count) {
  for (int64_t k = lo + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= hi;
       k += (int64_t)gridDim.x * blockDim.x) {
    double* sub = H + k + (k - 1) * n;
    const double s = fabs(H[(k - 1) + (k - 1) * n]) + fabs(H[k + k * n]);
    if (*sub != 0.0 && fabs(*sub) <= 0x1p-52 * s) {
      *sub = 0.0;
      atomicAdd(count, 1);
    }
  }
}

// Householder reflector (R2 convention) of length M <= 4 in one thread: x overwritten by v (v[0] = 1).
template <int M>
__device__ __forceinline__ void house_small(double (&x)[4], double& tau) {
  double t2 = 0.0;
#pragma unroll
  for (int r = 1; r < M; ++r) t2 = fma(x[r], x[r], t2);
  const double alpha = x[0];
  x[0] = 1.0;
  if (t2 == 0.0) {
    tau = 0.0;
#pragma unroll
    for (int r = 1; r < M; ++r) x[r] = 0.0;
    return;
  }
  const double nrm = sqrt(fma(alpha, alpha, t2));
  const double b = (alpha >= 0.0) ? -nrm : nrm;
  tau = (b - alpha) / b;
  const double d = 1.0 / (alpha - b);
#pragma unroll
  for (int r = 1; r < M; ++r) x[r] *= d;
}

// D <- P D P, P = I - tau w w^T acting on indices R0 .. R0+L-1 of the K x K register block D
template <int K, int R0, int L>
__device__ __forceinline__ void refl_both_small(double (&D)[K][K], const double (&w)[4], double tau) {
#pragma unroll
  for (int c = 0; c < K; ++c) {
    double a = 0.0;
#pragma unroll
    for (int r = 0; r < L; ++r) a = fma(w[r], D[R0 + r][c], a);
#pragma unroll
    for (int r = 0; r < L; ++r) D[R0 + r][c] = fma(-tau * a, w[r], D[R0 + r][c]);
  }
#pragma unroll
  for (int r = 0; r < K; ++r) {
    double a = 0.0;
#pragma unroll
    for (int c = 0; c < L; ++c) a = fma(D[r][R0 + c], w[c], a);
#pragma unroll
    for (int c = 0; c < L; ++c) D[r][R0 + c] = fma(-tau * a, w[c], D[r][R0 + c]);
  }
}

// The swap factor of the adjacent diagonal blocks A = T(i:i+P) and B = T(i+P:i+P+Q) of the
// quasi-triangular T (reading R23; oracle_swap's algorithm), one thread, all in
// registers (sizes fixed at compile time, pivoting by predicated moves): X solves A X - X B = C as
// the PQ x PQ Kronecker system (complete pivoting, pivots below 2^-52 max|K| raised to it); Q = P1
// (P2) the Householder QR factor of [-X; I_Q]; the check on the transformed (P+Q)^2 block
// (lower-left <= 10 * 2^-52 max|D|).  Writes w1 (sw[0..3]), w2 (sw[4..7]), tau1, tau2 (sw[8], sw[9])
// and the verdict (sw[10] = 1 accepted, 0 rejected).
template <int P, int Q>
__device__ __noinline__ void swap_factor(const double* T, int ld, int i, double* sw) {
  constexpr int K = P + Q, NK = P * Q;
  double D[K][K];
  double dn = 0.0;
#pragma unroll
  for (int c = 0; c < K; ++c)
#pragma unroll
    for (int r = 0; r < K; ++r) {
      D[r][c] = T[(i + r) + (i + c) * ld];
      dn = fmax(dn, fabs(D[r][c]));
    }
  double A[NK][NK], x[NK];
#pragma unroll
  for (int r = 0; r < NK; ++r)
#pragma unroll
    for (int c = 0; c < NK; ++c) A[r][c] = 0.0;
#pragma unroll
  for (int c = 0; c < Q; ++c)
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const int row = r + c * P;
#pragma unroll
      for (int t = 0; t < P; ++t) A[row][t + c * P] += D[r][t];          // A(r,t) X(t,c)
#pragma unroll
      for (int t = 0; t < Q; ++t) A[row][r + t * P] -= D[P + t][P + c];  // X(r,t) B(t,c)
      x[row] = D[r][P + c];                                              // C(r,c)
    }
  double km = 0.0;
#pragma unroll
  for (int r = 0; r < NK; ++r)
#pragma unroll
    for (int c = 0; c < NK; ++c) km = fmax(km, fabs(A[r][c]));
  const double smin = (km > 0.0 ? km : 1.0) * 0x1p-52;
  int perm[NK];
  double rinv[NK];
#pragma unroll
  for (int j = 0; j < NK; ++j) perm[j] = j;
#pragma unroll
  for (int j = 0; j < NK; ++j) {
    int pr = j, pc = j;
    double best = fabs(A[j][j]);
#pragma unroll
    for (int c = j; c < NK; ++c)
#pragma unroll
      for (int r = j; r < NK; ++r)
        if (fabs(A[r][c]) > best) { best = fabs(A[r][c]); pr = r; pc = c; }
#pragma unroll
    for (int r = j + 1; r < NK; ++r)
      if (pr == r) {
#pragma unroll
        for (int c = 0; c < NK; ++c) { const double t = A[j][c]; A[j][c] = A[r][c]; A[r][c] = t; }
        const double t = x[j]; x[j] = x[r]; x[r] = t;
      }
#pragma unroll
    for (int c = j + 1; c < NK; ++c)
      if (pc == c) {
#pragma unroll
        for (int r = 0; r < NK; ++r) { const double t = A[r][j]; A[r][j] = A[r][c]; A[r][c] = t; }
        const int t = perm[j]; perm[j] = perm[c]; perm[c] = t;
      }
    if (fabs(A[j][j]) < smin) A[j][j] = smin;
    rinv[j] = 1.0 / A[j][j];
#pragma unroll
    for (int r = j + 1; r < NK; ++r) {
      const double f = A[r][j] * rinv[j];
#pragma unroll
      for (int c = j; c < NK; ++c) A[r][c] = fma(-f, A[j][c], A[r][c]);
      x[r] = fma(-f, x[j], x[r]);
    }
  }
  double y[NK], X[NK];
#pragma unroll
  for (int j = NK - 1; j >= 0; --j) {
    double a = x[j];
#pragma unroll
    for (int c = j + 1; c < NK; ++c) a = fma(-A[j][c], y[c], a);
    y[j] = a * rinv[j];
  }
#pragma unroll
  for (int t = 0; t < NK; ++t) {
    X[t] = 0.0;
#pragma unroll
    for (int j = 0; j < NK; ++j)
      if (perm[j] == t) X[t] = y[j];
  }
  // Householder QR of M = [-X; I_Q]
  double w1[4] = {0.0, 0.0, 0.0, 0.0}, w2[4] = {0.0, 0.0, 0.0, 0.0};
  double tau1, tau2 = 0.0;
#pragma unroll
  for (int r = 0; r < K; ++r) w1[r] = (r < P) ? -X[r] : ((r == P) ? 1.0 : 0.0);
  house_small<K>(w1, tau1);
  if constexpr (Q == 2) {
    double m2[4];
#pragma unroll
    for (int r = 0; r < K; ++r) m2[r] = (r < P) ? -X[r + P] : ((r == P + 1) ? 1.0 : 0.0);
    double a = 0.0;
#pragma unroll
    for (int r = 0; r < K; ++r) a = fma(w1[r], m2[r], a);
#pragma unroll
    for (int r = 0; r < K; ++r) m2[r] = fma(-tau1 * a, w1[r], m2[r]);
#pragma unroll
    for (int r = 0; r < K - 1; ++r) w2[r] = m2[1 + r];
    house_small<K - 1>(w2, tau2);
  }
  refl_both_small<K, 0, K>(D, w1, tau1);
  if constexpr (Q == 2) refl_both_small<K, 1, K - 1>(D, w2, tau2);
  double low = 0.0;
#pragma unroll
  for (int c = 0; c < Q; ++c)
#pragma unroll
    for (int r = Q; r < K; ++r) low = fmax(low, fabs(D[r][c]));
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    sw[r] = w1[r];
    sw[4 + r] = w2[r];
  }
  sw[8] = tau1;
  sw[9] = tau2;
  sw[10] = (low <= 10.0 * 0x1p-52 * dn) ? 1.0 : 0.0;
}

// ---- the AED kernel: one CTA of kAedThreads threads (all phases are latency-bound chains of small
// reflector applications; with 256 threads every application over the window's <= 112 rows or
// columns is one pass, and T and U updates of a step run side by side) -------------------------
#ifndef HQR_AED_THREADS
#define HQR_AED_THREADS 256
#endif
constexpr int kAedThreads = HQR_AED_THREADS;

// A(r0 .. r0+m-1, c) -= tau w (w^T A(.., c)) for the columns c handled by thread t (stride nthr)
__device__ __forceinline__ void refl_left_col(double* A, int lda, int r0, int m, int c, const double* w, double tau) {
  double* a = A + r0 + c * lda;
  double s = 0.0;
  for (int i = 0; i < m; ++i) s = fma(w[i], a[i], s);
  const double ts = tau * s;
  for (int i = 0; i < m; ++i) a[i] = fma(-ts, w[i], a[i]);
}
// A(r, c0 .. c0+m-1) -= tau (A(r, ..) w) w^T for one row r
__device__ __forceinline__ void refl_right_row(double* A, int lda, int r, int c0, int m, const double* w, double tau) {
  double* a = A + r + c0 * lda;
  double s = 0.0;
  for (int i = 0; i < m; ++i) s = fma(a[i * lda], w[i], s);
  const double ts = tau * s;
  for (int i = 0; i < m; ++i) a[i * lda] = fma(-ts, w[i], a[i * lda]);
}

// Householder reflector of general length m (R2 convention) on x in SMEM (overwritten by v, v[0] = 1),
// the whole CTA; red: 1 double of SMEM scratch.  Returns tau, beta in every thread.
__device__ __forceinline__ void house_n_cta(double* x, int m, double& tau, double& beta, double* red, int tid,
                                            int nthr) {
  if (tid < 32) {
    double t2 = 0.0;
    for (int i = 1 + tid; i < m; i += 32) t2 = fma(x[i], x[i], t2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t2 += __shfl_xor_sync(0xffffffffu, t2, o);
    if (tid == 0) *red = t2;
  }
  __syncthreads();
  const double t2 = *red, alpha = x[0];
  __syncthreads();  // every thread has read x[0] and *red
  if (t2 == 0.0) {
    tau = 0.0;
    beta = alpha;
    for (int i = tid; i < m; i += nthr) x[i] = (i == 0) ? 1.0 : 0.0;
    __syncthreads();
    return;
  }
  const double nrm = sqrt(fma(alpha, alpha, t2));
  const double b = (alpha >= 0.0) ? -nrm : nrm;
  tau = (b - alpha) / b;
  const double d = alpha - b;
  for (int i = tid; i < m; i += nthr) x[i] = (i == 0) ? 1.0 : x[i] / d;
  beta = b;
  __syncthreads();
}

// x(0 .. L-1) (stride st) -= tau w (w^T x): one reflector of compile-time length L on a row / column
template <int L>
__device__ __forceinline__ void refl_vec(double* x, int st, const double (&w)[4], double tau) {
  double h[L];
#pragma unroll
  for (int r = 0; r < L; ++r) h[r] = x[r * st];
  double a = 0.0;
#pragma unroll
  for (int r = 0; r < L; ++r) a = fma(w[r], h[r], a);
  const double ta = tau * a;
#pragma unroll
  for (int r = 0; r < L; ++r) x[r * st] = fma(-ta, w[r], h[r]);
}

// Swap of the adjacent diagonal blocks A = T(i:i+P) and B = T(i+P:i+P+Q) of the quasi-triangular T in
// SMEM, U <- U Q (reading R23): thread 0 forms the factor (swap_factor); when it is accepted the CTA
// applies Q = P1 (P2) -- T's rows i..i+P+Q-1 (columns from i) and U's rows side by side, then T's
// columns -- and zeros the new lower-left block.  sw: 16 doubles of SMEM scratch.  Returns whether
// the swap was done (uniform).
template <int P, int Q>
__device__ bool swap_blocks_t(double* T, double* U, int ld, int nw, int i, double* sw, int tid, int nthr) {
  constexpr int K = P + Q;
  if (tid == 0) swap_factor<P, Q>(T, ld, i, sw);
  __syncthreads();
  if (sw[10] == 0.0) return false;
  double w1[4], w2[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    w1[r] = sw[r];
    w2[r] = sw[4 + r];
  }
  const double tau1 = sw[8], tau2 = sw[9];
  const int ncols = nw - i;
  for (int it = tid; it < ncols + nw; it += nthr) {
    if (it < ncols) {  // T(i.., c) from the left
      double* x = T + i + (i + it) * ld;
      refl_vec<K>(x, 1, w1, tau1);
      if constexpr (Q == 2) refl_vec<K - 1>(x + 1, 1, w2, tau2);
    } else {           // U(r, i..) from the right
      double* x = U + (it - ncols) + i * ld;
      refl_vec<K>(x, ld, w1, tau1);
      if constexpr (Q == 2) refl_vec<K - 1>(x + ld, ld, w2, tau2);
    }
  }
  __syncthreads();
  for (int r = tid; r < i + K; r += nthr) {  // T(r, i..) from the right
    double* x = T + r + i * ld;
    refl_vec<K>(x, ld, w1, tau1);
    if constexpr (Q == 2) refl_vec<K - 1>(x + ld, ld, w2, tau2);
  }
  __syncthreads();
  if (tid < P * Q) T[(i + Q + tid % P) + (i + tid / P) * ld] = 0.0;
  __syncthreads();
  return true;
}

__device__ bool swap_blocks(double* T, double* U, int ld, int nw, int i, int p, int q, double* sw, int tid,
                            int nthr) {
  if (p == 1 && q == 1) return swap_blocks_t<1, 1>(T, U, ld, nw, i, sw, tid, nthr);
  if (p == 1) return swap_blocks_t<1, 2>(T, U, ld, nw, i, sw, tid, nthr);
  if (q == 1) return swap_blocks_t<2, 1>(T, U, ld, nw, i, sw, tid, nthr);
  return swap_blocks_t<2, 2>(T, U, ld, nw, i, sw, tid, nthr);
}

// Aggressive early deflation (reading R22, R23; oracle_aed's algorithm): one CTA, window W = H(k0:k0+nw,
// k0:k0+nw) and its factor U in SMEM.  Real Schur form with U accumulated (Francis double-shift QR,
// every reflector on all window columns / rows), spike v = s U(0,:), deflation from the bottom
// (|v| <= thr on the block's rows; a failed block is moved above the blocks not yet evaluated by
// swap_blocks, a rejected swap halts the reordering: P:289-290), then -- when anything
// deflated -- the remaining spike reflected onto e1 and T(0:m,0:m) returned to Hessenberg form (U
// accumulated), T and the spike column written into H, U stored as a Q slot (KP x QLD, band metadata)
// for the update kernels.  res[0] = nd, res[1] = m (undeflated); ew / ei: the eigenvalues of the
// final blocks in window order.
__global__ void __launch_bounds__(kAedThreads, 1) aed_kernel(double* H, int64_t n, int64_t ilo, int64_t k0, int nw,
                                                            double thr, double* uslot, int KP, int QLD, double* ew,
                                                            double* ei, int* res) {
  extern __shared__ double sm[];
  const int ld = nw | 1;
  double* T = sm;
  double* U = T + nw * ld;
  double* v = U + nw * ld;   // spike / reflector work space (nw + 2)
  double* sw = v + nw + 2;   // swap factor / reduction scratch (16)
  const int tid = threadIdx.x, nthr = blockDim.x;
#ifdef HQR_AED_TIMING
  const long long tc0 = clock64();
  int nswaps = 0;
#endif
  for (int idx = tid; idx < nw * nw; idx += nthr) {
    const int r = idx % nw, c = idx / nw;
    T[r + c * ld] = H[(k0 + r) + (k0 + c) * n];
    U[r + c * ld] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
#define T_(r, c) T[(r) + (c) * ld]
  // ---- (1) real Schur form T = U^T W U --------------------------------------------------------
  int i = nw - 1, total = 0;
  while (i >= 0) {
    int its = 0, l = 0;
    for (;;) {
      for (l = i; l > 0; --l) {
        const double sd = fabs(T_(l - 1, l - 1)) + fabs(T_(l, l));
        if (fabs(T_(l, l - 1)) <= 0x1p-52 * sd) break;
      }
      __syncthreads();
      if (l > 0 && tid == 0) T_(l, l - 1) = 0.0;
      __syncthreads();
      if (l >= i - 1) break;
      if (++total > 30 * nw) {
        if (tid == 0) { res[0] = -1; res[1] = nw; }
        return;
      }
      ++its;
      double sigma, pi;
      if (its == 10 || its == 20) {
        const double sd = fabs(T_(i, i - 1)) + fabs(T_(i - 1, i - 2));
        const double h11 = 0.75 * sd + T_(i, i);
        sigma = 2.0 * h11;
        pi = h11 * h11 + 0.4375 * sd * sd;
      } else {
        const double a = T_(i - 1, i - 1), b = T_(i - 1, i), c = T_(i, i - 1), d = T_(i, i);
        sigma = a + d;
        pi = a * d - b * c;
      }
      for (int p = l - 1; p <= i - 2; ++p) {
        const int mm = (p <= i - 3) ? 3 : 2;
        double x0, x1, x2;
        if (p == l - 1) {
          const double h00 = T_(l, l), h01 = T_(l, l + 1), h10 = T_(l + 1, l), h11 = T_(l + 1, l + 1);
          const double h21 = T_(l + 2, l + 1);
          x0 = h00 * (h00 - sigma) + h01 * h10 + pi;
          x1 = h10 * (h00 + h11 - sigma);
          x2 = h10 * h21;
        } else {
          x0 = T_(p + 1, p);
          x1 = T_(p + 2, p);
          x2 = (mm == 3) ? T_(p + 3, p) : 0.0;
        }
        double v1, v2, tau, beta;
        house(x0, x1, x2, v1, v2, tau, beta);
        if (p == l - 1) __syncthreads();  // x0..x2 came from the columns the left application updates
        if (tau != 0.0) {
          // T(p+1.., c) from the left for c >= first (column p is overwritten by beta below) and
          // U(r, p+1..) from the right, side by side
          const int first = (p == l - 1) ? l : p + 1;
          const int ncols = nw - first;
          for (int it = tid; it < ncols + nw; it += nthr) {
            if (it < ncols) {
              double* hc = &T_(p + 1, first + it);
              const double h0 = hc[0], h1 = hc[1], h2 = (mm == 3) ? hc[2] : 0.0;
              const double tw = tau * fma(v2, h2, fma(v1, h1, h0));
              hc[0] = h0 - tw;
              hc[1] = fma(-tw, v1, h1);
              if (mm == 3) hc[2] = fma(-tw, v2, h2);
            } else {
              double* x = &U[(it - ncols) + (p + 1) * ld];
              const double h0 = x[0], h1 = x[ld], h2 = (mm == 3) ? x[2 * ld] : 0.0;
              const double tw = tau * fma(v2, h2, fma(v1, h1, h0));
              x[0] = h0 - tw;
              x[ld] = fma(-tw, v1, h1);
              if (mm == 3) x[2 * ld] = fma(-tw, v2, h2);
            }
          }
        }
        __syncthreads();  // left applications done; every thread has read x0..x2
        if (p >= l && tid < mm) T_(p + 1 + tid, p) = (tid == 0) ? beta : 0.0;
        if (tau != 0.0) {  // T(r, p+1..) from the right, rows 0 .. min(p+mm+1, i)
          const int rows = min(p + mm + 1, i) + 1;
          for (int r = tid; r < rows; r += nthr) {
            double* x = &T_(r, p + 1);
            const double h0 = x[0], h1 = x[ld], h2 = (mm == 3) ? x[2 * ld] : 0.0;
            const double tw = tau * fma(v2, h2, fma(v1, h1, h0));
            x[0] = h0 - tw;
            x[ld] = fma(-tw, v1, h1);
            if (mm == 3) x[2 * ld] = fma(-tw, v2, h2);
          }
        }
        __syncthreads();
      }
    }
    if (tid == 0) {
      if (l == i) {
        ew[i] = T_(i, i);
        ei[i] = 0.0;
      } else {
        eig2_dev(T_(i - 1, i - 1), T_(i - 1, i), T_(i, i - 1), T_(i, i), &ew[i - 1], &ei[i - 1], &ew[i], &ei[i]);
      }
    }
    i -= (l == i) ? 1 : 2;
    __syncthreads();
  }
  // ---- (2) spike, deflation from the bottom, failed blocks reordered to the top (R22, R23) ------
  // [0, ntop) the failed blocks, [ntop, m) not yet evaluated, [m, nw) deflated; uniform across threads
  const double s = (k0 > ilo) ? H[k0 + (k0 - 1) * n] : 0.0;
#ifdef HQR_AED_TIMING
  const long long tc1 = clock64();
#endif
  int m = nw, ntop = 0;
  while (m > ntop) {
    const int bs = (m - 2 >= ntop && T_(m - 1, m - 2) != 0.0) ? 2 : 1;
    bool ok = true;
    for (int j = m - bs; j < m; ++j) ok &= fabs(s * U[0 + j * ld]) <= thr;
    if (ok) {
      m -= bs;
      continue;
    }
#ifdef HQR_EXP_NOREORDER
    break;
#endif
    int cur = m - bs;
    bool moved = true;
    while (cur > ntop) {  // past each block above it
      const int p = (cur - 2 >= ntop && T_(cur - 1, cur - 2) != 0.0) ? 2 : 1;
      if (!swap_blocks(T, U, ld, nw, cur - p, p, bs, sw, tid, nthr)) {
        moved = false;
        break;
      }
#ifdef HQR_AED_TIMING
      ++nswaps;
#endif
      cur -= p;
    }
    if (!moved) break;  // a rejected swap halts the reordering
    ntop += bs;
  }
  // the eigenvalues of the final blocks, the spike of the undeflated part
  if (tid == 0) {
    for (int j = 0; j < nw;) {
      if (j + 1 < nw && T_(j + 1, j) != 0.0) {
        eig2_dev(T_(j, j), T_(j, j + 1), T_(j + 1, j), T_(j + 1, j + 1), &ew[j], &ei[j], &ew[j + 1], &ei[j + 1]);
        j += 2;
      } else {
        ew[j] = T_(j, j);
        ei[j] = 0.0;
        j += 1;
      }
    }
  }
  for (int j = tid; j < nw; j += nthr) v[j] = (j < m) ? s * U[0 + j * ld] : 0.0;
  __syncthreads();
  const int nd = nw - m;
#ifdef HQR_AED_TIMING
  const long long tc2 = clock64();
  if (tid == 0)
    printf("AEDT nw %d nd %d m %d ntop %d swaps %d schur %lld reorder %lld\n", nw, nd, m, ntop, nswaps, tc1 - tc0,
           tc2 - tc1);
#endif
  if (tid == 0) { res[0] = nd; res[1] = m; }
  if (nd == 0) return;  // H unchanged (the window is copied back only when something deflated)
  // ---- (3) reflect the spike onto e1, Hessenberg form of T(0:m, 0:m) ----------------------------
  double beta = v[0];
  double* w = v;  // work vector
  if (m > 1 && s != 0.0) {
    double tau;
    house_n_cta(w, m, tau, beta, sw + 12, tid, nthr);
    for (int c = tid; c < nw; c += nthr) refl_left_col(T, ld, 0, m, c, w, tau);
    __syncthreads();
    for (int it = tid; it < m + nw; it += nthr) {
      if (it < m) refl_right_row(T, ld, it, 0, m, w, tau);
      else refl_right_row(U, ld, it - m, 0, m, w, tau);
    }
    __syncthreads();
    for (int j = 0; j + 2 < m; ++j) {
      const int len = m - j - 1;
      for (int k = tid; k < len; k += nthr) w[k] = T_(j + 1 + k, j);
      __syncthreads();
      double tj, bj;
      house_n_cta(w, len, tj, bj, sw + 12, tid, nthr);
      for (int c = j + 1 + tid; c < nw; c += nthr) refl_left_col(T, ld, j + 1, len, c, w, tj);
      for (int k = tid; k < len; k += nthr) T_(j + 1 + k, j) = (k == 0) ? bj : 0.0;
      __syncthreads();
      for (int it = tid; it < m + nw; it += nthr) {
        if (it < m) refl_right_row(T, ld, it, j + 1, len, w, tj);
        else refl_right_row(U, ld, it - m, j + 1, len, w, tj);
      }
      __syncthreads();
    }
  }
  // ---- (4) write back: the window, the spike column; U as a Q slot -------------------------------
  for (int idx = tid; idx < nw * nw; idx += nthr) {
    const int r = idx % nw, c = idx / nw;
    H[(k0 + r) + (k0 + c) * n] = T_(r, c);
  }
  if (k0 > ilo)
    for (int r = tid; r < nw; r += nthr) H[(k0 + r) + (k0 - 1) * n] = (r == 0) ? beta : 0.0;
  store_q_slot(uslot, U, ld, nw, KP, QLD, tid / 32, nthr / 32, tid % 32);
#undef T_
}

}  // namespace

// sum of squares of n*n entries (||H||_F^2 for the AED deflation threshold), one atomic per block
__global__ void fro2_kernel(const double* __restrict__ H, int64_t count, double* out) {
  double acc = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x)
    acc = fma(H[k], H[k], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double a = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (threadIdx.x == 0) atomicAdd(out, a);
  }
}

int small_eig_max() { return kSmallMax; }

cudaError_t launch_fro2(const double* H, int64_t count, double* out, int num_sms, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  fro2_kernel<<<4 * num_sms, 256, 0, st>>>(H, count, out);
  return cudaGetLastError();
}

size_t aed_smem_bytes(int nw) { return ((size_t)2 * nw * (nw | 1) + nw + 2 + 16 + 14) * sizeof(double); }

cudaError_t launch_aed(double* H, int64_t n, int64_t ilo, int64_t k0, int nw, double thr, double* uslot, int KP,
                       int QLD, double* ew, double* ei, int* res, cudaStream_t st) {
  if (nw < 1 || nw > kMaxWindow) return cudaErrorInvalidValue;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(aed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)aed_smem_bytes(kMaxWindow));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  aed_kernel<<<1, kAedThreads, aed_smem_bytes(nw), st>>>(H, n, ilo, k0, nw, thr, uslot, KP, QLD, ew, ei, res);
  return cudaGetLastError();
}

cudaError_t launch_small_eig(const double* H, int64_t n, int64_t r0, int m, double* wr, double* wi, int* info,
                             cudaStream_t st) {
  if (m < 1 || m > kSmallMax) return cudaErrorInvalidValue;
  const size_t smem = (size_t)m * (m | 1) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(small_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)((size_t)kSmallMax * (kSmallMax | 1) * sizeof(double)));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  small_eig_kernel<<<1, 32, smem, st>>>(H, n, r0, m, wr, wi, info);
  return cudaGetLastError();
}

cudaError_t launch_deflate(double* H, int64_t n, int64_t lo, int64_t hi, int* count, cudaStream_t st) {
  if (hi <= lo) return cudaSuccess;
  const int64_t cnt = hi - lo;
  const int grid = (int)std::min<int64_t>((cnt + 255) / 256, 148);
  deflate_kernel<<<grid, 256, 0, st>>>(H, n, lo, hi, count);
  return cudaGetLastError();
}

}  // namespace hqr
