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

// Householder reflector of general length m (R2 convention) on x held in SMEM (overwritten by v,
// v[0] = 1); one warp; returns tau, beta in every lane.
__device__ __forceinline__ void house_n_warp(double* x, int m, double& tau, double& beta, int lane) {
  double t2 = 0.0;
  for (int i = 1 + lane; i < m; i += 32) t2 = fma(x[i], x[i], t2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t2 += __shfl_xor_sync(0xffffffffu, t2, o);
  const double alpha = x[0];
  __syncwarp();
  if (t2 == 0.0) {
    tau = 0.0;
    beta = alpha;
    for (int i = lane; i < m; i += 32) x[i] = (i == 0) ? 1.0 : 0.0;
    __syncwarp();
    return;
  }
  const double nrm = sqrt(fma(alpha, alpha, t2));
  const double b = (alpha >= 0.0) ? -nrm : nrm;
  tau = (b - alpha) / b;
  const double d = alpha - b;
  for (int i = lane; i < m; i += 32) x[i] = (i == 0) ? 1.0 : x[i] / d;
  beta = b;
  __syncwarp();
}

// A(r0 .. r0+m-1, c0 .. c1-1) -= tau w (w^T A) (column-major, ld lda); lanes across columns
__device__ __forceinline__ void refl_left_warp(double* A, int lda, int r0, int m, int c0, int c1, const double* w,
                                               double tau, int lane) {
  for (int c = c0 + lane; c < c1; c += 32) {
    double* a = A + r0 + c * lda;
    double s = 0.0;
    for (int i = 0; i < m; ++i) s = fma(w[i], a[i], s);
    const double ts = tau * s;
    for (int i = 0; i < m; ++i) a[i] = fma(-ts, w[i], a[i]);
  }
}
// A(r0 .. r1-1, c0 .. c0+m-1) -= tau (A w) w^T; lanes across rows
__device__ __forceinline__ void refl_right_warp(double* A, int lda, int r0, int r1, int c0, int m, const double* w,
                                                double tau, int lane) {
  for (int r = r0 + lane; r < r1; r += 32) {
    double* a = A + r + c0 * lda;
    double s = 0.0;
    for (int i = 0; i < m; ++i) s = fma(a[i * lda], w[i], s);
    const double ts = tau * s;
    for (int i = 0; i < m; ++i) a[i * lda] = fma(-ts, w[i], a[i * lda]);
  }
}

// Aggressive early deflation (reading R22; oracle_aed's algorithm): one warp, window W = H(k0:k0+nw,
// k0:k0+nw) and its factor U in SMEM.  Real Schur form with U accumulated (Francis double-shift QR,
// every reflector on all window columns / rows), spike v = s U(0,:), deflation from the bottom
// (|v| <= thr on the block's rows; the first failure stops it), then -- when anything deflated --
// the remaining spike reflected onto e1 and T(0:m,0:m) returned to Hessenberg form (U accumulated),
// T and the spike column written into H, U stored as a Q slot (KP x QLD, band metadata) for the
// update kernels.  res[0] = nd, res[1] = m (undeflated), eigenvalues: ew / ei (nw, window order).
__global__ void __launch_bounds__(32, 1) aed_kernel(double* H, int64_t n, int64_t ilo, int64_t k0, int nw,
                                                    double thr, double* uslot, int KP, int QLD, double* ew, double* ei,
                                                    int* res) {
  extern __shared__ double sm[];
  const int ld = nw | 1;
  double* T = sm;
  double* U = T + nw * ld;
  double* v = U + nw * ld;   // spike / reflector work space (nw + 2)
  const int lane = threadIdx.x;
  for (int c = 0; c < nw; ++c)
    for (int r = lane; r < nw; r += 32) {
      T[r + c * ld] = H[(k0 + r) + (k0 + c) * n];
      U[r + c * ld] = (r == c) ? 1.0 : 0.0;
    }
  __syncwarp();
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
      __syncwarp();
      if (l > 0 && lane == 0) T_(l, l - 1) = 0.0;
      __syncwarp();
      if (l >= i - 1) break;
      if (++total > 30 * nw) {
        if (lane == 0) { res[0] = -1; res[1] = nw; }
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
        __syncwarp();
        if (p >= l && lane < mm) T_(p + 1 + lane, p) = (lane == 0) ? beta : 0.0;
        if (tau != 0.0) {
          left_apply(&T_(p + 1, 0), ld, (p == l - 1) ? l : p + 1, nw, mm, v1, v2, tau, lane);  // all columns
          __syncwarp();
          Refl rf;
          rf.v1 = v1; rf.v2 = v2; rf.tau = tau; rf.pl = p; rf.m = mm;
          right_apply(&T_(0, p + 1), ld, min(p + mm + 1, i) + 1, rf, lane);  // rows 0 ..
          right_apply(&U[(p + 1) * ld], ld, nw, rf, lane);
        }
        __syncwarp();
      }
    }
    if (lane == 0) {
      if (l == i) {
        ew[i] = T_(i, i);
        ei[i] = 0.0;
      } else {
        eig2_dev(T_(i - 1, i - 1), T_(i - 1, i), T_(i, i - 1), T_(i, i), &ew[i - 1], &ei[i - 1], &ew[i], &ei[i]);
      }
    }
    i -= (l == i) ? 1 : 2;
    __syncwarp();
  }
  // ---- (2) spike and deflation from the bottom ------------------------------------------------
  const double s = (k0 > ilo) ? H[k0 + (k0 - 1) * n] : 0.0;
  for (int j = lane; j < nw; j += 32) v[j] = s * U[0 + j * ld];
  __syncwarp();
  int m = nw;
  for (;;) {  // uniform across lanes
    if (m == 0) break;
    const int bs = (m >= 2 && T_(m - 1, m - 2) != 0.0) ? 2 : 1;
    bool ok = true;
    for (int j = m - bs; j < m; ++j) ok &= fabs(v[j]) <= thr;
    if (!ok) break;
    __syncwarp();
    if (lane < bs) v[m - bs + lane] = 0.0;
    __syncwarp();
    m -= bs;
  }
  const int nd = nw - m;
  if (lane == 0) { res[0] = nd; res[1] = m; }
  if (nd == 0) return;  // H unchanged (the window is copied back only when something deflated)
  // ---- (3) reflect the spike onto e1, Hessenberg form of T(0:m, 0:m) ----------------------------
  double beta = v[0];
  double* w = v;  // work vector
  if (m > 1 && s != 0.0) {
    double tau;
    house_n_warp(w, m, tau, beta, lane);
    refl_left_warp(T, ld, 0, m, 0, nw, w, tau, lane);
    __syncwarp();
    refl_right_warp(T, ld, 0, m, 0, m, w, tau, lane);
    refl_right_warp(U, ld, 0, nw, 0, m, w, tau, lane);
    __syncwarp();
    for (int j = 0; j + 2 < m; ++j) {
      const int len = m - j - 1;
      for (int k = lane; k < len; k += 32) w[k] = T_(j + 1 + k, j);
      __syncwarp();
      double tj, bj;
      house_n_warp(w, len, tj, bj, lane);
      refl_left_warp(T, ld, j + 1, len, j + 1, nw, w, tj, lane);
      __syncwarp();
      for (int k = lane; k < len; k += 32) T_(j + 1 + k, j) = (k == 0) ? bj : 0.0;
      __syncwarp();
      refl_right_warp(T, ld, 0, m, j + 1, len, w, tj, lane);
      refl_right_warp(U, ld, 0, nw, j + 1, len, w, tj, lane);
      __syncwarp();
    }
  }
  // ---- (4) write back: the window, the spike column; U as a Q slot -------------------------------
  for (int c = 0; c < nw; ++c)
    for (int r = lane; r < nw; r += 32) H[(k0 + r) + (k0 + c) * n] = T_(r, c);
  if (k0 > ilo)
    for (int r = lane; r < nw; r += 32) H[(k0 + r) + (k0 - 1) * n] = (r == 0) ? beta : 0.0;
  __syncwarp();
  store_q_slot(uslot, U, ld, nw, KP, QLD, 0, 1, lane);
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

size_t aed_smem_bytes(int nw) { return ((size_t)2 * nw * (nw | 1) + nw + 32) * sizeof(double); }

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
  aed_kernel<<<1, 32, aed_smem_bytes(nw), st>>>(H, n, ilo, k0, nw, thr, uslot, KP, QLD, ew, ei, res);
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
