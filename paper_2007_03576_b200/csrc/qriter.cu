// qriter.cu -- pieces of the QR iteration around the sweep (partial; reading
// R21): the eigenvalues of a small Hessenberg block (the shifts of the next sweep, and the
// eigenvalues of the small blocks left at the end -- the role of the paper's small Schur task,
// P:367-372, here a Francis double-shift QR iteration in one CTA), and the deflation step that sets
// negligible subdiagonal entries to zero after a sweep (criterion R16).
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

}  // namespace

int small_eig_max() { return kSmallMax; }

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
