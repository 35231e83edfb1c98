// qz.cu -- generalized (QZ) multishift sweep on a Hessenberg-triangular pair (SURVEY §8(f)
// NEXT-4) for sm_100a: the chase kernel of one wavefront step.
//
// One CTA per diagonal window W = [w0, w1] (the QR sweep's windows: the bulge of a QZ step has the
// same footprint -- left reflectors on rows p+1..p+3, right-hand side reflectors on columns
// p+1..p+3 reaching H row p+4 -- so plan.hpp's window rule and wavefront apply unchanged).  H(W,W),
// T(W,W) and the two accumulated factors Q_W (left reflectors) and Z_W (right-hand side
// reflectors) live in shared memory; per chain-local step, two phases separated by a barrier:
//   phase 1  (a warp per bulge) the left reflector from H's column p (or the bulge vector
//            (H T^-1 - s I)(H T^-1 - s' I) e1, reading R17), beta / exact zeros in column p, applied
//            to rows p+1..p+m of H and T (lanes across columns) and accumulated into Q_W's columns;
//   phase 2  (same warp) the right-hand side reflectors (reading R18) that return T to triangular
//            form: from T's row p+3 (columns p+1..p+3), then from T's row p+2 (columns p+1..p+2), each
//            applied to the columns of H (rows <= p+4), T (rows <= the row) and Z_W, the zeroed T
//            entries stored as exact zeros and the diagonal as beta.
// Bulges are 3 apart: within a phase different bulges touch disjoint rows (phase 1) or disjoint
// columns (phase 2); a lower bulge's left reflector reads column p before the upper bulge's right
// reflectors change it (the sequential order), and a left and a right reflector meeting in one
// block commute.  The off-diagonal updates (Q_W^T on H and T rows right of W, Z_W on H and T
// columns above W, Qacc Q_W and Zacc Z_W) run on the FP64 DMMA update kernels of update.cu.
#include <climits>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "kernels.hpp"

namespace hqr {

namespace {

constexpr int kQZWarps = 16;
constexpr int kQZThreads = 32 * kQZWarps;

// Right application of P = I - tau u u^T (u of length m, 2 or 3) to `rows` rows of m consecutive
// SMEM columns starting at c1 (ld ldh); lanes across rows.
__device__ __forceinline__ void right_apply_u(double* c1, int ldh, int rows, int m, double u0, double u1,
                                              double u2, double tau, int lane) {
  if (m == 3) {
    for (int i = lane; i < rows; i += 32) {
      double* x = c1 + i;
      const double h0 = x[0], h1 = x[ldh], h2 = x[2 * ldh];
      const double tw = tau * fma(u2, h2, fma(u1, h1, u0 * h0));
      x[0] = fma(-tw, u0, h0);
      x[ldh] = fma(-tw, u1, h1);
      x[2 * ldh] = fma(-tw, u2, h2);
    }
  } else {
    for (int i = lane; i < rows; i += 32) {
      double* x = c1 + i;
      const double h0 = x[0], h1 = x[ldh];
      const double tw = tau * fma(u1, h1, u0 * h0);
      x[0] = fma(-tw, u0, h0);
      x[ldh] = fma(-tw, u1, h1);
    }
  }
}

// R17: the bulge vector from the top-left corners of the H and T windows and the pair c4
__device__ __forceinline__ void qz_intro_vector(const double* Hs, const double* Ts, int ldh, const double* c4,
                                                double& x0, double& x1, double& x2) {
  const double h00 = Hs[0], h10 = Hs[1], h01 = Hs[ldh], h11 = Hs[1 + ldh], h21 = Hs[2 + ldh];
  const double t00 = Ts[0], t01 = Ts[ldh], t11 = Ts[1 + ldh];
  const double sigma = c4[0] + c4[1], pi = c4[0] * c4[1] - c4[2] * c4[3];
  const double a = h00 / t00, b = h10 / t00;
  const double y1 = b / t11;
  const double y0 = (a - t01 * y1) / t00;
  x0 = h00 * y0 + h01 * y1 - sigma * a + pi;
  x1 = h10 * y0 + h11 * y1 - sigma * b;
  x2 = h21 * y1;
}

__global__ void __launch_bounds__(kQZThreads, 1) qz_chase_kernel(StepArgs a, double* T, double* zslots) {
  extern __shared__ double sm[];
  const WindowDesc W = a.wins[a.win_begin + blockIdx.x];
  const int kw = W.w1 - W.w0 + 1;
  const int ldh = kw | 1;
  double* Hs = sm;
  double* Ts = Hs + kw * ldh;
  double* Qs = Ts + kw * ldh;
  double* Zs = Qs + kw * ldh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int w0 = W.w0, ilo = W.ilo, ihi = W.ihi, nbc = W.nbc;
  {
    const double* gh = a.H + (int64_t)w0 * n + w0;
    const double* gt = T + (int64_t)w0 * n + w0;
    for (int c = warp; c < kw; c += kQZWarps)
      for (int r = lane; r < kw; r += 32) {
        Hs[r + c * ldh] = gh[r + (int64_t)c * n];
        Ts[r + c * ldh] = gt[r + (int64_t)c * n];
        const double id = (r == c) ? 1.0 : 0.0;
        Qs[r + c * ldh] = id;
        Zs[r + c * ldh] = id;
      }
  }
  __syncthreads();
  const int rmaxH = ihi - w0;
  for (int t = W.t0; t <= W.t1; ++t) {
    // ---- phase 1: left reflectors (H column p), applied to H and T rows and to Q_W --------------
    for (int jj = warp; jj < nbc; jj += kQZWarps) {
      const int p = ilo - 1 + t - 3 * jj;
      if (p >= ilo - 1 && p <= ihi - 2) {
        const int pl = p - w0;
        const int m = (p <= ihi - 3) ? 3 : 2;
        double x0, x1, x2;
        if (p == ilo - 1) {
          qz_intro_vector(Hs, Ts, ldh, a.coef + 4 * (W.b0 + jj), x0, x1, x2);
        } else {
          const double* col = Hs + pl * ldh + pl;
          x0 = col[1];
          x1 = col[2];
          x2 = (m == 3) ? col[3] : 0.0;
        }
        double v1, v2, tau, beta;
        house(x0, x1, x2, v1, v2, tau, beta);
        __syncwarp();
        if (lane == 0 && p >= ilo) {
          double* col = Hs + pl * ldh + pl;
          col[1] = beta;
          col[2] = 0.0;
          if (m == 3) col[3] = 0.0;
        }
        if (tau != 0.0) {
          const int c0 = (p == ilo - 1) ? 0 : pl + 1;
          for (int c = c0 + lane; c < kw; c += 32) {  // H rows pl+1..pl+m
            double* hc = Hs + (pl + 1) + c * ldh;
            const double h0 = hc[0], h1 = hc[1], h2 = (m == 3) ? hc[2] : 0.0;
            const double tw = tau * fma(v2, h2, fma(v1, h1, h0));
            hc[0] = h0 - tw;
            hc[1] = fma(-tw, v1, h1);
            if (m == 3) hc[2] = fma(-tw, v2, h2);
          }
          for (int c = pl + 1 + lane; c < kw; c += 32) {  // T rows pl+1..pl+m (upper triangular)
            double* tc = Ts + (pl + 1) + c * ldh;
            const double h0 = tc[0], h1 = tc[1], h2 = (m == 3) ? tc[2] : 0.0;
            const double tw = tau * fma(v2, h2, fma(v1, h1, h0));
            tc[0] = h0 - tw;
            tc[1] = fma(-tw, v1, h1);
            if (m == 3) tc[2] = fma(-tw, v2, h2);
          }
          right_apply_u(Qs + (pl + 1) * ldh, ldh, kw, m, 1.0, v1, v2, tau, lane);  // Q_W <- Q_W P
        }
      }
    }
    __syncthreads();
    // ---- phase 2: right-hand side reflectors restoring T (rows p+3, then p+2) -------------------
    for (int jj = warp; jj < nbc; jj += kQZWarps) {
      const int p = ilo - 1 + t - 3 * jj;
      if (p < ilo - 1 || p > ihi - 2) continue;
      const int pl = p - w0;
      const int m = (p <= ihi - 3) ? 3 : 2;
      for (int mm = m; mm >= 2; --mm) {
        const int row = pl + mm;  // local T row whose entries left of the diagonal are zeroed
        const double* tr = Ts + row + (pl + 1) * ldh;
        // R18: the R2 reflector of the reversed row, reversed
        const double r0 = tr[0], r1 = tr[ldh], r2 = (mm == 3) ? tr[2 * ldh] : 0.0;
        double v1, v2, tau, beta;
        if (mm == 3) house(r2, r1, r0, v1, v2, tau, beta);
        else house(r1, r0, 0.0, v1, v2, tau, beta);
        const double u0 = (mm == 3) ? v2 : v1, u1 = (mm == 3) ? v1 : 1.0, u2 = 1.0;
        if (tau != 0.0) {
          right_apply_u(Hs + (pl + 1) * ldh, ldh, min(pl + 4, rmaxH) + 1, mm, u0, u1, u2, tau, lane);
          right_apply_u(Ts + (pl + 1) * ldh, ldh, row + 1, mm, u0, u1, u2, tau, lane);
          right_apply_u(Zs + (pl + 1) * ldh, ldh, kw, mm, u0, u1, u2, tau, lane);
        }
        __syncwarp();
        if (lane == 0) {  // R9: exact zeros left of the diagonal, beta on it
          double* trw = Ts + row + (pl + 1) * ldh;
          for (int i = 0; i < mm - 1; ++i) trw[i * ldh] = 0.0;
          trw[(mm - 1) * ldh] = beta;
        }
        __syncwarp();
      }
    }
    __syncthreads();
  }
  {
    double* gh = a.H + (int64_t)w0 * n + w0;
    double* gt = T + (int64_t)w0 * n + w0;
    for (int c = warp; c < kw; c += kQZWarps)
      for (int r = lane; r < kw; r += 32) {
        gh[r + (int64_t)c * n] = Hs[r + c * ldh];
        gt[r + (int64_t)c * n] = Ts[r + c * ldh];
      }
  }
  const int KP = a.KP, QLD = a.QLD;
  const size_t slot = (size_t)(W.slot + a.slot_offset) * KP * QLD;
  store_q_slot(a.qslots + slot, Qs, ldh, kw, KP, QLD, warp, kQZWarps, lane);
  store_q_slot(zslots + slot, Zs, ldh, kw, KP, QLD, warp, kQZWarps, lane);
}

}  // namespace

size_t qz_chase_smem_bytes(int kw) { return (size_t)4 * kw * (kw | 1) * sizeof(double); }

cudaError_t launch_qz_chase(const StepArgs& a, double* T, double* zslots, int max_kw, cudaStream_t st) {
  const size_t smem = qz_chase_smem_bytes(max_kw);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(qz_chase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  qz_chase_kernel<<<a.win_count, kQZThreads, smem, st>>>(a, T, zslots);
  return cudaGetLastError();
}

}  // namespace hqr
