// chase.cu -- bulge-chase kernel ("push bulges") for sm_100a.
//
// One CTA per diagonal window W = [w0, w1] of one bulge chain.  The window
// block H(W, W) and its accumulated orthogonal factor Q_W ("accumulator matrix") live in
// shared memory for the whole window; the chain's bulges are chased for chain-local steps
// [t0, t1] (plan.hpp), then H(W, W) is written back and Q_W is stored for the off-diagonal
// update kernels (update.cu).  Every reflector follows the textbook double-shift step
// (P:198-203): bulge introduction from the first column of (H - s I)(H - s' I), 3x3
// Householder reflectors chasing the bulge, a final 2x2 reflector at p = ihi - 2.
//
// Per step, two phases separated by __syncthreads:
//   phase 1  (one warp per bulge) compute the reflector from column p (or the intro vector),
//            store beta / exact zeros in column p, apply it from the left to rows p+1..p+m,
//            columns p+1..w1 (lanes across columns);
//   phase 2  apply every reflector from the right to columns p+1..p+m, rows w0..p+m+1 of the
//            window and rows 0..p0+3 of Q_W, p0 the chain's deepest bulge (lanes across rows).
// Bulges are 3 apart, so within a phase different bulges touch disjoint rows (phase 1) or
// disjoint columns (phase 2).  Phase 1 of bulge j writes beta into H[p+1,p] before phase 2 of the
// bulge above (at p-3) updates that entry -- the sequential order.
//
// SMEM layout: column-major H window and Q_W with an odd leading dimension (kw | 1): a warp
// walking a row (phase 1) or a column (phase 2) hits 32 distinct banks.
#include <climits>
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace hqr {

namespace {

constexpr int kChaseThreads = 256;
constexpr int kChaseWarps = kChaseThreads / 32;

// Householder reflector (reading R2): P = I - tau v v^T, v = [1, v1, v2],
// P x = beta e1 with beta = -sign(x0) ||x||, sign(0) = +1; zero tail -> identity.
__device__ __forceinline__ void house(int m, double x0, double x1, double x2, double& v1,
                                      double& v2, double& tau, double& beta) {
  double tail2 = x1 * x1 + (m == 3 ? x2 * x2 : 0.0);
  if (tail2 == 0.0) {
    v1 = 0.0; v2 = 0.0; tau = 0.0; beta = x0;
    return;
  }
  double nrm = sqrt(x0 * x0 + tail2);
  double b = (x0 >= 0.0) ? -nrm : nrm;
  tau = (b - x0) / b;
  double d = x0 - b;
  v1 = x1 / d;
  v2 = (m == 3) ? x2 / d : 0.0;
  beta = b;
}

__global__ void __launch_bounds__(kChaseThreads) chase_kernel(StepArgs a) {
  extern __shared__ double sm[];
  const WindowDesc W = a.wins[a.win_begin + blockIdx.x];
  const int kw = W.w1 - W.w0 + 1;
  const int ldh = kw | 1;
  double* Hs = sm;
  double* Qs = Hs + (size_t)kw * ldh;
  double* R = Qs + (size_t)kw * ldh;            // per bulge: v1, v2, tau
  int* Rp = reinterpret_cast<int*>(R + 3 * W.nbc);  // per bulge: local p (INT_MIN = inactive)
  int* Rm = Rp + W.nbc;                              // per bulge: m (2 or 3)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n, w0 = W.w0;
  const int64_t ilo = a.ilo, ihi = a.ihi;

  // load the window (coalesced along columns), Q_W = I
  for (int idx = tid; idx < kw * kw; idx += kChaseThreads) {
    int c = idx / kw, r = idx - c * kw;
    Hs[r + c * ldh] = a.H[(w0 + r) + (w0 + c) * n];
    Qs[r + c * ldh] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();

  const int rmaxH = (int)(ihi - w0);  // last window row inside the active block
  for (int t = W.t0; t <= W.t1; ++t) {
    // ---- phase 1: reflectors + left application ------------------------------------------
    for (int jj = warp; jj < W.nbc; jj += kChaseWarps) {
      const int64_t p = ilo - 1 + t - 3 * (int64_t)jj;
      if (p < ilo - 1 || p > ihi - 2) {
        if (lane == 0) Rp[jj] = INT_MIN;
        continue;
      }
      const int pl = (int)(p - w0);
      const int m = (p <= ihi - 3) ? 3 : 2;
      double x0, x1, x2;
      if (p == ilo - 1) {  // bulge introduction; window starts at ilo so local (0,0)
        const int j = W.b0 + jj;
        const double sigma = a.coef[2 * j], pi = a.coef[2 * j + 1];
        const double h00 = Hs[0], h10 = Hs[1], h01 = Hs[ldh], h11 = Hs[1 + ldh], h21 = Hs[2 + ldh];
        x0 = h00 * (h00 - sigma) + h01 * h10 + pi;
        x1 = h10 * (h00 + h11 - sigma);
        x2 = h10 * h21;
      } else {
        const double* col = Hs + (size_t)pl * ldh;
        x0 = col[pl + 1];
        x1 = col[pl + 2];
        x2 = (m == 3) ? col[pl + 3] : 0.0;
      }
      double v1, v2, tau, beta;
      house(m, x0, x1, x2, v1, v2, tau, beta);
      __syncwarp();
      if (lane == 0) {
        if (p >= ilo) {
          double* col = Hs + (size_t)pl * ldh;
          col[pl + 1] = beta;
          col[pl + 2] = 0.0;
          if (m == 3) col[pl + 3] = 0.0;
        }
        R[3 * jj] = v1; R[3 * jj + 1] = v2; R[3 * jj + 2] = tau;
        Rp[jj] = pl; Rm[jj] = m;
      }
      if (tau != 0.0) {
        const int c0 = (p == ilo - 1) ? 0 : pl + 1;
        for (int c = c0 + lane; c < kw; c += 32) {
          double* hc = Hs + (size_t)c * ldh + (pl + 1);
          double h0 = hc[0], h1 = hc[1], h2 = (m == 3) ? hc[2] : 0.0;
          double tw = tau * (h0 + v1 * h1 + v2 * h2);
          hc[0] = h0 - tw;
          hc[1] = h1 - tw * v1;
          if (m == 3) hc[2] = h2 - tw * v2;
        }
      }
    }
    __syncthreads();
    // ---- phase 2: right application to the window and to Q_W --------------------------------
    // rows of Q_W below the deepest reflector so far (the chain's bulge 0 at p0 = ilo-1+t touches
    // rows <= p0+3, and positions only grow) are still identity rows: skip them
    const int rQ0 = (int)(ilo - 1 + t - w0 + 3);
    for (int jj = warp; jj < W.nbc; jj += kChaseWarps) {
      const int pl = Rp[jj];
      if (pl == INT_MIN) continue;
      const double tau = R[3 * jj + 2];
      if (tau == 0.0) continue;
      const double v1 = R[3 * jj], v2 = R[3 * jj + 1];
      const int m = Rm[jj];
      double* c1 = Hs + (size_t)(pl + 1) * ldh;
      const int rH = min(pl + m + 1, rmaxH);
      for (int r = lane; r <= rH; r += 32) {
        double h0 = c1[r], h1 = c1[r + ldh], h2 = (m == 3) ? c1[r + 2 * ldh] : 0.0;
        double tw = tau * (h0 + v1 * h1 + v2 * h2);
        c1[r] = h0 - tw;
        c1[r + ldh] = h1 - tw * v1;
        if (m == 3) c1[r + 2 * ldh] = h2 - tw * v2;
      }
      double* q1 = Qs + (size_t)(pl + 1) * ldh;
      const int rQ = min(rQ0, kw - 1);
      for (int r = lane; r <= rQ; r += 32) {
        double q0 = q1[r], qa = q1[r + ldh], qb = (m == 3) ? q1[r + 2 * ldh] : 0.0;
        double tw = tau * (q0 + v1 * qa + v2 * qb);
        q1[r] = q0 - tw;
        q1[r + ldh] = qa - tw * v1;
        if (m == 3) q1[r + 2 * ldh] = qb - tw * v2;
      }
    }
    __syncthreads();
  }

  // write back the window and store Q_W (column-major, ld = KP, zero padded to KP x KP)
  for (int idx = tid; idx < kw * kw; idx += kChaseThreads) {
    int c = idx / kw, r = idx - c * kw;
    a.H[(w0 + r) + (w0 + c) * n] = Hs[r + c * ldh];
  }
  const int KP = a.KP;
  double* Q = a.qslots + (size_t)W.slot * KP * KP;
  for (int idx = tid; idx < KP * KP; idx += kChaseThreads) {
    int c = idx / KP, r = idx - c * KP;
    Q[idx] = (r < kw && c < kw) ? Qs[r + c * ldh] : 0.0;
  }
}

}  // namespace

size_t chase_smem_bytes(int kw, int nbc) {
  int ldh = kw | 1;
  return (size_t)2 * kw * ldh * sizeof(double) + (size_t)nbc * (3 * sizeof(double) + 2 * sizeof(int));
}

cudaError_t launch_chase(const StepArgs& a, int max_kw, int max_nbc, cudaStream_t st) {
  size_t smem = chase_smem_bytes(max_kw, max_nbc);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(chase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  chase_kernel<<<a.win_count, kChaseThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace hqr
