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
// Warp roles.  16 chase warps run the steps; per step two phases separated by a named barrier:
//   phase 1  (one warp per bulge) compute the reflector from column p (or the intro vector),
//            store beta / exact zeros in column p, apply it from the left to rows p+1..p+m,
//            columns p+1..w1 (lanes across columns), publish it in an SMEM ring;
//   phase 2  (same warp) apply it from the right to columns p+1..p+m of the window rows
//            w0..p+m+1 (lanes across rows).
// 8 accumulation warps take the reflectors from the ring (mbarrier full/empty handshake, up to
// kRing steps behind) and apply them to Q_W rows 0..p0+3 (p0 = the chain's deepest bulge; deeper
// rows of Q_W are still identity rows).  Q_W is not read by the chase, so its update leaves the
// chase's critical path; the accumulation warps keep the steps in order (a named barrier) because
// neighbouring bulges of consecutive steps share a column.
// Bulges are 3 apart, so within a phase different bulges touch disjoint rows (phase 1) or
// disjoint columns (phase 2).  Phase 1 of bulge j writes beta into H[p+1,p] before phase 2 of the
// bulge above (at p-3) updates that entry -- the sequential order.
//
// The kernel is latency-bound (a chain of small dependent reflectors): one chase warp per bulge,
// 32-bit indices, the common 3-reflector specialised, one square root and one division per
// reflector.
//
// SMEM layout: column-major H window and Q_W with an odd leading dimension (kw | 1): a warp
// walking a row (phase 1) or a column (phase 2) hits 32 distinct banks.
#include <climits>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "kernels.hpp"

namespace hqr {

namespace {

constexpr int kHWarps = 16;                      // chase warps: reflectors, left, right (window)
constexpr int kQWarps = 8;                       // accumulation warps: Q_W <- Q_W P
constexpr int kChaseThreads = 32 * (kHWarps + kQWarps);
constexpr int kRing = 8;                         // steps of reflectors in flight to the Q warps
constexpr int kMaxRingBulges = 64;               // bulges per step the ring holds

__global__ void __launch_bounds__(kChaseThreads, 1) chase_kernel(StepArgs a) {
  extern __shared__ double sm[];
  __shared__ Refl ring[kRing][kMaxRingBulges];
  __shared__ __align__(8) uint64_t full[kRing], empty[kRing];
  const WindowDesc W = a.wins[a.win_begin + blockIdx.x];
  const int kw = W.w1 - W.w0 + 1;
  const int ldh = kw | 1;
  double* Hs = sm;
  double* Qs = Hs + kw * ldh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int w0 = W.w0;
  const int ilo = W.ilo, ihi = W.ihi;  // the active block of this window's chain
  const int nbc = W.nbc;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&full[i], kHWarps);
      mbar_init(&empty[i], kQWarps);
    }
  }
  // load the window (coalesced along columns), Q_W = I
  {
    const double* g = a.H + (int64_t)(w0 - a.hcol0) * n + w0;
    for (int c = warp; c < kw; c += kHWarps + kQWarps) {
      const double* gc = g + (int64_t)c * n;
      for (int r = lane; r < kw; r += 32) {
        Hs[r + c * ldh] = gc[r];
        Qs[r + c * ldh] = (r == c) ? 1.0 : 0.0;
      }
    }
  }
  __syncthreads();

  const int rmaxH = ihi - w0;  // last window row inside the active block
  if (warp < kHWarps) {
    // ======================= chase warps =======================
    for (int t = W.t0; t <= W.t1; ++t) {
      const int j = t - W.t0, slot = j % kRing;
      if (j >= kRing) mbar_wait(&empty[slot], (unsigned)((j / kRing) - 1) & 1);
      // ---- phase 1: reflectors + left application (warp -> bulges warp, warp + 16, ...) ------
      for (int jj = warp; jj < nbc; jj += kHWarps) {
        Refl R;
        R.pl = INT_MIN;
        R.m = 3;
        const int p = ilo - 1 + t - 3 * jj;
        if (p >= ilo - 1 && p <= ihi - 2) {
          const int pl = p - w0;
          const int m = (p <= ihi - 3) ? 3 : 2;
          double x0, x1, x2;
          if (p == ilo - 1) {  // bulge introduction; the window starts at ilo
            intro_vector(Hs, ldh, a.coef + 4 * (W.b0 + jj), x0, x1, x2);
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
            R.v1 = v1; R.v2 = v2; R.tau = tau; R.pl = pl; R.m = m;
            left_apply(Hs + (pl + 1), ldh, (p == ilo - 1) ? 0 : pl + 1, kw, m, v1, v2, tau, lane);
          }
        }
        if (lane == 0) ring[slot][jj] = R;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[slot]);   // this warp's reflectors of step t are published
      named_sync(1, 32 * kHWarps);                // phase 1 of every bulge before any phase 2
      // ---- phase 2: right application to the window rows w0..p+m+1 -------------------------
      for (int jj = warp; jj < nbc; jj += kHWarps) {
        const Refl R = ring[slot][jj];
        if (R.pl == INT_MIN) continue;
        right_apply(Hs + (R.pl + 1) * ldh, ldh, min(R.pl + R.m + 1, rmaxH) + 1, R, lane);
      }
      named_sync(1, 32 * kHWarps);
    }
  } else {
    // ============ accumulation warps: Q_W(:, p+1..p+m) <- Q_W(:, p+1..p+m) P, one step behind ====
    const int qw = warp - kHWarps;
    for (int t = W.t0; t <= W.t1; ++t) {
      const int j = t - W.t0, slot = j % kRing;
      mbar_wait(&full[slot], (unsigned)(j / kRing) & 1);
      // rows of Q_W below the chain's deepest reflector so far are still identity rows
      const int rQ = min(ilo - 1 + t - w0 + 3, kw - 1);
      for (int jj = qw; jj < nbc; jj += kQWarps) {
        const Refl R = ring[slot][jj];
        if (R.pl == INT_MIN) continue;
        const int q0 = q_first_row(W, jj);
        right_apply(Qs + (R.pl + 1) * ldh + q0, ldh, rQ + 1 - q0, R, lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      named_sync(2, 32 * kQWarps);  // steps in order: neighbouring bulges share a column
    }
  }
  __syncthreads();
  aftermath_scan(Hs, ldh, W, a.aftermath, threadIdx.x, kChaseThreads);  // a9 (check only)

  // write back the window; store Q_W column-major with ld = QLD (= the update kernels' SMEM
  // layout), zero padded to KP x QLD
  {
    double* g = a.H + (int64_t)(w0 - a.hcol0) * n + w0;
    for (int c = warp; c < kw; c += kHWarps + kQWarps) {
      double* gc = g + (int64_t)c * n;
      for (int r = lane; r < kw; r += 32) gc[r] = Hs[r + c * ldh];
    }
  }
  const int KP = a.KP, QLD = a.QLD;
  double* Q = a.qslots + (size_t)(W.slot + a.slot_offset) * KP * QLD;
  store_q_slot(Q, Qs, ldh, kw, KP, QLD, warp, kHWarps + kQWarps, lane);
  if (a.wstats) {
    __syncthreads();
    if (threadIdx.x == 0) a.wstats[a.win_begin + blockIdx.x] = band_units(Q, KP, QLD);
  }
}

}  // namespace

size_t chase_smem_bytes(int kw, int nbc) {
  (void)nbc;
  const int ldh = kw | 1;
  return (size_t)2 * kw * ldh * sizeof(double);
}

cudaError_t launch_chase(const StepArgs& a, int max_kw, int max_nbc, cudaStream_t st) {
  if (max_nbc > kMaxRingBulges) return cudaErrorInvalidConfiguration;
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
