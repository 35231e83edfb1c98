// device_common.cuh -- sm_100a device helpers shared by the product kernels (update.cu, chase.cu,
// step.cu): FP64 mma.sync, mbarrier / bulk-copy / 2-D TMA wrappers, tile geometry.  Product path.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdio>

#include "kernels.hpp"

namespace hqr {

// TMA-path panel tiles and SMEM ring depth (update.cu bulk kernels, step.cu): Q_W (KP x pad_ld(KP))
// stays resident next to a ring of stages_of(KP) panel tiles.  KP = 96: 32-wide tiles, five stages
// (76.8 + 5 x 27.6 KB): with three consumer groups a group's next tile is loaded about two thirds
// of a tile time ahead (measured: 40-wide x 4 stages 153.4 ms, 32 x 5 146.1 ms, 24 x 6 153.9 ms).
// (left_cols / right_rows: kernels.hpp)
__host__ __device__ constexpr int stages_of(int KP) { return KP <= 64 ? 4 : KP == 96 ? 5 : 2; }
// Panel leading dimension: an m8n8k4 fragment load (per half-warp: 4 consecutive doubles x 4 strided
// rows) is conflict-free iff the stride is an odd multiple of 4 doubles: smallest such ld >= x.
__host__ __device__ constexpr int panel_ld(int x) { return x + ((4 - x) % 8 + 8) % 8; }
// cp.async (odd n) kernels keep their own tiles
__host__ __device__ constexpr int gen_left_cols(int KP) { return KP <= 64 ? 64 : KP == 96 ? 48 : 32; }
__host__ __device__ constexpr int gen_right_rows(int KP) { return KP <= 64 ? 64 : KP == 96 ? 48 : 32; }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ---- async copy / mbarrier helpers ---------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
#if defined(HQR_WATCHDOG) || defined(HQR_CLOOP)  // debugging builds only
__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
#endif
#if defined(HQR_CLOOP)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity, int tag = 0) {
  while (!mbar_try(bar, parity)) {
  }
}
#elif defined(HQR_WATCHDOG)  // bounded waits that report where they hung, then trap
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity, int tag = 0) {
  long long it = 0;
  while (!mbar_try(bar, parity)) {
#ifndef HQR_WD_LIMIT
#define HQR_WD_LIMIT 26
#endif
    if (++it == (1ll << HQR_WD_LIMIT)) {
#ifndef HQR_WD_NOPRINT
      printf("hqr watchdog: block %d thread %d tag %d bar smem+%u parity %u\n", blockIdx.x, threadIdx.x, tag,
             smem_u32(bar), parity);
#endif
      __trap();
    }
  }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity, int tag = 0) {
  (void)tag;
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
#endif
// non-blocking test of a phase (parity as mbar_wait)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
// 1-D bulk copy global -> shared through the TMA engine; completes tx bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// 2-D tensor (TMA) load of one box at (row c0, column c1); completes box bytes on `bar`
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(smem_u32(smem)), "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }


__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

// Householder reflector (reading R2): P = I - tau v v^T, v = [1, v1, v2],
// P x = beta e1 with beta = -sign(x0) ||x||, sign(0) = +1; zero tail -> identity.  Computed on x
// scaled by a power of two (R15: exact, so the result rounds exactly like the unscaled formulas
// wherever those stay finite, and stays finite where they would not).
// With d = x0 - beta and r = 1 / (d * beta): v_i = x_i / d = x_i * beta * r, tau = -d / beta = -d*d*r.
// The chase's critical path is a chain of these (one per bulge and step), so the square root and
// the reciprocal use the hardware approximations refined by Newton steps (rounding-level
// differences from IEEE sqrt / division, reading R10) instead of the long IEEE sequences.
// One Newton step each: house() follows rsqrt with a Newton correction of sqrt(s) and rcp with a
// final correction, each of which doubles the correct bits again (tools/house_lat.cu: no difference
// from IEEE sqrt / division over 2^20 random reflectors across 2^+-200; 41 cycles shorter chain).
__device__ __forceinline__ double rsqrt_nr(double s) {  // 1 / sqrt(s) to ~2^-40, s > 0 normal
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
  return y * fma(-0.5 * s * y, y, 1.5);  // Newton: ~2x the correct bits per step
}
__device__ __forceinline__ double rcp_nr(double q) {  // 1 / q, q != 0 normal
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = r * fma(-q, r, 2.0);
  return fma(r, fma(-q, r, 1.0), r);  // final correction
}
__device__ __forceinline__ void house(double x0, double x1, double x2, double& v1, double& v2,
                                      double& tau, double& beta) {
#ifdef HQR_EXP_CHEAPHOUSE  // timing experiment only (wrong results): no reflector arithmetic
  v1 = x1 * 0.5; v2 = x2 * 0.5; tau = (x1 != 0.0) ? 0.25 : 0.0; beta = x0;
  return;
#endif
  // R15 scale 2^-e, branch-free (the chase's critical path; registers are tight in the fused
  // kernel): for max|x| outside [2^-1022, 2^1021) -- entries the update GEMMs could not carry
  // either -- the unscaled formulas are used
  const double amax = fmax(fabs(x0), fmax(fabs(x1), fabs(x2)));
  const long long E = __double_as_longlong(amax) >> 52;   // biased exponent (amax >= 0)
  const bool ok = (E >= 1) & (E <= 2044);
  const double down = ok ? __longlong_as_double((2045 - E) << 52) : 1.0;
  x1 *= down; x2 *= down;
  const double tail2 = fma(x1, x1, x2 * x2);
  if (tail2 == 0.0) {  // zero tail: identity, beta = x0
    v1 = 0.0; v2 = 0.0; tau = 0.0; beta = x0;
    return;
  }
  const double xs0 = x0 * down;
  const double s = fma(xs0, xs0, tail2);
  const double y = rsqrt_nr(s);
  double nrm = s * y;
  nrm = fma(0.5 * y, fma(-nrm, nrm, s), nrm);  // sqrt(s), Newton-corrected
  const double b = (xs0 >= 0.0) ? -nrm : nrm;
  const double d = xs0 - b;
  const double r = rcp_nr(d * b);
  const double br = b * r;
  v1 = x1 * br;
  v2 = x2 * br;
  tau = -d * d * r;
  beta = b * (ok ? __longlong_as_double((E + 1) << 52) : 1.0);
}

// Bulge introduction (a2; reading R1): x = the first column of (H - s I)(H - s' I) at the top of the
// active block, from the window's top-left 3x3 corner Hs (ld ldh) and the pair c4 = (re, re', im,
// im'): x0 = h00 (h00 - sigma) + h01 h10 + pi, x1 = h10 (h00 + h11 - sigma), x2 = h10 h21 with
// sigma = re + re', pi = re re' - im im', all inputs scaled by one power of two first (R15: x is
// then 2^-2e times the unscaled vector, which has the same reflector).  Once per bulge and sweep.
__device__ __forceinline__ void intro_vector(const double* Hs, int ldh, const double* c4, double& x0,
                                             double& x1, double& x2) {
  double h00 = Hs[0], h10 = Hs[1], h01 = Hs[ldh], h11 = Hs[1 + ldh], h21 = Hs[2 + ldh];
  double re0 = c4[0], re1 = c4[1], im0 = c4[2], im1 = c4[3];
  const double amax = fmax(fmax(fmax(fabs(h00), fabs(h10)), fmax(fabs(h01), fabs(h11))),
                           fmax(fmax(fabs(h21), fabs(re0)), fmax(fmax(fabs(re1), fabs(im0)), fabs(im1))));
  const long long E = __double_as_longlong(amax) >> 52;  // R15 (as house: [2^-1022, 2^1021))
  if (E >= 1 && E <= 2044) {
    const double down = __longlong_as_double((2045 - E) << 52);
    h00 *= down; h10 *= down; h01 *= down; h11 *= down; h21 *= down;
    re0 *= down; re1 *= down; im0 *= down; im1 *= down;
  }
  const double sigma = re0 + re1, pi = re0 * re1 - im0 * im1;
  x0 = h00 * (h00 - sigma) + h01 * h10 + pi;
  x1 = h10 * (h00 + h11 - sigma);
  x2 = h10 * h21;
}

// Aftermath subdiagonal scan (check only, reading R16) of rows [W.scan_lo, W.scan_hi]
// after W's chase, from its SMEM copy Hs (ld ldh): flags[i] = 2 if h(i+1,i) == 0, 1 if
// |h(i+1,i)| <= 2^-52 (|h(i,i)| + |h(i+1,i+1)|), else 0.  The boundary rows ilo-1 / ihi (outside
// the window) hold h(i+1, i) = 0, verified at entry (-10) and never written by the sweep: 2.
// No mutation.
__device__ __forceinline__ void aftermath_scan(const double* Hs, int ldh, const WindowDesc& W,
                                               signed char* flags, int tid, int nthreads) {
  if (!flags || W.scan_hi < W.scan_lo) return;
  for (int i = W.scan_lo + tid; i <= W.scan_hi; i += nthreads) {
    const int l = i - W.w0;
    signed char f = 2;
    if (l >= 0 && l + 1 < W.w1 - W.w0 + 1) {
      const double s = Hs[(l + 1) + l * ldh];
      const double d = fabs(Hs[l + l * ldh]) + fabs(Hs[(l + 1) + (l + 1) * ldh]);
      f = (s == 0.0) ? 2 : (fabs(s) <= 0x1p-52 * d) ? 1 : 0;
    }
    flags[i] = f;
  }
}

struct Refl {      // one reflector in the ring: P = I - tau v v^T acting on local columns pl+1..pl+m
  double v1, v2, tau;
  int pl, m;       // pl = INT_MIN: no reflector (inactive bulge or tau = 0)
};


// First Q_W row bulge jj of window W can reach.  Q_W starts as I at the window's first step; a
// row's support then grows only through the reflectors that touch it, and its right end follows
// the deepest bulge that ever touched it (a deeper bulge starts 3 columns further right and is
// never reached).  Rows above bulge jj's first reflector (local columns pf+1..pf+3) belong to
// bulges above it, so they stay zero in bulge jj's columns; a bulge introduced in this window
// (pf = ilo-1) can reach every row.
__device__ __forceinline__ int q_first_row(const WindowDesc& W, int jj) {
  const int tf = max(W.t0, 3 * jj);  // bulge jj's first step in this window (p >= ilo - 1)
  const int pf = W.ilo - 1 + tf - 3 * jj;
  return pf <= W.ilo - 1 ? 0 : pf - W.w0 + 1;
}

// Apply reflector r from the right to `rows` rows of three (two) consecutive SMEM columns starting
// at c1 (ld = ldh); lanes across rows.  (Batching two rows per lane before updating measured no
// faster: phase 2 1232 vs 1141 cycles per step.)
__device__ __forceinline__ void right_apply(double* c1, int ldh, int rows, const Refl& r, int lane) {
#ifdef HQR_EXP_NOQ
  if (rows > 64) return;  // timing experiment only (wrong results): skip long (Q_W) applications
#endif
  if (r.m == 3) {
    for (int i = lane; i < rows; i += 32) {
      double* x = c1 + i;
      const double h0 = x[0], h1 = x[ldh], h2 = x[2 * ldh];
      const double tw = r.tau * fma(r.v2, h2, fma(r.v1, h1, h0));
      x[0] = h0 - tw;
      x[ldh] = fma(-tw, r.v1, h1);
      x[2 * ldh] = fma(-tw, r.v2, h2);
    }
  } else {
    for (int i = lane; i < rows; i += 32) {
      double* x = c1 + i;
      const double h0 = x[0], h1 = x[ldh];
      const double tw = r.tau * fma(r.v1, h1, h0);
      x[0] = h0 - tw;
      x[ldh] = fma(-tw, r.v1, h1);
    }
  }
}

// Apply reflector (v1, v2, tau; m = 3 or 2 rows) from the left to rows hrow[0..m-1] of the SMEM
// columns c0..kw-1 (column-major, ld = ldh); lanes across columns.
__device__ __forceinline__ void left_apply(double* hrow, int ldh, int c0, int kw, int m, double v1, double v2,
                                           double tau, int lane) {
#ifdef HQR_EXP_NOLEFT
  return;  // timing experiment only (wrong results)
#endif
  if (m == 3) {
    for (int c = c0 + lane; c < kw; c += 32) {
      double* hc = hrow + c * ldh;
      const double h0 = hc[0], h1 = hc[1], h2 = hc[2];
      const double tw = tau * fma(v2, h2, fma(v1, h1, h0));
      hc[0] = h0 - tw;
      hc[1] = fma(-tw, v1, h1);
      hc[2] = fma(-tw, v2, h2);
    }
  } else {
    for (int c = c0 + lane; c < kw; c += 32) {
      double* hc = hrow + c * ldh;
      const double h0 = hc[0], h1 = hc[1];
      const double tw = tau * fma(v1, h1, h0);
      hc[0] = h0 - tw;
      hc[1] = fma(-tw, v1, h1);
    }
  }
}

// Store the accumulated factor Q_W (kw x kw in SMEM, Qs[r + c*ldq]) into its workspace slot
// (KP x QLD doubles, column-major, ld = QLD, zero padded), and record the support of every block of
// 8 columns in the slot's padding rows (never read as matrix entries, QLD >= KP + 4):
//   slot[KP + 8b*QLD] = klo_b, slot[KP + 1 + 8b*QLD] = khi_b,
// multiples of 4 with Q_W[r][c] == 0 for every r outside [klo_b, khi_b), c in [8b, 8b+8) (empty
// block: 0, 0).  The update GEMMs skip the K steps outside a block's extent: the skipped products
// are exact zeros, so the result is unchanged.  The support is a band (each bulge passing a row
// extends its support at most 2 columns left and about s columns right) that covers
// ~60% of a k = 96 window; it is read from the data, not assumed.
__device__ __forceinline__ void store_q_slot(double* __restrict__ Q, const double* __restrict__ Qs, int ldq,
                                             int kw, int KP, int QLD, int warp, int nwarps, int lane) {
  for (int b = warp; b < KP / 8; b += nwarps) {
    int lo = INT_MAX, hi = -1;
    for (int c = 8 * b; c < 8 * b + 8; ++c) {
      double* qc = Q + (size_t)c * QLD;
      for (int r = lane; r < QLD; r += 32) {
        const double v = (r < kw && c < kw) ? Qs[r + c * ldq] : 0.0;
        qc[r] = v;
        if (v != 0.0) {
          lo = min(lo, r);
          hi = max(hi, r);
        }
      }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    __syncwarp();
    if (lane == 0) {
      const bool empty = hi < 0;
      Q[KP + (size_t)8 * b * QLD] = empty ? 0.0 : (double)(lo & ~3);
      Q[KP + 1 + (size_t)8 * b * QLD] = empty ? 0.0 : (double)((hi + 4) & ~3);
    }
  }
}

// After store_q_slot (and a CTA barrier): the window's executed DMMA work per update row/column,
// U = sum over the four Q_W column quarters and over the K segments consume_tile cuts from the
// quarter's block extents of 8 x (active blocks) x (segment length) -- exactly what consume_tile
// multiplies.  One thread.
__device__ __forceinline__ double band_units(const double* __restrict__ Q, int KP, int QLD) {
  const int NB = KP / 32;  // 8-column blocks per quarter
  double u = 0.0;
  for (int qq = 0; qq < 4; ++qq) {
    int lo[4], hi[4], kbeg = KP, kend = 0;
    for (int b = 0; b < NB; ++b) {
      lo[b] = (int)Q[KP + (size_t)8 * (qq * NB + b) * QLD];
      hi[b] = (int)Q[KP + 1 + (size_t)8 * (qq * NB + b) * QLD];
      if (hi[b] > lo[b]) {
        kbeg = min(kbeg, lo[b]);
        kend = max(kend, hi[b]);
      } else {
        lo[b] = KP; hi[b] = 0;
      }
    }
    for (int k = kbeg; k < kend;) {
      int f = NB, l = -1, nxt = kend;
      for (int b = 0; b < NB; ++b) {
        if (lo[b] <= k && k < hi[b]) { f = min(f, b); l = max(l, b); }
        if (lo[b] > k) nxt = min(nxt, lo[b]);
        if (hi[b] > k) nxt = min(nxt, hi[b]);
      }
      if (l >= f) u += 8.0 * (double)(l - f + 1) * (double)(nxt - k);
      k = nxt;
    }
  }
  return u;
}

}  // namespace hqr
