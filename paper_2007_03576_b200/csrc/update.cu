// update.cu -- off-diagonal update kernels ("left update" / "right update", PAPER.md P:400-404,
// P:452-453) on the FP64 tensor cores of sm_100a.
//
// After a wavefront step, every window W = [w0, w1] has its accumulated factor Q_W (k x k).  The
// deferred BLAS-3 updates ("only later applied to the relevant off-diagonal regions using
// matrix-matrix multiplications") are
//   left   H(W, w1+1 : n)  <- Q_W^T H(W, w1+1 : n)         (rows of the window, all columns right)
//   right  H(0 : w0, W)    <- H(0 : w0, W) Q_W             (all rows above the window)
//   Z      Z(:, W)         <- Z(:, W) Q_W                  ("Q <- Q Q_1 ... Q_k")
// Windows of one step are disjoint, so their left updates touch disjoint rows and their right / Z
// updates disjoint columns.  The left and right updates of two different windows meet in blocks
// H(W_c, W_c') and are ordered (left kernel, then right kernel).
//
// Tensor-core path: FP64 mma.sync.m8n8k4 (SASS DMMA.8x8x4; tcgen05 has no f64 kind, SURVEY
// §7.3 H3).  Structure of Q_W: a band -- every bulge passing a row extends its support at most 2
// columns to the left and about s columns to the right -- so each 8-column block of Q_W has a short
// nonzero row range; the chase records it next to Q_W (store_q_slot) and the tile K loops skip the
// zero K steps (~30% fewer flops at k = 96).
//
// Main path (n even, "bulk" kernels): 8 consumer warps + 1 producer warp per CTA.  The producer
// streams panel tiles into a 2-stage SMEM ring with the bulk-copy (TMA) engine
// (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP): one 1-D copy per panel column, 16-byte
// aligned by starting at an even row.  Q_W (stored by the chase kernel in this SMEM layout) arrives
// in one shot per window.  Consumers wait on the stage's mbarrier, run the DMMA K loop, release the
// stage, then store the accumulators in place.  Generic path (n odd): same tiling, 8-byte cp.async.
// SMEM tiles use a leading dimension = 4 (mod 16) doubles: conflict-free m8n8k4 fragment loads.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "device_common.cuh"
#include "gemm_tile.cuh"
#include "kernels.hpp"

namespace hqr {

namespace {

constexpr int kConsumerWarps = 8;
constexpr int kThreadsGeneric = 256;
constexpr int kThreadsBulk = 288;  // 8 consumer warps + 1 producer warp
constexpr int kMaxStepWindows = 128;

// per-CTA item decoder: the step's windows with their tile counts (prefix sums in SMEM)
struct StepItems {
  int64_t pre[kMaxStepWindows + 1];
  WindowDesc w[kMaxStepWindows];
  int64_t rt[kMaxStepWindows];  // right kernel: H row tiles per window
};

__device__ __forceinline__ int decode_item(const StepItems& si, int nw, int64_t it, int64_t& tile) {
  int i = 0;
  while (i + 1 < nw && si.pre[i + 1] <= it) ++i;
  tile = it - si.pre[i];
  return i;
}

// ================================================================================================
// TMA-path update kernel (n even).  LEFT:  out[KP x NT] = Q_W^T[KP x KP] * P[KP x NT],
//   P = H(W, c0 : c0+NT); A = Q_W^T with Qs[m*QLD + k] = Q[k + m*QLD] (the chase kernel's slot
//   layout, one 1-D bulk copy per window), B = panel, one 2-D TMA box {LDP rows, NT columns} at
//   (w0 - ro, c0), ro = w0 & 1 (TMA's innermost coordinate must be 16-byte aligned):
//   Ps[nn*LDP + ro + k] = H[(w0+k) + (c0+nn)*n]  (LDP >= KP + 1).
// RIGHT: out[MT x KP] = P[MT x KP] * Q_W[KP x KP], P = H(r0 : r0+MT, W) (rows above W) or
//   Z(r0 : r0+MT, W); A = panel, one TMA box {LDP rows, KP columns} at (r0, w0):
//   Ps[k*LDP + m] = M[(r0+m) + (w0+k)*n]; B = Qs[nn*QLD + k].
// LDP = 4 (mod 16) doubles makes the m8n8k4 fragment loads conflict-free; the box rows beyond the
// window / tile (other matrix rows, or TMA's zero fill outside the matrix) are multiplied by the
// zero padding of Q_W or land in output rows that are never stored.
//   Items of window i: ceil(w0/MT) tiles of H rows [0, w0) (right_mode != 2), then ceil(n/MT) tiles
//   of Z rows [0, n) (Z != nullptr and right_mode != 1).
// Warp roles: warp 8 = producer (TMA), warps 0-3 = consumer group 0, warps 4-7 = group 1.
// The groups ping-pong: group q computes the CTA's items j = q (mod 2) out of the SMEM ring
// (item j in stage j mod NS, NS = 3 for KP <= 96), so one group's epilogue (register -> HBM
// stores) overlaps the other group's DMMA main loop, and the next item of a group is already
// loading while its previous one is multiplied.  Inside a
// group, 2 x 2 warps tile the output (gemm_tile.cuh); each 8-column block of Q_W multiplies only
// its recorded K extent.
// ================================================================================================
template <int KP, bool LEFT>
__global__ void __launch_bounds__(kThreadsBulk, 1)
    bulk_update_kernel(StepArgs a, int64_t total_items, const __grid_constant__ CUtensorMap tmH,
                       const __grid_constant__ CUtensorMap tmZ) {
  using G = Geom<KP, LEFT>;
  constexpr int NT = G::NT, MT = G::MT, QLD = G::QLD, STAGE = G::STAGE;
  constexpr int NS = stages_of(KP);
  extern __shared__ __align__(1024) double sm[];
  double* Qs = sm;                       // KP x QLD
  double* Ps = Qs + KP * QLD;            // NS stages (128-byte aligned: TMA destinations)
  __shared__ StepItems si;
  __shared__ __align__(8) uint64_t full[NS], empty[NS], qfull, qempty;
  __shared__ int seq[NS];  // item whose panel stage s holds (published by the producer)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n;
  const int nw = a.win_count;
  const int64_t ztiles = (!LEFT && a.Z && a.right_mode != 1) ? (a.zrows + MT - 1) / MT : 0;
  if (tid == 0) {
    si.pre[0] = 0;
    for (int i = 0; i < nw; ++i) {
      WindowDesc w = a.wins[a.win_begin + i];
      si.w[i] = w;
      if (LEFT) {
        int64_t c, cnt;
        left_range(a, w, c, cnt);
        si.rt[i] = c;  // LEFT: first column of the window's range
        si.pre[i + 1] = si.pre[i] + (cnt + NT - 1) / NT;
      } else {
        int64_t lo, hi;
        right_row_range(a, w, lo, hi);
        si.rt[i] = (a.right_mode == 2) ? 0 : (hi - lo + MT - 1) / MT;
        si.pre[i + 1] = si.pre[i] + si.rt[i] + ztiles;
      }
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    mbar_init(&qfull, 1);
    mbar_init(&qempty, kConsumerWarps);
    for (int s = 0; s < NS; ++s) seq[s] = -1;
  }
  for (int i = tid; i < NS * STAGE; i += kThreadsBulk) Ps[i] = 0.0;
  fence_proxy_async();
  __syncthreads();

  const int64_t G0 = gridDim.x;
  const int64_t it0 = total_items * blockIdx.x / G0, it1 = total_items * (blockIdx.x + 1) / G0;
  auto tile_ref = [&](int wi, int64_t tile) {
    const WindowDesc& w = si.w[wi];
    TileRef t;
    t.w0 = w.w0; t.kw = w.w1 - w.w0 + 1; t.nbc = w.nbc;
    if (LEFT) {
      t.M = a.H; t.c0 = si.rt[wi] + tile * NT; t.lc1 = a.lc1; t.ld = n; t.cb = a.hcol0; t.isZ = false;
      t.r0 = t.r1 = 0; t.lcs = si.rt[wi];
    } else if (tile < si.rt[wi]) {
      int64_t lo, hi;
      right_row_range(a, w, lo, hi);
      t.M = a.H; t.r0 = lo + tile * MT; t.r1 = hi; t.ld = n; t.cb = a.hcol0; t.isZ = false;
      t.c0 = t.lc1 = 0;
    } else {
      t.M = a.Z; t.r0 = (tile - si.rt[wi]) * MT; t.r1 = a.zrows; t.ld = a.ldz; t.cb = 0; t.isZ = true;
      t.c0 = t.lc1 = 0;
    }
    return t;
  };

  if (warp == kConsumerWarps) {
    // ---------------- producer warp: TMA ----------------
    int cur = -1;
    unsigned nq = 0;
    for (int64_t it = it0; it < it1; ++it) {
      int64_t tile;
      const int wi = decode_item(si, nw, it, tile);
      const WindowDesc& w = si.w[wi];
      if (wi != cur) {
        // producer waits: lane 0 alone (a lane that saw the phase may publish before its siblings
        // poll again, and the barrier could then complete another phase)
        if (cur >= 0 && lane == 0) mbar_wait(&qempty, (nq - 1) & 1);  // both groups done with Q_W
        __syncwarp();
        const double* Q = a.qslots + (size_t)(w.slot + a.slot_offset) * KP * QLD;
        constexpr unsigned qbytes = KP * QLD * 8, chunk = qbytes / 32;
        if (lane == 0) mbar_arrive_tx(&qfull, qbytes);
        __syncwarp();
        bulk_g2s(reinterpret_cast<char*>(Qs) + lane * chunk, reinterpret_cast<const char*>(Q) + lane * chunk,
                 chunk, &qfull);
        cur = wi;
        ++nq;
      }
      const int64_t j = it - it0;
      const int s = (int)(j % NS);
      if (j >= NS && lane == 0) mbar_wait(&empty[s], (unsigned)((j / NS) - 1) & 1);
      __syncwarp();
      if (lane == 0) {
        *reinterpret_cast<volatile int*>(&seq[s]) = (int)j;
        produce_tile<KP, LEFT>(Ps + s * STAGE, &full[s], &tmH, &tmZ, tile_ref(wi, tile));
      }
      __syncwarp();
    }
  } else {
    // ---------------- consumer groups: group q takes items j = q (mod 2) ----------------
    const int q = warp >> 2, i4 = warp & 3;
    int cur = -1;
    unsigned nq = 0;
    for (int64_t it = it0; it < it1; ++it) {
      int64_t tile;
      const int wi = decode_item(si, nw, it, tile);
      if (wi != cur) {
        if (cur >= 0) {  // this group has finished all its tiles of the previous window
          __syncwarp();
          if (lane == 0) mbar_arrive(&qempty);
        }
        mbar_wait(&qfull, nq & 1);
        cur = wi;
        ++nq;
      }
      const int64_t j = it - it0;
      if ((int)(j & 1) != q) continue;
      const int s = (int)(j % NS);
      // the stage's previous phase belongs to the other group and may still be in flight (a parity
      // wait cannot tell phase p from p - 2): wait until the producer has published item j first
      while (*reinterpret_cast<volatile int*>(&seq[s]) != (int)j) {
      }
      mbar_wait(&full[s], (unsigned)(j / NS) & 1);
      // quarters: the two warps of an SM sub-partition (groups 0, 1) take opposite quarters
      consume_tile<KP, LEFT>(Qs, Ps + s * STAGE, &empty[s], tile_ref(wi, tile), (i4 + 2 * q) & 3, lane);
    }
  }
}

// ================================================================================================
// Generic path (odd n: columns are not 16-byte aligned): 8 warps, 8-byte cp.async double buffer.
// ================================================================================================
template <int KP>
__global__ void __launch_bounds__(kThreadsGeneric, 1) left_generic_kernel(StepArgs a, int64_t total_items) {
  constexpr int NT = gen_left_cols(KP);
  constexpr int QLD = pad_ld(KP);
  constexpr int LD = pad_ld(KP);
  constexpr int WM = KP / 4, WN = NT / 2;
  constexpr int FM = WM / 8, FN = WN / 8;
  extern __shared__ __align__(1024) double sm[];
  double* As = sm;                    // KP x QLD
  double* Bs = As + KP * QLD;         // 2 x NT x LD
  __shared__ StepItems si;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp & 3) * WM, wn0 = (warp >> 2) * WN;
  const int64_t n = a.n;
  const int nw = a.win_count;
  if (tid == 0) {
    si.pre[0] = 0;
    for (int i = 0; i < nw; ++i) {
      WindowDesc w = a.wins[a.win_begin + i];
      si.w[i] = w;
      int64_t c, cnt;
      left_range(a, w, c, cnt);
      si.rt[i] = c;
      si.pre[i + 1] = si.pre[i] + (cnt + NT - 1) / NT;
    }
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  const int64_t it0 = total_items * blockIdx.x / G, it1 = total_items * (blockIdx.x + 1) / G;
  auto load_panel = [&](int wi, int64_t tile, int buf) {
    const WindowDesc& w = si.w[wi];
    const int kw = w.w1 - w.w0 + 1;
    const int64_t c0 = si.rt[wi] + tile * NT;
    double* B = Bs + buf * NT * LD;
    for (int f = tid; f < NT * KP; f += kThreadsGeneric) {
      int nn = f / KP, k = f - nn * KP;
      int64_t col = c0 + nn;
      bool ok = (k < kw) && (col < a.lc1);
      cp_async8(B + nn * LD + k, ok ? a.H + (w.w0 + k) + (col - a.hcol0) * n : a.H, ok);
    }
  };
  auto load_q = [&](int wi) {
    const double* Q = a.qslots + (size_t)(si.w[wi].slot + a.slot_offset) * KP * QLD;
    for (int f = tid; f < KP * QLD; f += kThreadsGeneric) cp_async8(As + f, Q + f, true);
  };
  int cur = -1, buf = 0;
  bool pref = false;
  for (int64_t it = it0; it < it1; ++it) {
    int64_t tile;
    const int wi = decode_item(si, nw, it, tile);
    if (wi != cur) {
      cp_async_wait<0>();
      __syncthreads();
      load_q(wi);
      load_panel(wi, tile, buf);
      cp_async_commit();
      cur = wi;
    } else if (!pref) {
      load_panel(wi, tile, buf);
      cp_async_commit();
    }
    pref = false;
    if (it + 1 < it1) {
      int64_t tile2;
      const int wi2 = decode_item(si, nw, it + 1, tile2);
      if (wi2 == wi) {
        load_panel(wi2, tile2, buf ^ 1);
        cp_async_commit();
        pref = true;
      }
    }
    if (pref) cp_async_wait<1>(); else cp_async_wait<0>();
    __syncthreads();
    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* B = Bs + buf * NT * LD;
    const int lr = lane >> 2, lk = lane & 3;
#pragma unroll 4
    for (int kk = 0; kk < KP; kk += 4) {
      double fa[FM], fb[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) fa[i] = As[(wm0 + 8 * i + lr) * QLD + kk + lk];
#pragma unroll
      for (int j = 0; j < FN; ++j) fb[j] = B[(wn0 + 8 * j + lr) * LD + kk + lk];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j], fa[i], fb[j]);
    }
    const WindowDesc& w = si.w[wi];
    const int kw = w.w1 - w.w0 + 1;
    const int64_t c0 = si.rt[wi] + tile * NT;
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int m = wm0 + 8 * i + lr;
      if (m >= kw) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t col = c0 + wn0 + 8 * j + 2 * lk + e;
          if (col < a.lc1) a.H[(w.w0 + m) + (col - a.hcol0) * n] = acc[i][j][e];
        }
    }
    __syncthreads();
    buf ^= 1;
  }
}

template <int KP>
__global__ void __launch_bounds__(kThreadsGeneric, 1) right_generic_kernel(StepArgs a, int64_t total_items) {
  constexpr int MT = gen_right_rows(KP);
  constexpr int QLD = pad_ld(KP);
  constexpr int LDP = pad_ld(MT);
  constexpr int WM = MT / 2, WN = KP / 4;
  constexpr int FM = WM / 8, FN = WN / 8;
  extern __shared__ __align__(1024) double sm[];
  double* Bs = sm;                    // Q: KP(n) x QLD
  double* As = Bs + KP * QLD;         // 2 x KP(k) x LDP
  __shared__ StepItems si;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp & 1) * WM, wn0 = (warp >> 1) * WN;
  const int64_t n = a.n;
  const int nw = a.win_count;
  const int64_t ztiles = (a.Z && a.right_mode != 1) ? (a.zrows + MT - 1) / MT : 0;
  if (tid == 0) {
    si.pre[0] = 0;
    for (int i = 0; i < nw; ++i) {
      WindowDesc w = a.wins[a.win_begin + i];
      si.w[i] = w;
      int64_t lo, hi;
      right_row_range(a, w, lo, hi);
      si.rt[i] = (a.right_mode == 2) ? 0 : (hi - lo + MT - 1) / MT;
      si.pre[i + 1] = si.pre[i] + si.rt[i] + ztiles;
    }
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  const int64_t it0 = total_items * blockIdx.x / G, it1 = total_items * (blockIdx.x + 1) / G;
  auto panel = [&](int wi, int64_t tile, double*& M, int64_t& r0, int64_t& r1, int64_t& ld,
                   int64_t& cb) {
    if (tile < si.rt[wi]) {
      int64_t lo, hi;
      right_row_range(a, si.w[wi], lo, hi);
      M = a.H; r0 = lo + tile * MT; r1 = hi; ld = n; cb = a.hcol0;
    } else {
      M = a.Z; r0 = (tile - si.rt[wi]) * MT; r1 = a.zrows; ld = a.ldz; cb = 0;
    }
  };
  auto load_panel = [&](int wi, int64_t tile, int buf) {
    const WindowDesc& w = si.w[wi];
    const int kw = w.w1 - w.w0 + 1;
    double* M;
    int64_t r0, r1, ld, cb;
    panel(wi, tile, M, r0, r1, ld, cb);
    double* A = As + buf * KP * LDP;
    for (int f = tid; f < KP * MT; f += kThreadsGeneric) {
      int k = f / MT, mm = f - k * MT;
      int64_t row = r0 + mm;
      bool ok = (k < kw) && (row < r1);
      cp_async8(A + k * LDP + mm, ok ? M + row + (w.w0 + k - cb) * ld : M, ok);
    }
  };
  auto load_q = [&](int wi) {
    const double* Q = a.qslots + (size_t)(si.w[wi].slot + a.slot_offset) * KP * QLD;
    for (int f = tid; f < KP * QLD; f += kThreadsGeneric) cp_async8(Bs + f, Q + f, true);
  };
  int cur = -1, buf = 0;
  bool pref = false;
  for (int64_t it = it0; it < it1; ++it) {
    int64_t tile;
    const int wi = decode_item(si, nw, it, tile);
    if (wi != cur) {
      cp_async_wait<0>();
      __syncthreads();
      load_q(wi);
      load_panel(wi, tile, buf);
      cp_async_commit();
      cur = wi;
    } else if (!pref) {
      load_panel(wi, tile, buf);
      cp_async_commit();
    }
    pref = false;
    if (it + 1 < it1) {
      int64_t tile2;
      const int wi2 = decode_item(si, nw, it + 1, tile2);
      if (wi2 == wi) {
        load_panel(wi2, tile2, buf ^ 1);
        cp_async_commit();
        pref = true;
      }
    }
    if (pref) cp_async_wait<1>(); else cp_async_wait<0>();
    __syncthreads();
    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* A = As + buf * KP * LDP;
    const int lr = lane >> 2, lk = lane & 3;
#pragma unroll 4
    for (int kk = 0; kk < KP; kk += 4) {
      double fa[FM], fb[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) fa[i] = A[(kk + lk) * LDP + wm0 + 8 * i + lr];
#pragma unroll
      for (int j = 0; j < FN; ++j) fb[j] = Bs[(wn0 + 8 * j + lr) * QLD + kk + lk];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j], fa[i], fb[j]);
    }
    const WindowDesc& w = si.w[wi];
    const int kw = w.w1 - w.w0 + 1;
    double* M;
    int64_t r0, r1, ld, cb;
    panel(wi, tile, M, r0, r1, ld, cb);
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int64_t row = r0 + wm0 + 8 * i + lr;
      if (row >= r1) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wn0 + 8 * j + 2 * lk + e;
          if (col < kw) M[row + (w.w0 + col - cb) * ld] = acc[i][j][e];
        }
    }
    __syncthreads();
    buf ^= 1;
  }
}

// ---- launchers -------------------------------------------------------------------------------
template <int KP> constexpr size_t left_bulk_smem() {
  return (size_t)(KP * pad_ld(KP) + stages_of(KP) * left_cols(KP) * pad_ld(KP)) * sizeof(double);
}
template <int KP> constexpr size_t right_bulk_smem() {
  return (size_t)(KP * pad_ld(KP) + stages_of(KP) * KP * panel_ld(right_rows(KP))) * sizeof(double);
}
template <int KP> constexpr size_t left_generic_smem() {
  return (size_t)(KP * pad_ld(KP) + 2 * gen_left_cols(KP) * pad_ld(KP)) * sizeof(double);
}
template <int KP> constexpr size_t right_generic_smem() {
  return (size_t)(KP * pad_ld(KP) + 2 * KP * pad_ld(gen_right_rows(KP))) * sizeof(double);
}

template <typename K>
cudaError_t set_smem(K kern, size_t smem, bool& configured) {
  if (configured) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) configured = true;
  return e;
}

template <int KP, bool LEFT>
cudaError_t launch_t(const StepArgs& a, const TensorMaps& tm, int64_t items, int grid, cudaStream_t st) {
  if (tm.valid) {
    static bool c = false;
    const size_t smem = LEFT ? left_bulk_smem<KP>() : right_bulk_smem<KP>();
    cudaError_t e = set_smem(bulk_update_kernel<KP, LEFT>, smem, c);
    if (e != cudaSuccess) return e;
    bulk_update_kernel<KP, LEFT><<<grid, kThreadsBulk, smem, st>>>(a, items, LEFT ? tm.left_H : tm.right_H,
                                                                     tm.right_Z);
    return cudaGetLastError();
  }
  static bool c = false;
  if (LEFT) {
    cudaError_t e = set_smem(left_generic_kernel<KP>, left_generic_smem<KP>(), c);
    if (e != cudaSuccess) return e;
    left_generic_kernel<KP><<<grid, kThreadsGeneric, left_generic_smem<KP>(), st>>>(a, items);
  } else {
    cudaError_t e = set_smem(right_generic_kernel<KP>, right_generic_smem<KP>(), c);
    if (e != cudaSuccess) return e;
    right_generic_kernel<KP><<<grid, kThreadsGeneric, right_generic_smem<KP>(), st>>>(a, items);
  }
  return cudaGetLastError();
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

cudaError_t encode_2d(CUtensorMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld,
                      unsigned box_rows, unsigned box_cols) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) return cudaErrorNotSupported;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {box_rows, box_cols};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace

cudaError_t make_tensor_maps(TensorMaps* tm, const double* H, int64_t hcols, const double* Z,
                             int64_t zrows, int64_t ldz, int64_t n, int KP) {
  tm->valid = false;
  // TMA needs 16-byte aligned bases and leading dimensions (even n, even ldz)
  if ((n & 1) || n < 2 || n > (int64_t)1 << 31 || (reinterpret_cast<uintptr_t>(H) & 15) ||
      (Z && ((reinterpret_cast<uintptr_t>(Z) & 15) || (ldz & 1) || zrows < 1)))
    return cudaSuccess;  // generic (cp.async) path
  cudaError_t e = encode_2d(&tm->left_H, H, n, hcols, n, pad_ld(KP), left_cols(KP));
  if (e == cudaSuccess) e = encode_2d(&tm->right_H, H, n, hcols, n, panel_ld(right_rows(KP)), KP);
  if (e == cudaSuccess) e = Z ? encode_2d(&tm->right_Z, Z, zrows, n, ldz, panel_ld(right_rows(KP)), KP)
                              : encode_2d(&tm->right_Z, H, n, hcols, n, panel_ld(right_rows(KP)), KP);
  if (e != cudaSuccess) return e;
  tm->valid = true;
  return cudaSuccess;
}

cudaError_t launch_left(const StepArgs& a, const WindowDesc* hw, int num_sms, const TensorMaps& tm,
                        cudaStream_t st, int64_t* items_out, double* flops, double* bytes) {
  int64_t items = 0;
  double f = 0, b = 0;
  const int NT = tm.valid ? left_cols(a.KP) : gen_left_cols(a.KP);
  for (int i = 0; i < a.win_count; ++i) {
    int64_t c0, cols;
    left_range(a, hw[i], c0, cols);
    int64_t kw = hw[i].w1 - hw[i].w0 + 1;
    items += (cols + NT - 1) / NT;
    f += 2.0 * kw * kw * (double)cols;
    b += 16.0 * kw * (double)cols;
  }
  *items_out = items;
  *flops = f;
  *bytes = b;
  if (items == 0) return cudaSuccess;
  if (a.win_count > kMaxStepWindows) return cudaErrorInvalidValue;
  int grid = (int)std::min<int64_t>(items, num_sms);
  switch (a.KP) {
    case 32: return launch_t<32, true>(a, tm, items, grid, st);
    case 64: return launch_t<64, true>(a, tm, items, grid, st);
    case 96: return launch_t<96, true>(a, tm, items, grid, st);
    case 128: return launch_t<128, true>(a, tm, items, grid, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_right(const StepArgs& a, const WindowDesc* hw, int num_sms, const TensorMaps& tm,
                         cudaStream_t st, int64_t* items_out, double* flops, double* bytes) {
  int64_t items = 0;
  double f = 0, b = 0;
  const int MT = tm.valid ? right_rows(a.KP) : gen_right_rows(a.KP);
  const bool do_h = a.right_mode != 2, do_z = a.Z && a.right_mode != 1;
  const int64_t zt = do_z ? (a.zrows + MT - 1) / MT : 0;
  for (int i = 0; i < a.win_count; ++i) {
    int64_t kw = hw[i].w1 - hw[i].w0 + 1;
    int64_t lo, hi;
    right_row_range(a, hw[i], lo, hi);
    items += (do_h ? (hi - lo + MT - 1) / MT : 0) + zt;
    double rows = (do_h ? (double)(hi - lo) : 0.0) + (do_z ? (double)a.zrows : 0.0);
    f += 2.0 * kw * kw * rows;
    b += 16.0 * kw * rows;
  }
  *items_out = items;
  *flops = f;
  *bytes = b;
  if (items == 0) return cudaSuccess;
  if (a.win_count > kMaxStepWindows) return cudaErrorInvalidValue;
  int grid = (int)std::min<int64_t>(items, num_sms);
  switch (a.KP) {
    case 32: return launch_t<32, false>(a, tm, items, grid, st);
    case 64: return launch_t<64, false>(a, tm, items, grid, st);
    case 96: return launch_t<96, false>(a, tm, items, grid, st);
    case 128: return launch_t<128, false>(a, tm, items, grid, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hqr
