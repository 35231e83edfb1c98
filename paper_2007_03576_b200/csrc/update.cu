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
// §7.3 H3).  Each CTA (8 warps) keeps Q_W resident in SMEM for a contiguous run of tiles of the
// same window and double-buffers the panel tiles with cp.async, so the next panel streams from
// HBM while the current one is multiplied.  SMEM tiles use a leading dimension = 4 (mod 16)
// doubles, which makes the m8n8k4 fragment loads (lane -> row lane/4, k lane%4) conflict-free.
// Results go straight from the accumulator registers to HBM (in place: every output tile depends
// only on its own input panel tile).
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.hpp"

namespace hqr {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxStepWindows = 128;  // windows per step handled by the in-kernel item decoder

__host__ __device__ constexpr int pad_ld(int x) { return x + (((4 - x) % 16) + 16) % 16; }
// tile widths: 64 columns / rows, 32 when the 128-wide factor leaves too little SMEM for two panels
__host__ __device__ constexpr int left_cols(int KP) { return KP <= 96 ? 64 : 32; }
__host__ __device__ constexpr int right_rows(int KP) { return KP <= 96 ? 64 : 32; }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// per-CTA item decoder: the step's windows with their tile counts (prefix sums in SMEM)
struct StepItems {
  int nw;
  int64_t pre[kMaxStepWindows + 1];
};

// ----------------------------------------------------------------------------------------------
// Left update: out[KP x 64] = Q_W^T[KP x KP] * P[KP x 64], P = H(W, c0 : c0+64)
// A operand (Q^T) in SMEM as As[m][k] = Q[k + m*KP] (contiguous in k), B operand (panel) as
// Bs[n][k] = H[(w0+k) + (c0+n)*ld] (contiguous in k).  Warps: 4 (m) x 2 (n), warp tile KP/4 x 32.
// ----------------------------------------------------------------------------------------------
template <int KP>
__global__ void __launch_bounds__(kThreads, 1) left_kernel(StepArgs a, int64_t total_items) {
  constexpr int NT = left_cols(KP);
  constexpr int LD = pad_ld(KP);
  constexpr int WM = KP / 4, WN = NT / 2;
  constexpr int FM = WM / 8, FN = WN / 8;
  extern __shared__ double sm[];
  double* As = sm;                    // KP x LD
  double* Bs = As + KP * LD;          // 2 x NT x LD
  __shared__ StepItems si;
  __shared__ WindowDesc sw[kMaxStepWindows];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp & 3) * WM, wn0 = (warp >> 2) * WN;
  const int64_t n = a.n;

  if (tid == 0) {
    si.nw = a.win_count;
    si.pre[0] = 0;
    for (int i = 0; i < a.win_count; ++i) {
      WindowDesc w = a.wins[a.win_begin + i];
      sw[i] = w;
      int64_t cols = n - 1 - w.w1;
      si.pre[i + 1] = si.pre[i] + (cols + NT - 1) / NT;
    }
  }
  __syncthreads();

  const int64_t G = gridDim.x;
  const int64_t it0 = total_items * blockIdx.x / G, it1 = total_items * (blockIdx.x + 1) / G;
  auto decode = [&](int64_t it, int& wi, int64_t& tile) {
    int i = 0;
    while (si.pre[i + 1] <= it) ++i;
    wi = i;
    tile = it - si.pre[i];
  };
  auto load_panel = [&](int wi, int64_t tile, int buf) {
    const WindowDesc& w = sw[wi];
    const int kw = w.w1 - w.w0 + 1;
    const int64_t c0 = w.w1 + 1 + tile * NT;
    double* B = Bs + buf * NT * LD;
    for (int f = tid; f < NT * KP; f += kThreads) {
      int nn = f / KP, k = f - nn * KP;
      int64_t col = c0 + nn;
      bool ok = (k < kw) && (col < n);
      const double* g = ok ? a.H + (w.w0 + k) + col * n : a.H;
      cp_async8(B + nn * LD + k, g, ok);
    }
  };
  auto load_q = [&](int wi) {
    const double* Q = a.qslots + (size_t)sw[wi].slot * KP * KP;
    for (int f = tid; f < KP * KP; f += kThreads) {
      int m = f / KP, k = f - m * KP;
      cp_async8(As + m * LD + k, Q + f, true);
    }
  };

  int cur = -1, buf = 0;
  bool pref = false;
  for (int64_t it = it0; it < it1; ++it) {
    int wi;
    int64_t tile;
    decode(it, wi, tile);
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
      int wi2;
      int64_t tile2;
      decode(it + 1, wi2, tile2);
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
      for (int i = 0; i < FM; ++i) fa[i] = As[(wm0 + 8 * i + lr) * LD + kk + lk];
#pragma unroll
      for (int j = 0; j < FN; ++j) fb[j] = B[(wn0 + 8 * j + lr) * LD + kk + lk];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j], fa[i], fb[j]);
    }
    // store (in place)
    const WindowDesc& w = sw[wi];
    const int kw = w.w1 - w.w0 + 1;
    const int64_t c0 = w.w1 + 1 + tile * NT;
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int m = wm0 + 8 * i + lr;
      if (m >= kw) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t col = c0 + wn0 + 8 * j + 2 * lk + e;
          if (col < n) a.H[(w.w0 + m) + col * n] = acc[i][j][e];
        }
      }
    }
    __syncthreads();
    buf ^= 1;
  }
}

// ----------------------------------------------------------------------------------------------
// Right / Z update: out[64 x KP] = P[64 x KP] * Q_W[KP x KP], P = H(r0:r0+64, W) or Z(r0:r0+64, W)
// A operand (panel) in SMEM as As[k][m] = P[(r0+m) + (w0+k)*ld] (contiguous in m), B operand as
// Bs[n][k] = Q[k + n*KP] (contiguous in k).  Warps: 2 (m) x 4 (n), warp tile 32 x KP/4.
// Items of window i: ceil(w0/64) tiles of H rows [0, w0), then (Z != nullptr) ceil(n/64) tiles of
// Z rows [0, n).
// ----------------------------------------------------------------------------------------------
template <int KP>
__global__ void __launch_bounds__(kThreads, 1) right_kernel(StepArgs a, int64_t total_items) {
  constexpr int MT = right_rows(KP);
  constexpr int LDQ = pad_ld(KP);
  constexpr int LDP = pad_ld(MT);
  constexpr int WM = MT / 2, WN = KP / 4;
  constexpr int FM = WM / 8, FN = WN / 8;
  extern __shared__ double sm[];
  double* Bs = sm;                    // Q: KP(n) x LDQ
  double* As = Bs + KP * LDQ;         // 2 x KP(k) x LDP
  __shared__ StepItems si;
  __shared__ WindowDesc sw[kMaxStepWindows];
  __shared__ int64_t rtiles[kMaxStepWindows];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp & 1) * WM, wn0 = (warp >> 1) * WN;
  const int64_t n = a.n;
  const int64_t ztiles = a.Z ? (n + MT - 1) / MT : 0;

  if (tid == 0) {
    si.nw = a.win_count;
    si.pre[0] = 0;
    for (int i = 0; i < a.win_count; ++i) {
      WindowDesc w = a.wins[a.win_begin + i];
      sw[i] = w;
      rtiles[i] = ((int64_t)w.w0 + MT - 1) / MT;
      si.pre[i + 1] = si.pre[i] + rtiles[i] + ztiles;
    }
  }
  __syncthreads();

  const int64_t G = gridDim.x;
  const int64_t it0 = total_items * blockIdx.x / G, it1 = total_items * (blockIdx.x + 1) / G;
  auto decode = [&](int64_t it, int& wi, int64_t& tile) {
    int i = 0;
    while (si.pre[i + 1] <= it) ++i;
    wi = i;
    tile = it - si.pre[i];
  };
  // panel rows [r0, r1) of matrix M (H or Z)
  auto panel = [&](int wi, int64_t tile, double*& M, int64_t& r0, int64_t& r1) {
    if (tile < rtiles[wi]) {
      M = a.H; r0 = tile * MT; r1 = sw[wi].w0;
    } else {
      M = a.Z; r0 = (tile - rtiles[wi]) * MT; r1 = n;
    }
  };
  auto load_panel = [&](int wi, int64_t tile, int buf) {
    const WindowDesc& w = sw[wi];
    const int kw = w.w1 - w.w0 + 1;
    double* M; int64_t r0, r1;
    panel(wi, tile, M, r0, r1);
    double* A = As + buf * KP * LDP;
    for (int f = tid; f < KP * MT; f += kThreads) {
      int k = f / MT, mm = f - k * MT;
      int64_t row = r0 + mm;
      bool ok = (k < kw) && (row < r1);
      const double* g = ok ? M + row + (w.w0 + k) * n : M;
      cp_async8(A + k * LDP + mm, g, ok);
    }
  };
  auto load_q = [&](int wi) {
    const double* Q = a.qslots + (size_t)sw[wi].slot * KP * KP;
    for (int f = tid; f < KP * KP; f += kThreads) {
      int nn = f / KP, k = f - nn * KP;
      cp_async8(Bs + nn * LDQ + k, Q + f, true);
    }
  };

  int cur = -1, buf = 0;
  bool pref = false;
  for (int64_t it = it0; it < it1; ++it) {
    int wi;
    int64_t tile;
    decode(it, wi, tile);
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
      int wi2;
      int64_t tile2;
      decode(it + 1, wi2, tile2);
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
      for (int j = 0; j < FN; ++j) fb[j] = Bs[(wn0 + 8 * j + lr) * LDQ + kk + lk];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j], fa[i], fb[j]);
    }
    const WindowDesc& w = sw[wi];
    const int kw = w.w1 - w.w0 + 1;
    double* M; int64_t r0, r1;
    panel(wi, tile, M, r0, r1);
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int64_t row = r0 + wm0 + 8 * i + lr;
      if (row >= r1) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wn0 + 8 * j + 2 * lk + e;
          if (col < kw) M[row + (w.w0 + col) * n] = acc[i][j][e];
        }
      }
    }
    __syncthreads();
    buf ^= 1;
  }
}

template <int KP>
size_t left_smem() { return (size_t)(KP * pad_ld(KP) + 2 * left_cols(KP) * pad_ld(KP)) * sizeof(double); }
template <int KP>
size_t right_smem() { return (size_t)(KP * pad_ld(KP) + 2 * KP * pad_ld(right_rows(KP))) * sizeof(double); }

template <int KP>
cudaError_t launch_left_t(const StepArgs& a, int64_t items, int grid, cudaStream_t st) {
  static bool configured = false;
  size_t smem = left_smem<KP>();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(left_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  left_kernel<KP><<<grid, kThreads, smem, st>>>(a, items);
  return cudaGetLastError();
}

template <int KP>
cudaError_t launch_right_t(const StepArgs& a, int64_t items, int grid, cudaStream_t st) {
  static bool configured = false;
  size_t smem = right_smem<KP>();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(right_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  right_kernel<KP><<<grid, kThreads, smem, st>>>(a, items);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_left(const StepArgs& a, const WindowDesc* hw, int num_sms, cudaStream_t st,
                        int64_t* items_out, double* flops, double* bytes) {
  int64_t items = 0;
  double f = 0, b = 0;
  for (int i = 0; i < a.win_count; ++i) {
    int64_t cols = a.n - 1 - hw[i].w1;
    int64_t kw = hw[i].w1 - hw[i].w0 + 1;
    items += (cols + left_cols(a.KP) - 1) / left_cols(a.KP);
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
    case 32: return launch_left_t<32>(a, items, grid, st);
    case 64: return launch_left_t<64>(a, items, grid, st);
    case 96: return launch_left_t<96>(a, items, grid, st);
    case 128: return launch_left_t<128>(a, items, grid, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_right(const StepArgs& a, const WindowDesc* hw, int num_sms, cudaStream_t st,
                         int64_t* items_out, double* flops, double* bytes) {
  int64_t items = 0;
  double f = 0, b = 0;
  const int MT = right_rows(a.KP);
  const int64_t zt = a.Z ? (a.n + MT - 1) / MT : 0;
  for (int i = 0; i < a.win_count; ++i) {
    int64_t kw = hw[i].w1 - hw[i].w0 + 1;
    items += (hw[i].w0 + MT - 1) / MT + zt;
    double rows = (double)hw[i].w0 + (a.Z ? (double)a.n : 0.0);
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
    case 32: return launch_right_t<32>(a, items, grid, st);
    case 64: return launch_right_t<64>(a, items, grid, st);
    case 96: return launch_right_t<96>(a, items, grid, st);
    case 128: return launch_right_t<128>(a, items, grid, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hqr
