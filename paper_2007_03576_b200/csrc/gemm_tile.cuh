// gemm_tile.cuh -- one off-diagonal update tile on the FP64 tensor cores (mma.sync m8n8k4, SASS
// DMMA.8x8x4), shared by the per-step update kernels (update.cu) and the fused step kernel
// (step.cu).  Product path.
//
// LEFT  out[KP x NT] = Q_W^T[KP x KP] * P[KP x NT], P = H(W, c0 : c0+NT)
// RIGHT out[MT x KP] = P[MT x KP] * Q_W[KP x KP],  P = H(r0 : r0+MT, W) or Z(r0 : r0+MT, W)
// SMEM: Q_W resident as Qs[c*QLD + k] = Q_W[k][c] (the chase kernel's slot layout); the panel is one
// 2-D TMA box: LEFT Ps[nn*LDP + ro + k] = H[(w0+k) + (c0+nn)*n] (ro = w0 & 1: TMA's innermost
// coordinate must be 16-byte aligned), RIGHT Ps[k*LDP + m] = M[(r0+m) + (w0+k)*ld].  LDP = an odd
// multiple of 4 doubles makes the fragment loads conflict-free.  Box rows beyond the window / tile
// (other matrix rows, or TMA's zero fill outside the matrix) meet the zero padding of Q_W or land
// in output rows that are never stored.
// A consumer group = 4 warps, one quarter of the Q_W columns each (LEFT: output rows, RIGHT: output
// columns) times the whole other dimension; a warp multiplies only the K extent of its quarter (the
// band store_q_slot records next to Q_W).  Accumulators hold transposed output blocks so a thread
// owns two consecutive output rows of one column: 16-byte stores into column-major storage.
#pragma once
#include "device_common.cuh"

namespace hqr {

template <int KP, bool LEFT>
struct Geom {
  static constexpr int NT = left_cols(KP), MT = right_rows(KP);
  static constexpr int QLD = pad_ld(KP);
  static constexpr int LDP = LEFT ? pad_ld(KP) : panel_ld(MT);
  static constexpr int STAGE = LEFT ? NT * LDP : KP * LDP;        // doubles per SMEM stage
  static constexpr int OM = LEFT ? KP : MT, ON = LEFT ? NT : KP;  // output tile
  // warp tile: one quarter of the Q_W columns x the whole other output dimension
  static constexpr int WM = LEFT ? OM / 4 : OM;
  static constexpr int WN = LEFT ? ON : ON / 4;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static_assert(!LEFT || LDP >= KP + 1, "left panel box must hold the odd-row shift");
  static_assert((STAGE * 8) % 128 == 0 && (KP * QLD * 8) % 128 == 0, "TMA destinations 128-byte aligned");
};

// Where one tile lives.  LEFT: columns [c0, c0 + NT) of H, clipped at lc1.  RIGHT: rows [r0, r1)
// of M (H or Z), element (r, global column j) at M + r + (j - cb) * ld.
struct TileRef {
  int w0, kw, nbc;
  double* M;
  int64_t c0, lc1;   // LEFT
  int64_t lcs;       // LEFT: first column stored (columns [c0, lcs) are multiplied, not stored)
  int64_t r0, r1;    // RIGHT
  int64_t ld, cb;    // M's leading dimension and column base (LEFT: n, hcol0)
  bool isZ;
};

// Producer (one lane): arm the stage barrier with the box size and issue the TMA box load.
template <int KP, bool LEFT>
__device__ __forceinline__ void produce_tile(double* dst, uint64_t* full, const CUtensorMap* tmH,
                                             const CUtensorMap* tmZ, const TileRef& t) {
  using G = Geom<KP, LEFT>;
  mbar_arrive_tx(full, (unsigned)(G::STAGE * 8));  // TMA always lands the full box
  if (LEFT)
    tma_load_2d(dst, tmH, t.w0 & ~1, (int)(t.c0 - t.cb), full);
  else
    tma_load_2d(dst, t.isZ ? tmZ : tmH, (int)t.r0, (int)(t.w0 - t.cb), full);
}

// K steps [ks, ke) of one warp, multiplying only the Q_W column blocks F..L of its quarter (LEFT:
// fragment rows i, RIGHT: fragment columns jn); software-pipelined: the fragments of k-step k+4 are
// loaded before the DMMAs of step k.  The extents are multiples of 4 (store_q_slot).
template <int FM, int FN, bool LEFT, int F, int L>
__device__ __forceinline__ void kseg(double (&acc)[FN][FM][2], const double* A, int a_i, int a_k,
                                     const double* B, int b_j, int b_k, int ks, int ke) {
  constexpr int I0 = LEFT ? F : 0, I1 = LEFT ? L : FM - 1;
  constexpr int J0 = LEFT ? 0 : F, J1 = LEFT ? FN - 1 : L;
  double fa[2][FM], fb[2][FN];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int i = 0; i < FM; ++i) fa[h][i] = 0.0;
#pragma unroll
    for (int jn = 0; jn < FN; ++jn) fb[h][jn] = 0.0;
  }
  auto load = [&](int h, int k) {
#pragma unroll
    for (int i = I0; i <= I1; ++i) fa[h][i] = A[i * a_i + k * a_k];
#pragma unroll
    for (int jn = J0; jn <= J1; ++jn) fb[h][jn] = B[jn * b_j + k * b_k];
  };
  load(0, ks);
  // an odd k-step count peels one step; then branch-free pairs (a data-dependent exit inside the
  // pair made every pair a WARPSYNC + branch: tools/tile_ceiling.cu, in-tile executed DMMA rate
  // 31.9 -> 34.4 TF/s)
  auto mul = [&](int h) {
#pragma unroll
    for (int jn = J0; jn <= J1; ++jn)
#pragma unroll
      for (int i = I0; i <= I1; ++i) dmma(acc[jn][i], fb[h][jn], fa[h][i]);
  };
  int kk = ks;
  if ((ke - ks) & 4) {
    mul(0);
    kk += 4;
    if (kk < ke) load(0, kk);
  }
  for (; kk < ke; kk += 8) {
    load(1, kk + 4);
    mul(0);
    if (kk + 8 < ke) load(0, kk + 8);
    mul(1);
  }
}

// runtime (f, l) -> kseg<F, L> for every 0 <= F <= L < NB
template <int FM, int FN, bool LEFT, int NB, int F = 0, int L = 0>
__device__ __forceinline__ void kseg_dispatch(int f, int l, double (&acc)[FN][FM][2], const double* A, int a_i,
                                              int a_k, const double* B, int b_j, int b_k, int ks, int ke) {
  if constexpr (F < NB) {
    if constexpr (L < NB) {
      if (f == F && l == L) {
        kseg<FM, FN, LEFT, F, L>(acc, A, a_i, a_k, B, b_j, b_k, ks, ke);
        return;
      }
      kseg_dispatch<FM, FN, LEFT, NB, F, L + 1>(f, l, acc, A, a_i, a_k, B, b_j, b_k, ks, ke);
    } else {
      kseg_dispatch<FM, FN, LEFT, NB, F + 1, F + 1>(f, l, acc, A, a_i, a_k, B, b_j, b_k, ks, ke);
    }
  }
}

struct NoMid {
  __device__ void operator()() const {}
};

// One consumer warp: the output rows (LEFT) / columns (RIGHT) of Q_W column quarter `qq` (0..3)
// times the whole other tile dimension.  K loop over the stage `P` with Q_W in `Qs`, release the
// stage (`empty`), run `mid()`, store the tile in place.  Each 8-column block b of the quarter is
// multiplied only over its K extent [klo_b, khi_b) (store_q_slot's band extents): the K axis is cut
// at the extents' boundaries into segments with a fixed set of active blocks, each run by an
// unrolled loop over exactly those blocks (no predicated DMMAs).
template <int KP, bool LEFT, class Mid = NoMid>
__device__ __forceinline__ void consume_tile(const double* Qs, const double* P, uint64_t* empty,
                                             const TileRef& t, int qq, int lane, Mid mid = Mid()) {
  using G = Geom<KP, LEFT>;
  constexpr int FM = G::FM, FN = G::FN, WM = G::WM, WN = G::WN, QLD = G::QLD, LDP = G::LDP;
  constexpr int NB = LEFT ? FM : FN;  // Q_W column blocks of this warp
  (void)WM; (void)WN;
  const int qb0 = qq * NB;            // first Q_W column block
  const int lr = lane >> 2, lk = lane & 3;
  int lo[NB], hi[NB];
  int kbeg = KP, kend = 0;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
#ifdef HQR_BENCH_NO_TRIM  // benchmark-only knob (tools/gemm_bench.cu), never set in the product build
    lo[b] = 0; hi[b] = KP;
#else
    const double* meta = Qs + (size_t)(8 * (qb0 + b)) * QLD + KP;
    lo[b] = (int)meta[0];
    hi[b] = (int)meta[1];
#endif
    if (hi[b] > lo[b]) {
      kbeg = min(kbeg, lo[b]);
      kend = max(kend, hi[b]);
    } else {
      lo[b] = KP; hi[b] = 0;  // empty block: never active
    }
  }
  double acc[FN][FM][2];
#pragma unroll
  for (int jn = 0; jn < FN; ++jn)
#pragma unroll
    for (int i = 0; i < FM; ++i) acc[jn][i][0] = acc[jn][i][1] = 0.0;
  const double* A;
  const double* B;
  int a_i, a_k, b_j, b_k;
  if (LEFT) {
    A = Qs + (8 * qb0 + lr) * QLD + lk;             a_i = 8 * QLD; a_k = 1;
    B = P + lr * LDP + (t.w0 & 1) + lk;             b_j = 8 * LDP; b_k = 1;
  } else {
    A = P + lk * LDP + lr;                          a_i = 8;       a_k = LDP;
    B = Qs + (8 * qb0 + lr) * QLD + lk;             b_j = 8 * QLD; b_k = 1;
  }
  // K segments between consecutive block extent boundaries; in each, the active blocks form a
  // contiguous range [f, l] (the band: lo and hi grow with the block; a non-contiguous set would
  // be covered by its hull, whose extra blocks are zero there) and only they are multiplied
  for (int k = kbeg; k < kend;) {
    int f = NB, l = -1, nxt = kend;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (lo[b] <= k && k < hi[b]) {
        f = min(f, b);
        l = max(l, b);
      }
      if (lo[b] > k) nxt = min(nxt, lo[b]);
      if (hi[b] > k) nxt = min(nxt, hi[b]);
    }
    if (l >= f) kseg_dispatch<FM, FN, LEFT, NB>(f, l, acc, A, a_i, a_k, B, b_j, b_k, k, nxt);
    k = nxt;
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);
  mid();
#ifdef HQR_BENCH_NO_STORE  // benchmark-only knob (tools/gemm_bench.cu), never set in the product build
  if (acc[0][0][0] != 12345.678) return;
#endif
  // epilogue: thread (lr, lk) owns out[m = m0 + 8i + 2lk + {0,1}][n = n0 + 8jn + lr]
  if (LEFT) {
    const bool even = (t.w0 & 1) == 0;
#pragma unroll
    for (int jn = 0; jn < FN; ++jn) {
      const int64_t col = t.c0 + 8 * jn + lr;
      if (col < t.lcs || col >= t.lc1) continue;
      double* cp = t.M + (col - t.cb) * t.ld + t.w0;
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        const int m = 8 * (qb0 + i) + 2 * lk;
        if (even && m + 1 < t.kw) {
          *reinterpret_cast<double2*>(cp + m) = make_double2(acc[jn][i][0], acc[jn][i][1]);
        } else {
          if (m < t.kw) cp[m] = acc[jn][i][0];
          if (m + 1 < t.kw) cp[m + 1] = acc[jn][i][1];
        }
      }
    }
  } else {
#pragma unroll
    for (int jn = 0; jn < FN; ++jn) {
      const int col = 8 * (qb0 + jn) + lr;
      if (col >= t.kw) continue;
      double* cp = t.M + (t.w0 + col - t.cb) * t.ld;
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        const int64_t row = t.r0 + 8 * i + 2 * lk;  // even: 16-byte aligned pair
        if (row + 1 < t.r1) {
          *reinterpret_cast<double2*>(cp + row) = make_double2(acc[jn][i][0], acc[jn][i][1]);
        } else if (row < t.r1) {
          cp[row] = acc[jn][i][0];
        }
      }
    }
  }
}

}  // namespace hqr
