// kernels.hpp -- launch interface between the orchestration (hqr_api.cu) and the sm_100a kernels
// (chase.cu, update.cu).  Product path only; shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda.h>  // CUtensorMap (header only; the encoder is fetched through cudaGetDriverEntryPoint)
#include <cuda_runtime.h>

#include "plan.hpp"

namespace hqr {

// Schedule / debugging knobs read from the environment exist only in tuning builds
// (-DHQR_TUNING, never the product build): the product library's schedule is fixed.
inline const char* tuning_env(const char* name) {
#ifdef HQR_TUNING
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Arguments of one wavefront step (device pointers).
struct StepArgs {
  double* H;                 // this rank's H columns: global column j at H + (j - hcol0) * n (ld = n)
  double* Z;                 // this rank's Z rows [0, zrows) x n columns, ld = ldz; or nullptr
  int64_t n;
  int64_t hcol0;             // global index of local H column 0
  int64_t lc0, lc1;          // left update: global columns [lc0, lc1) held (and updated) here
  int64_t zrows, ldz;        // local Z rows and leading dimension
  int64_t ilo, ihi;
  const WindowDesc* wins;    // device copy of plan.windows
  int win_begin, win_count;  // this step's windows
  const double* coef;        // per bulge j: its shift pair coef[4j..4j+3] = (re_2j, re_2j+1,
                             // im_2j, im_2j+1); sigma / pi are formed in the chase (scaled, R15)
  double* qslots;            // Q slot s at qslots + s*KP*QLD: column-major, ld = QLD, zero padded
  int KP;                    // padded factor side (32, 64, 96 or 128)
  int QLD;                   // Q slot leading dimension = pad_ld(KP) (the update kernels' SMEM ld)
  int slot_offset;           // this step's Q slot set: window slot s lives at slot s + slot_offset
  int right_mode;            // right kernel: 0 = H rows above W and Z, 1 = H only, 2 = Z only
  int step;                  // wavefront step index (debug timing only)
  double* wstats;            // nullable: per plan window, the executed DMMA work units of its factor
                             // (record_band); wstats[win_begin + i] for window i of the step
  signed char* aftermath;    // nullable: per row, the subdiagonal scan flags (R16), written by the
                             // chases of windows with scan rows (WindowDesc::scan_lo/hi)
  int64_t rrow_lo, rrow_hi;  // right kernel, H rows: rrow_hi <= 0 -> [0, w0) (default); else
                             // [rrow_lo, min(rrow_hi, w0)), rrow_lo even (sharded near / far split)
};

// H rows [lo, hi) of window w's right update (update.cu; see StepArgs::rrow_lo / rrow_hi)
__host__ __device__ inline void right_row_range(const StepArgs& a, const WindowDesc& w, int64_t& lo,
                                                int64_t& hi) {
  lo = 0;
  hi = w.w0;
  if (a.rrow_hi > 0) {
    lo = a.rrow_lo;
    if (a.rrow_hi < hi) hi = a.rrow_hi;
  }
  if (hi < lo) hi = lo;
}

// One CTA per window: chase the step's bulges inside SMEM-resident windows, accumulate Q_W.
cudaError_t launch_chase(const StepArgs& a, int max_kw, int max_nbc, cudaStream_t st);
size_t chase_smem_bytes(int kw, int nbc);

// QZ (qz.cu): one CTA per window of the pair (H, T); Q_W to a.qslots, Z_W to zslots (same layout).
cudaError_t launch_qz_chase(const StepArgs& a, double* T, double* zslots, int max_kw, cudaStream_t st);
size_t qz_chase_smem_bytes(int kw);
// Largest window side of the QZ chase (H, T, Q_W, Z_W all SMEM-resident: 4 k (k|1) doubles)
constexpr int kMaxWindowQZ = 80;

// QR iteration pieces (qriter.cu): eigenvalues of a small Hessenberg block H(r0:r0+m, r0:r0+m)
// (one CTA, m <= small_eig_max(); *info = 0 or the number not found) and the deflation step.
int small_eig_max();
cudaError_t launch_small_eig(const double* H, int64_t n, int64_t r0, int m, double* wr, double* wi, int* info,
                             cudaStream_t st);
cudaError_t launch_deflate(double* H, int64_t n, int64_t lo, int64_t hi, int* count, cudaStream_t st);
// out[0] <- sum of squares of H[0 .. count)
cudaError_t launch_fro2(const double* H, int64_t count, double* out, int num_sms, cudaStream_t st);
// AED on the window [k0, k0+nw) (nw <= kMaxWindow) of the block starting at ilo (qriter.cu); U to
// uslot (KP x QLD Q slot), eigenvalues of the window to ew / ei, res = {nd, m}.
cudaError_t launch_aed(double* H, int64_t n, int64_t ilo, int64_t k0, int nw, double thr, double* uslot, int KP,
                       int QLD, double* ew, double* ei, int* res, cudaStream_t st);

// 2-D TMA descriptors of H and Z (column-major, n x n) with the update kernels' SMEM boxes.
// Valid only for even n (TMA global strides must be multiples of 16 bytes).
struct TensorMaps {
  CUtensorMap left_H;   // box {pad_ld(KP) rows, left_cols(KP) columns}
  CUtensorMap right_H;  // box {panel_ld(right_rows(KP)) rows, KP columns}
  CUtensorMap right_Z;
  bool valid = false;
};
// H: n x hcols (local columns incl. halo), ld n; Z: zrows x n, ld ldz (nullptr: no Z map).
cudaError_t make_tensor_maps(TensorMaps* tm, const double* H, int64_t hcols, const double* Z,
                             int64_t zrows, int64_t ldz, int64_t n, int KP);

// Off-diagonal updates of one step.  Left: H(W, w1+1:n) <- Q_W^T H(W, w1+1:n) for every window.
// Right (+Z): H(0:w0, W) <- H(0:w0, W) Q_W and Z(:, W) <- Z(:, W) Q_W.
// host_wins: the step's windows on the host (to size the grid).  Returns the number of items
// (tiles) through *items and the launch's GEMM flops through *flops.
cudaError_t launch_left(const StepArgs& a, const WindowDesc* host_wins, int num_sms,
                        const TensorMaps& tm, cudaStream_t st, int64_t* items, double* flops,
                        double* bytes);
cudaError_t launch_right(const StepArgs& a, const WindowDesc* host_wins, int num_sms,
                         const TensorMaps& tm, cudaStream_t st, int64_t* items, double* flops,
                         double* bytes);
// Left-update column range of window w on this rank: [c, c + cnt)
__host__ __device__ inline void left_range(const StepArgs& a, const WindowDesc& w, int64_t& c,
                                           int64_t& cnt) {
  c = (int64_t)w.w1 + 1 > a.lc0 ? (int64_t)w.w1 + 1 : a.lc0;
  cnt = a.lc1 - c;
  if (cnt < 0) cnt = 0;
}

// The fused kernel's left tiles start at the multiple of 8 at or below c (c_al): their boundaries then
// fall on the 8-column cells of the task dependency grid (hqr_api.cu build_task_deps), so two tiles of
// one window never share a cell -- with c itself as the origin, every window whose w1 + 1 is not a
// multiple of 8 (strides s = k - 3 nbc - 1 other than 56, or ilo not a multiple of 8) chained all its
// left tiles one after another.  The columns [c_al, c) are multiplied but not stored (TileRef::lcs).
// cnt counts from c_al (0 when the window has no columns right of it).
__host__ __device__ inline void left_range_al(const StepArgs& a, const WindowDesc& w, int64_t& c,
                                              int64_t& c_al, int64_t& cnt) {
  left_range(a, w, c, cnt);
  c_al = c & ~(int64_t)7;
  if (c_al < a.lc0) c_al = c;
  if (cnt > 0) cnt = a.lc1 - c_al;
}

// Q slot sets in flight: the Z update of step g may trail the chase of step g + kQSets - 1
constexpr int kQSets = 4;

// Largest window side whose chase fits in SMEM (H window + Q_W both resident).
constexpr int kMaxWindow = 112;

// Panel tile width (LEFT: H columns) / height (RIGHT: H or Z rows) of the TMA-path update tiles.
__host__ __device__ constexpr int left_cols(int KP) { return KP <= 64 ? 64 : 32; }
__host__ __device__ constexpr int right_rows(int KP) { return KP <= 64 ? 64 : 32; }

inline int padded_kp(int kw) { return kw <= 32 ? 32 : kw <= 64 ? 64 : kw <= 96 ? 96 : 128; }

// SMEM leading dimension = 4 (mod 16) doubles: conflict-free mma.m8n8k4 fragment loads
__host__ __device__ constexpr int pad_ld(int x) { return x + (((4 - x) % 16) + 16) % 16; }

}  // namespace hqr
