/*
 * hqr.h -- C ABI of the B200-native multishift QR sweep (libhqr_b200.so).
 *
 * The operation (PAPER.md = the paper's LaTeX body, cited as P:<line>):
 *   One small-bulge multishift QR sweep on an upper-Hessenberg fp64 matrix H with a given shift set:
 *     H <- Q^T H Q,  Z <- Z Q                                   (one QR iteration)
 *   where Q is the product of all 3x3 (final: 2x2) Householder reflectors of the nshifts/2
 *   tightly-coupled bulges introduced at the top of the active block [ilo, ihi] and chased to its
 *   bottom (P:198-206 double-shift step, P:227-233 tightly-coupled multi-shift chains with
 *   accumulated window factors and BLAS-3 off-diagonal updates, P:257-258 several chains,
 *   P:376-386 "push bulges", P:400-404 / P:452-453 left/right update tasks).
 *   Bulge j uses shifts (2j, 2j+1): the first column of (H - s I)(H - s' I) restricted to the block.
 *   The sweep is the exact (up to rounding order) result of nshifts/2 sequential Francis double
 *   steps (implicit-Q theorem); conventions are fixed in DESIGN.md "Readings" (R1-R12).
 *
 * Layout: H and Z are n x n IEEE binary64, column-major, leading dimension n (element (i,j) at
 * i + j*n).  Indices are 0-based.  Updates span the full matrix ("wantt": rows 0..ilo-1 and columns
 * ihi+1..n-1 of H are updated; all n rows of Z).
 *
 * Ownership: the caller owns H, Z and the shift arrays; the library modifies H and Z in place, never
 * frees or retains caller memory, and owns all workspace (device buffers, streams, events, CUDA
 * graphs) between hqr_setup and hqr_teardown.
 *
 * Return codes (LAPACK INFO style): 0 ok; -i argument i invalid (see hqr_sweep); 1000 + cudaError_t
 * on a CUDA runtime failure; 2000 + ncclResult_t on an NCCL failure; -100 library not set up;
 * -101 no CUDA device / unsupported device (the library never falls back to the CPU).
 */
#ifndef HQR_B200_H
#define HQR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hqr_config {
  int device;           /* CUDA device ordinal used by this process                              */
  int rank;             /* this process's rank, 0 <= rank < world                                */
  int world;            /* number of processes (one per GPU); 1 = single GPU                     */
  const void* nccl_id;  /* world > 1: 128-byte ncclUniqueId created by rank 0 and shared with all */
                        /* ranks (e.g. through torch.distributed); world == 1: NULL              */
  int64_t n_max;        /* largest n this setup will sweep (workspace hint; 0 = grow on demand)  */
  int flags;            /* bit 0: HQR_FLAG_NO_GRAPH -- launch kernels directly instead of         */
                        /*        replaying a captured CUDA graph                                 */
                        /* bit 1: HQR_FLAG_PROFILE  -- time every launch with CUDA events         */
                        /* bit 2: HQR_FLAG_NO_FUSE  -- separate chase / left / right launches     */
                        /*        instead of the fused step kernel                                */
                        /* bit 3: HQR_FLAG_NCCL_SELF -- world == 1 only: create a one-rank NCCL   */
                        /*        communicator, so hqr_sweep_dist runs its NCCL transport (the     */
                        /*        grouped broadcasts on the comm stream) on one GPU (tests)       */
  /* Shard boundaries (world > 1): NULL = the sqrt-balanced default of
   * hqr_dist_layout for every n.  Otherwise both arrays hold world + 1 entries for n = n_max:
   * col_bounds[r] .. col_bounds[r+1] are rank r's H columns, row_bounds[..] its Z rows; 0 = b[0] <
   * ... < b[world] = n_max, even, H shards >= HQR_MAX_WINDOW + 8 columns (else hqr_setup returns -1;
   * a sweep with another n returns -11).  The arrays are copied; the caller keeps ownership. */
  const int64_t* col_bounds;
  const int64_t* row_bounds;
  int window_max;       /* largest window side this setup will use (0 = HQR_MAX_WINDOW; must be   */
                        /* <= HQR_MAX_WINDOW, else -1): the effective side is min(window, N,      */
                        /* window_max)                                                            */
} hqr_config;

#define HQR_FLAG_NO_GRAPH 1
#define HQR_FLAG_PROFILE 2
#define HQR_FLAG_NO_FUSE 4
#define HQR_FLAG_NCCL_SELF 8

/* Initialise the library on cfg->device: streams, events, workspace, NCCL communicator (world > 1).
 * Returns 0, -1 (cfg NULL or inconsistent rank/world/nccl_id/bounds/window_max), -101 (no usable
 * sm_100 device), 1000+cudaError_t, 2000+ncclResult_t.  Calling it again re-initialises (tears
 * down first). */
int hqr_setup(const hqr_config* cfg);

/*
 * One multishift QR sweep, in place.  Synchronous: returns after the device has finished.
 *   H         [in,out] n x n column-major; device pointer, or host pointer (pinned or pageable, in
 *                      which case the library stages it through its own device memory and the
 *                      host<->device copies are part of the call).  Must be upper Hessenberg (zero
 *                      below the first subdiagonal; a host H is uploaded by row chunks from the
 *                      subdiagonal on, and entries below it may come back as zeros) with
 *                      H[ilo, ilo-1] == 0 (ilo > 0) and H[ihi+1, ihi] == 0 (ihi < n-1).
 *   Z         [in,out] n x n column-major (device or host), or NULL to skip Z <- Z Q.
 *   n         matrix order, n >= 1
 *   ilo, ihi  active block [ilo, ihi], 0 <= ilo <= ihi < n, N = ihi - ilo + 1 >= 3
 *   shifts_re, shifts_im  [in] host arrays of nshifts doubles; consecutive pairs (2j, 2j+1) form bulge
 *                      j; a non-real shift must be followed by its exact conjugate; real pairs are
 *                      any two reals.
 *   nshifts   even, 2 <= nshifts <= N
 *   window    diagonal-window side k (performance knob only; never changes the mathematical result):
 *             the effective side is min(window, N, window_max); window <= 0 is -9; a window
 *             smaller than the block must be >= 8 (-9); window >= N is accepted and means one
 *             window holding the whole block (SURVEY §8(b) lists "> N" as -9; we accept it
 *             because N < 8 blocks -- valid sweeps -- have no other legal window; R5).
 * Returns 0 or: -1 H NULL; -3 n < 1; -4 ilo < 0 or ilo > ihi; -5 ihi >= n or N < 3;
 *   -6 non-finite shift; -7 conjugate partner not exact / mixed real-complex pair;
 *   -8 nshifts odd, < 2 or > N; -9 window out of range; -10 block not decoupled
 *   (H[ilo,ilo-1] != 0 or H[ihi+1,ihi] != 0); -100 not set up; 1000+cudaError_t; 2000+ncclResult_t.
 * Matrix entries are assumed finite (no NaN/Inf scan).  Entry: the library's stream waits for work
 * queued on the legacy default stream (so H / Z writes issued there before the call are seen).
 * With world > 1 (hqr_setup) it is a collective called by every rank with identical scalars and
 * shifts, H and Z being this rank's LOCAL shards in the hqr_dist_layout layout (exactly
 * hqr_sweep_dist; host pointers are not accepted there).
 */
int hqr_sweep(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, const double* shifts_re,
              const double* shifts_im, int nshifts, int window);

/*
 * One sweep over several decoupled active blocks at once (concurrent processing
 * of independent unreduced blocks; BASELINE configs[4]).  Block i is [ilo[i], ihi[i]] with
 * nshifts[i] shifts, taken consecutively from shifts_re / shifts_im (block 0 first).  Blocks must be
 * ascending and disjoint (ihi[i] < ilo[i+1]) and each decoupled from its neighbours.  The result
 * equals sweeping the blocks one after another (their similarities commute); all blocks' windows
 * share each wavefront step.  Codes as hqr_sweep, with -4 also for nblocks < 1, NULL block arrays,
 * or overlapping / unsorted blocks.
 */
int hqr_sweep_multi(double* H, double* Z, int64_t n, int nblocks, const int64_t* ilo,
                    const int64_t* ihi, const double* shifts_re, const double* shifts_im,
                    const int* nshifts, int window);

/*
 * Several sweeps of one active block, overlapped ("two
 * bulge chasing steps can be overlapped"): sweep i uses nshifts[i] shifts, taken
 * consecutively from shifts_re / shifts_im (sweep 0 first), and is applied after sweep i-1 -- the
 * result is hqr_sweep called nsweeps times in order.  The shift sets are inputs here (known up
 * front), so sweep i+1's bulge chains enter the wavefront right behind sweep i's last chain and
 * its introduction and chase run while sweep i's right / Z updates drain.  Single GPU.  Codes as
 * hqr_sweep (each sweep's shifts validated as there), -8 also for nsweeps < 1 or nshifts NULL,
 * -1 after a world > 1 setup.
 */
int hqr_sweeps(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, int nsweeps,
               const double* shifts_re, const double* shifts_im, const int* nshifts, int window);

/*
 * Generalized (QZ) multishift sweep (PAPER.md P:208-213 the double-shift QZ
 * step, P:412-439 push bulges on a Hessenberg-triangular pair): (H, T) <- Q_s^T (H, T) Z_s,
 * Q <- Q Q_s, Z <- Z Z_s, where the sweep is the product of nshifts/2 double-shift QZ steps (pair 0
 * first): bulge vector (H T^-1 - s I)(H T^-1 - s' I) e1 (R17), left Householder
 * reflectors from H's columns, right-hand side reflectors from T's rows restoring T's triangular
 * form (R18).  H is upper Hessenberg, T upper triangular with T[ilo,ilo], T[ilo+1,ilo+1] != 0 (no
 * infinite eigenvalues at the top; the paper's push-infinities task is out of scope), both n x n
 * column-major on the DEVICE (host pointers: -1).  Q, Z: n x n device or NULL (skip).  Window side
 * min(window, N, HQR_MAX_WINDOW_QZ).  Single GPU.  Codes as hqr_sweep, plus -2 (T NULL, or a zero
 * leading diagonal entry of T in the block).
 */
int hqr_qz_sweep(double* H, double* T, double* Q, double* Z, int64_t n, int64_t ilo, int64_t ihi,
                 const double* shifts_re, const double* shifts_im, int nshifts, int window);
#define HQR_MAX_WINDOW_QZ 80

/*
 * QR iteration around the sweep (PAPER.md P:270-297 AED and shifts, P:370-381,
 * P:1142-1189 deflation; R21 / R22): repeatedly take the bottom unreduced block [l, hi] of
 * [ilo, ihi] (h(l, l-1) = 0) and
 *   (a) if it has at most nmin rows, compute its eigenvalues with the one-CTA Francis double-shift QR
 *       solver and continue above it;
 *   (b) aed_window > 0: aggressive early deflation on its trailing min(aed_window, N) window -- real
 *       Schur form of the window (U accumulated), spike s U(0,:), deflation from the bottom of the
 *       blocks whose spike entries are <= u ||H||_F (the paper's default norm-stable condition, R22),
 *       each failed block moved above the blocks not yet evaluated (R23), Hessenberg re-reduction,
 *       U propagated to the rest of H and to Z by the DMMA update kernels (hqr_aed); more than 14%
 *       deflated -> next round at once;
 *   (c) sweep the block (hqr_sweep's fused path, window `window`) with up to nshifts shifts: the
 *       bottom-most failed AED candidates (aed_window > 0) or the eigenvalues of the trailing
 *       nshifts x nshifts block (aed_window == 0, R21), complex pairs first, reals paired; then set
 *       every |h(k,k-1)| <= 2^-52 (|h(k-1,k-1)| + |h(k,k)|) to zero.
 * H, Z (Z may be NULL) are n x n device matrices changed only by orthogonal similarities, so on
 * return Z^T H0 Z = H (Z0 = I) with H reduced to blocks of at most nmin rows.  wr, wi: host arrays of
 * n doubles receiving the eigenvalues of rows ilo..ihi (conjugate pairs adjacent).  *sweeps_out
 * (nullable): sweeps run.  Returns 0; > 0 = ihi' + 1 when max_sweeps was reached with rows ilo..ihi'
 * unfinished (LAPACK INFO style); -1 H NULL / host pointer / world > 1; -3 n; -4 ilo; -5 ihi; -6
 * nshifts odd, < 2 or > 128; -7 window < 1; -8 nmin < 2 or > 128; -9 aed_window 1, < 0 or >
 * HQR_MAX_WINDOW; -10 wr / wi NULL; -100 not set up; 1000+cudaError_t.  After the call hqr_get_stats
 * reports launches_chase = AED steps and window_eff = eigenvalues deflated by AED.
 */
int hqr_qr_iterate(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, int nshifts, int window,
                   int nmin, int aed_window, int max_sweeps, double* wr, double* wi, int* sweeps_out);

/*
 * One aggressive-early-deflation step (the AED window, its Schur form, the spike,
 * the deflation check, the reordering of failed candidates "above the remaining unevaluated diagonal
 * blocks" P:289-290, the Hessenberg reduction of the remaining spike P:292; the norm-stable deflation
 * condition P:1142-1189; failed swaps halt the reordering P:893-894; R22 / R23) on
 * the window W = H(k0 : k0+nw, k0 : k0+nw) of the n x n device matrix H (column-major, ld n), where
 * rows k0 .. k0+nw-1 are the trailing rows of an unreduced block starting at row ilo (the caller
 * guarantees h(k0+nw, k0+nw-1) = 0 or k0 + nw = n; s = h(k0, k0-1), 0 when k0 = ilo):
 *   T = U^T W U real Schur form (Francis double-shift QR in one CTA); from the bottom, a 1x1 / 2x2
 *   block of T deflates when every spike entry s U(0, j) of its rows is <= thr (thr is the caller's
 *   threshold, e.g. 2^-53 ||H||_F); a failed block is moved to the top of the not-yet-evaluated
 *   blocks by swaps of adjacent diagonal blocks (Sylvester equation + QR, rejected when too
 *   ill-conditioned, which ends the check); when nd > 0 blocks deflated: the remaining spike is
 *   reflected onto e1, T(0:m, 0:m) reduced to Hessenberg form, T and the spike column (beta, 0, ..)
 *   written into H, H(window, k0+nw:) <- U^T H(..), H(0:k0, window) <- H(..) U, Z(:, window) <- Z U.
 *   When nd = 0, H and Z are unchanged.
 * Z may be NULL.  ew, ei: host arrays of nw doubles receiving the eigenvalues of the final blocks in
 * window order -- [0, m) the undeflated candidates (the next sweep's shifts), [m, nw) the deflated
 * eigenvalues of rows k0+m .. k0+nw-1.  *nd_out = nw - m deflated (-1: the Schur iteration did not
 * converge, nothing changed), *nund_out = m.  Returns 0; -1 H NULL / host pointer / world > 1; -3 n;
 * -4 ilo / k0 / nw outside H; -9 nw < 2 or > HQR_MAX_WINDOW; -10 an output pointer NULL; -100 not set
 * up; 1000+cudaError_t.  Synchronous on return.
 */
int hqr_aed(double* H, double* Z, int64_t n, int64_t ilo, int64_t k0, int nw, double thr, double* ew,
            double* ei, int* nd_out, int* nund_out);

/*
 * ---- Sharded sweep over several GPUs -------------------------------------------
 * Layout for `world` ranks (one process per GPU): rank r owns H columns [cb[r], cb[r+1]) -- all n
 * rows, column-major, ld = n -- and must allocate `halo` further columns after them (work space for
 * a neighbour's lent columns), and owns Z rows [rb[r], rb[r+1]) -- all n columns, column-major,
 * ld = rb[r+1] - rb[r].  cb[r] = n sqrt(r / world) and rb[r] = n r / world, rounded down to even.
 * hqr_dist_layout writes cb[0..world], rb[0..world], halo (any pointer may be NULL).  Returns 0,
 * -1 (n < 1), -2 (world < 1) or -11 (a shard would be narrower than HQR_MAX_WINDOW + 8 columns).
 */
int hqr_dist_layout(int64_t n, int world, int64_t* col_bounds, int64_t* row_bounds, int* halo);

/* Host-only: per wavefront step, what rank `rank` does (for tests).  out[6*s .. 6*s+5] =
 * {step, lend_out, lend_in, lc0, lc1, n_owned_windows}.  Returns 0, the number of steps when out is
 * NULL or cap < steps, or the negative codes of hqr_sweep / hqr_dist_layout (-7: bad rank). */
int hqr_dist_query(int64_t n, int64_t ilo, int64_t ihi, int nshifts, int window, int world,
                   int rank, int64_t* out, int64_t cap);

/* 128-byte ncclUniqueId for hqr_config.nccl_id (call on rank 0, share the bytes). */
int hqr_nccl_unique_id(void* out);

/*
 * Collective: one sweep of the distributed matrix (every rank calls it with identical scalars and
 * shifts after hqr_setup with world > 1).  H_local / Z_local: this rank's device shards in the
 * hqr_dist_layout layout (Z_local may be NULL).  Each window's factor is broadcast from the rank
 * owning its first column (ncclBroadcast over NVLink); a window straddling a shard boundary borrows
 * the neighbour's leading columns for the step (ncclSend/Recv).  Codes as hqr_sweep plus -11.
 */
int hqr_sweep_dist(double* H_local, double* Z_local, int64_t n, int64_t ilo, int64_t ihi,
                   const double* shifts_re, const double* shifts_im, int nshifts, int window);

/* hqr_sweep_dist over several decoupled blocks (as hqr_sweep_multi; BASELINE configs[4] sharded):
 * every block's windows share the wavefront steps and the shard roles.  Codes as hqr_sweep_multi
 * plus -11. */
int hqr_sweep_dist_multi(double* H_local, double* Z_local, int64_t n, int nblocks, const int64_t* ilo,
                         const int64_t* ihi, const double* shifts_re, const double* shifts_im,
                         const int* nshifts, int window);

/*
 * The sharded algorithm with `vworld` virtual ranks on this one GPU (test / single-GPU check of the
 * multi-GPU path): H, Z are full device matrices (as in hqr_sweep); the library scatters them into
 * per-rank shards, runs exactly the per-rank kernel sequence of hqr_sweep_dist with device copies
 * in place of NCCL transfers, and gathers the result.  Codes as hqr_sweep plus -10 (vworld < 1)
 * and -11.
 */
int hqr_sweep_virtual(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi,
                      const double* shifts_re, const double* shifts_im, int nshifts, int window,
                      int vworld);

/*
 * Aftermath vector of the last successful single-GPU sweep (hqr_sweep / hqr_sweep_multi /
 * hqr_sweeps: the push-bulges tasks of the last bulge
 * chain scan the subdiagonal for blocks decoupled during the sweep).  Check only: H is not
 * modified.  flags[i] (host array of n int8) for row i:
 *    2  h(i+1, i) == 0 exactly (decoupled)
 *    1  0 < |h(i+1, i)| <= 2^-52 (|h(i,i)| + |h(i+1,i+1)|)  (negligible: deflatable)
 *    0  otherwise
 *   -1  not scanned (outside [ilo-1, ihi] of every active block, or i = n-1)
 * computed by the chases of each block's last (topmost) chain from the final entries.
 * Returns 0, -1 (flags NULL), -3 (n differs from the last sweep's n), -100 (no sweep yet).
 */
int hqr_get_aftermath(signed char* flags, int64_t n);

/* hqr_sweep_virtual over several decoupled blocks (hqr_sweep_dist_multi's kernel sequence). */
int hqr_sweep_virtual_multi(double* H, double* Z, int64_t n, int nblocks, const int64_t* ilo,
                            const int64_t* ihi, const double* shifts_re, const double* shifts_im,
                            const int* nshifts, int window, int vworld);

/* Release everything hqr_setup acquired.  Returns 0 (also when not set up) or 1000+cudaError_t. */
int hqr_teardown(void);

/* Largest effective window side the chase kernel supports (SMEM-resident window + factor). */
#define HQR_MAX_WINDOW 112
/* Library default window side (the bench's and the Python binding's default argument). */
#define HQR_DEFAULT_WINDOW 96

/*
 * Host-only introspection of the wavefront plan (no GPU needed; used by the tests).
 *   info[0..9] <- {k_eff, nbc_max, s, lag, nchains, nsteps, nwindows, max_kw, max_nbc, nb}
 *   windows    <- nwindows rows of 12 int32
 *                 {step, chain, w0, w1, t0, t1, b0, nbc, slot, last, ilo, ihi}
 *                 (may be NULL or cap too small: only info is written then)
 * Returns 0 or the same negative argument codes as hqr_sweep (matrix values are not inspected).
 */
int hqr_plan_query(int64_t n, int64_t ilo, int64_t ihi, int nshifts, int window, int32_t* info,
                   int32_t* windows, int64_t cap);
int hqr_plan_query_multi(int64_t n, int nblocks, const int64_t* ilo, const int64_t* ihi,
                         const int* nshifts, int window, int32_t* info, int32_t* windows,
                         int64_t cap);

int hqr_plan_query_sweeps(int64_t n, int64_t ilo, int64_t ihi, int nsweeps, const int* nshifts,
                          int window, int32_t* info, int32_t* windows, int64_t cap);

/* Statistics of the last successful hqr_sweep on this process. */
typedef struct hqr_stats {
  int64_t kernels_launched;   /* kernels of this library launched by the last sweep              */
  int64_t steps;              /* wavefront steps                                                  */
  int64_t windows;            /* chase-kernel CTAs (diagonal windows)                             */
  double flops_update;        /* GEMM flops of the off-diagonal update kernels (2*M*N*K, real kw) */
  double flops_chase;         /* flops of the in-window chase (reflector applications)           */
  double bytes_update;        /* algorithmic HBM bytes of the update kernels (panel read+write)   */
  double ms_chase;            /* HQR_FLAG_PROFILE only: summed CUDA-event time per kernel class    */
  double ms_left;
  double ms_right;            /* right update + fused Z update                                    */
  double ms_step;             /* fused step kernels (updates of step g + chase of step g+1)       */
  double ms_total;            /* CUDA-event time of the whole sweep (device work only)            */
  int64_t h2d_bytes, d2h_bytes; /* staging copies (host-pointer calls)                           */
  int launches_left, launches_right, launches_chase;
  int window_eff;             /* effective window side                                           */
  double flops_dmma;          /* executed FP64 tensor-core flops of the last single-GPU sweep: the
                                 update GEMMs restricted to the band extents the kernels multiply
                                 (computed on demand by hqr_get_stats; 0 if unavailable)           */
  double flops_alg;           /* design-independent F_alg (every reflector applied directly, SURVEY
                                 Appendix B) of the last call's sweeps; hqr_qr_iterate: summed over
                                 its sweeps                                                          */
  int crit_sms;               /* CTAs of the persistent launch that served only the critical queue
                                 (chases and their near tiles; 0: one queue) -- DESIGN.md §6        */
  int pad_;
} hqr_stats;

int hqr_get_stats(hqr_stats* out);

/* Static description of an error code. */
const char* hqr_error_string(int code);

#ifdef __cplusplus
}
#endif

#endif /* HQR_B200_H */
