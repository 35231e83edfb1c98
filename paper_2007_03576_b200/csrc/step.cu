// step.cu -- fused wavefront step: one persistent launch per step that runs the off-diagonal
// updates of step g AND the chase of step g+1, prioritised the way the paper's task insertion does
// (push-bulges and left updates first, right updates that feed the next chase
// next, far right updates and the Q (here: Z) updates last; updates that do not feed
// back to the bulge chase form a separate, low-priority subgraph).
//
// Work of step g as a queue of tasks, claimed by the resident CTAs (one per SM) in this order:
//   L   left-update chunks of every window                         (feed the next chase)
//   Rn  right-update chunks, rows [sp, w0) ("below the dashed line")  wait: all L done
//   C   chase of every window of step g+1                          wait: all L and Rn done
//   Z   Z-update chunks                                            (independent)
//   Rf  right-update chunks, rows [0, min(sp, w0))                 wait: all L done
// sp = the smallest first row of any later window (a suffix minimum over the plan, rounded down to
// even): no later chase, left or near-right update touches rows < sp of these columns, so the far
// right updates and Z overlap the next chase.  A task waits only on tasks earlier in the queue, all
// CTAs are resident, so the queue cannot deadlock.  L before R orders the blocks H(W_c, W_c') that
// a left update of the upper window and a right update of the lower window both modify.
// The GEMM chunks reuse the TMA/DMMA tile of gemm_tile.cuh (one Q_W per chunk); the chase runs the
// two-phase step of chase.cu with the CTA's 9 warps.
#include <cuda_runtime.h>

#include <algorithm>

#include "device_common.cuh"
#include "gemm_tile.cuh"
#include "kernels.hpp"
#include "step.hpp"

namespace hqr {

namespace {

constexpr int kStepThreads = 288;  // 8 consumer warps + 1 producer warp (GEMM); 9 chase warps
constexpr int kStepWarps = kStepThreads / 32;

__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;\n" ::: "memory"); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---- chase of one window with the CTA's 9 warps (same arithmetic as chase.cu) ------------------
struct ChaseSmem {
  double v1[kMaxChaseBulges], v2[kMaxChaseBulges], tau[kMaxChaseBulges];
  int pl[kMaxChaseBulges], m[kMaxChaseBulges];
};

__device__ void chase_window_9w(const StepArgs& a, const WindowDesc& W, double* sm, ChaseSmem& R) {
  const int kw = W.w1 - W.w0 + 1;
  const int ldh = kw | 1;
  double* Hs = sm;
  double* Qs = Hs + kw * ldh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int w0 = W.w0;
  const int ilo = W.ilo, ihi = W.ihi, nbc = W.nbc;
  {
    const double* g = a.H + (int64_t)(w0 - a.hcol0) * n + w0;
    for (int c = warp; c < kw; c += kStepWarps) {
      const double* gc = g + (int64_t)c * n;
      for (int r = lane; r < kw; r += 32) {
        Hs[r + c * ldh] = __ldcg(gc + r);  // L2: written by other SMs in this launch
        Qs[r + c * ldh] = (r == c) ? 1.0 : 0.0;
      }
    }
  }
  __syncthreads();
  const int rmaxH = ihi - w0;
  for (int t = W.t0; t <= W.t1; ++t) {
    const int rQ = min(ilo - 1 + t - w0 + 3, kw - 1);
    for (int jj = warp; jj < nbc; jj += kStepWarps) {
      const int p = ilo - 1 + t - 3 * jj;
      if (p < ilo - 1 || p > ihi - 2) {
        if (lane == 0) R.pl[jj] = INT_MIN;
        continue;
      }
      const int pl = p - w0;
      const int m = (p <= ihi - 3) ? 3 : 2;
      double x0, x1, x2;
      if (p == ilo - 1) {
        const int jb = W.b0 + jj;
        const double sigma = a.coef[2 * jb], pi = a.coef[2 * jb + 1];
        const double h00 = Hs[0], h10 = Hs[1], h01 = Hs[ldh], h11 = Hs[1 + ldh], h21 = Hs[2 + ldh];
        x0 = h00 * (h00 - sigma) + h01 * h10 + pi;
        x1 = h10 * (h00 + h11 - sigma);
        x2 = h10 * h21;
      } else {
        const double* col = Hs + pl * ldh + pl;
        x0 = col[1];
        x1 = col[2];
        x2 = (m == 3) ? col[3] : 0.0;
      }
      double v1, v2, tau, beta;
      house(x0, x1, x2, v1, v2, tau, beta);
      __syncwarp();
      if (lane == 0) {
        if (p >= ilo) {
          double* col = Hs + pl * ldh + pl;
          col[1] = beta;
          col[2] = 0.0;
          if (m == 3) col[3] = 0.0;
        }
        R.v1[jj] = v1; R.v2[jj] = v2; R.tau[jj] = tau;
        R.pl[jj] = (tau == 0.0) ? INT_MIN : pl;
        R.m[jj] = m;
      }
      if (tau == 0.0) continue;
      const int c0 = (p == ilo - 1) ? 0 : pl + 1;
      double* hrow = Hs + (pl + 1);
      for (int c = c0 + lane; c < kw; c += 32) {
        double* hc = hrow + c * ldh;
        const double h0 = hc[0], h1 = hc[1], h2 = (m == 3) ? hc[2] : 0.0;
        const double tw = tau * fma(v2, h2, fma(v1, h1, h0));
        hc[0] = h0 - tw;
        hc[1] = fma(-tw, v1, h1);
        if (m == 3) hc[2] = fma(-tw, v2, h2);
      }
    }
    __syncthreads();
    for (int jj = warp; jj < nbc; jj += kStepWarps) {
      Refl r;
      r.pl = R.pl[jj];
      if (r.pl == INT_MIN) continue;
      r.v1 = R.v1[jj]; r.v2 = R.v2[jj]; r.tau = R.tau[jj]; r.m = R.m[jj];
      right_apply(Hs + (r.pl + 1) * ldh, ldh, min(r.pl + r.m + 1, rmaxH) + 1, r, lane);
      right_apply(Qs + (r.pl + 1) * ldh, ldh, rQ + 1, r, lane);
    }
    __syncthreads();
  }
  {
    double* g = a.H + (int64_t)(w0 - a.hcol0) * n + w0;
    for (int c = warp; c < kw; c += kStepWarps) {
      double* gc = g + (int64_t)c * n;
      for (int r = lane; r < kw; r += 32) gc[r] = Hs[r + c * ldh];
    }
  }
  const int KP = a.KP, QLD = a.QLD;
  double* Q = a.qslots + (size_t)(W.slot + a.slot_offset) * KP * QLD;
  store_q_slot(Q, Qs, ldh, kw, KP, QLD, warp, kStepWarps, lane);
}

// ---- one GEMM chunk: `ntiles` tiles of one window, Q_W loaded once -----------------------------
template <int KP, bool LEFT>
__device__ void gemm_chunk(const StepArgs& a, const WindowDesc& w, const Task& T, double* sm,
                           uint64_t* full, uint64_t* empty, uint64_t* qfull, int& j, unsigned& nq,
                           const CUtensorMap* tmL, const CUtensorMap* tmR, const CUtensorMap* tmZ,
                           int stage_stride) {
  using G = Geom<KP, LEFT>;
  constexpr int NS = stages_of(KP), QLD = G::QLD;
  double* Qs = sm;
  double* Ps = sm + KP * QLD;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto tile_ref = [&](int i) {
    TileRef t;
    t.w0 = w.w0; t.kw = w.w1 - w.w0 + 1; t.nbc = w.nbc;
    if (LEFT) {
      int64_t c, cnt;
      left_range(a, w, c, cnt);
      t.M = a.H; t.c0 = c + (int64_t)(T.tile0 + i) * G::NT; t.lc1 = a.lc1; t.ld = a.n; t.cb = a.hcol0;
      t.isZ = false; t.r0 = t.r1 = 0;
    } else if (T.type == kTaskZ) {
      t.M = a.Z; t.r0 = (int64_t)(T.tile0 + i) * G::MT; t.r1 = a.zrows; t.ld = a.ldz; t.cb = 0;
      t.isZ = true; t.c0 = t.lc1 = 0;
    } else {
      t.M = a.H; t.r0 = T.r_lo + (int64_t)(T.tile0 + i) * G::MT; t.r1 = T.r_hi; t.ld = a.n;
      t.cb = a.hcol0; t.isZ = false; t.c0 = t.lc1 = 0;
    }
    return t;
  };
  if (warp == 8) {
    const double* Q = a.qslots + (size_t)(w.slot + a.slot_offset) * KP * QLD;
    constexpr unsigned qbytes = KP * QLD * 8, chunk = qbytes / 32;
    fence_proxy_async_all();  // generic writes of earlier tasks before this task's TMA reads
    if (lane == 0) mbar_arrive_tx(qfull, qbytes);
    __syncwarp();
    bulk_g2s(reinterpret_cast<char*>(Qs) + lane * chunk, reinterpret_cast<const char*>(Q) + lane * chunk,
             chunk, qfull);
    for (int i = 0; i < T.ntiles; ++i) {
      const int jj = j + i, s = jj % NS;
      if (jj >= NS) mbar_wait(&empty[s], (unsigned)((jj / NS) - 1) & 1);
      if (lane == 0)
        produce_tile<KP, LEFT>(Ps + s * stage_stride, &full[s], LEFT ? tmL : tmR, tmZ, tile_ref(i));
      __syncwarp();
    }
  } else {
    const int q = warp >> 2, i4 = warp & 3;
    mbar_wait(qfull, nq & 1);
    for (int i = 0; i < T.ntiles; ++i) {
      const int jj = j + i, s = jj % NS;
      if ((jj & 1) != q) continue;
      mbar_wait(&full[s], (unsigned)(jj / NS) & 1);
      consume_tile<KP, LEFT>(Qs, Ps + s * stage_stride, &empty[s], tile_ref(i), q, i4, lane);
    }
  }
  j += T.ntiles;
  ++nq;
}

template <int KP>
__global__ void __launch_bounds__(kStepThreads, 1)
    step_kernel(StepArgs a, StepArgs an, const Task* __restrict__ tasks, int ntasks, int nL, int nRn,
                StepCounters* ctr, const __grid_constant__ CUtensorMap tmL,
                const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmZ) {
  constexpr int NS = stages_of(KP);
  constexpr int SS = Geom<KP, true>::STAGE > Geom<KP, false>::STAGE ? Geom<KP, true>::STAGE
                                                                    : Geom<KP, false>::STAGE;
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS], qfull;
  __shared__ Task cur;
  __shared__ int cur_idx;
  __shared__ WindowDesc cw;
  __shared__ ChaseSmem R;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    mbar_init(&qfull, 1);
  }
  fence_proxy_async();
  __syncthreads();
  int j = 0;        // tiles through the ring so far (identical in every warp)
  unsigned nq = 0;  // Q_W loads so far
  for (;;) {
    if (tid == 0) {
      const int t = atomicAdd(&ctr->next, 1);
      cur_idx = t;
      if (t < ntasks) {
        cur = tasks[t];
        const Task& T = cur;
        // dependencies: on tasks earlier in the queue only
        if (T.type == kTaskRight || T.type == kTaskChase)
          while (ld_acquire(&ctr->l_done) < nL) __nanosleep(64);
        if (T.type == kTaskChase)
          while (ld_acquire(&ctr->rn_done) < nRn) __nanosleep(64);
        cw = (T.type == kTaskChase) ? an.wins[an.win_begin + T.win] : a.wins[a.win_begin + T.win];
      }
    }
    __syncthreads();
    const int t = cur_idx;
    if (t >= ntasks) break;
    const Task T = cur;
    const WindowDesc w = cw;
    if (T.type == kTaskChase) {
      chase_window_9w(an, w, sm, R);
    } else if (T.type == kTaskLeft) {
      gemm_chunk<KP, true>(a, w, T, sm, full, empty, &qfull, j, nq, &tmL, &tmR, &tmZ, SS);
    } else {
      gemm_chunk<KP, false>(a, w, T, sm, full, empty, &qfull, j, nq, &tmL, &tmR, &tmZ, SS);
    }
    __syncthreads();  // every store of the task issued; the SMEM may be reused
    if (tid == 0) {
      __threadfence();
      fence_proxy_async_all();
      if (T.type == kTaskLeft) atomicAdd(&ctr->l_done, 1);
      else if (T.type == kTaskRight && t < nL + nRn) atomicAdd(&ctr->rn_done, 1);
    }
  }
}

template <int KP>
size_t step_smem(int max_kw) {
  constexpr int SS = Geom<KP, true>::STAGE > Geom<KP, false>::STAGE ? Geom<KP, true>::STAGE
                                                                    : Geom<KP, false>::STAGE;
  size_t gemm = (size_t)(KP * pad_ld(KP) + stages_of(KP) * SS) * sizeof(double);
  size_t chase = (size_t)2 * max_kw * (max_kw | 1) * sizeof(double);
  return std::max(gemm, chase);
}

template <int KP>
cudaError_t launch_step_t(const StepArgs& a, const StepArgs& an, const Task* tasks, int ntasks, int nL,
                          int nRn, StepCounters* ctr, const TensorMaps& tm, int max_kw, int num_sms,
                          cudaStream_t st) {
  static size_t configured = 0;
  const size_t smem = step_smem<KP>(max_kw);
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(step_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int grid = std::max(1, std::min(ntasks, num_sms));
  step_kernel<KP><<<grid, kStepThreads, smem, st>>>(a, an, tasks, ntasks, nL, nRn, ctr, tm.left_H,
                                                     tm.right_H, tm.right_Z);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_step(const StepArgs& a, const StepArgs& an, const Task* tasks, int ntasks, int nL,
                        int nRn, StepCounters* ctr, const TensorMaps& tm, int max_kw, int num_sms,
                        cudaStream_t st) {
  if (!tm.valid) return cudaErrorNotSupported;
  switch (a.KP) {
    case 32: return launch_step_t<32>(a, an, tasks, ntasks, nL, nRn, ctr, tm, max_kw, num_sms, st);
    case 64: return launch_step_t<64>(a, an, tasks, ntasks, nL, nRn, ctr, tm, max_kw, num_sms, st);
    case 96: return launch_step_t<96>(a, an, tasks, ntasks, nL, nRn, ctr, tm, max_kw, num_sms, st);
    case 128: return launch_step_t<128>(a, an, tasks, ntasks, nL, nRn, ctr, tm, max_kw, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

// Host: the task queue of one step (L, Rn, C, Z, Rf).  Chunk sizes (tiles per task) per phase:
// cs.left, cs.near for L / Rn (they gate the next chase: small), cs.bulk for Z / Rf; the last
// cs.tail tiles of the queue use chunks of cs.tail_chunk so the CTAs finish together.
void build_step_tasks(const StepArgs& a, const WindowDesc* wins, int nwin, const WindowDesc* next_wins,
                      int nnext, int64_t sp, const ChunkSizes& cs, std::vector<Task>* out, int* nL,
                      int* nRn) {
  const int NT = left_cols(a.KP), MT = right_rows(a.KP);
  auto add = [&](int type, int win, int64_t tiles, int64_t r_lo, int64_t r_hi, int chunk) {
    for (int64_t t0 = 0; t0 < tiles; t0 += chunk) {
      Task T{};
      T.type = type; T.win = win; T.tile0 = (int32_t)t0;
      T.ntiles = (int32_t)std::min<int64_t>(chunk, tiles - t0);
      T.r_lo = r_lo; T.r_hi = r_hi;
      out->push_back(T);
    }
  };
  const size_t base = out->size();
  for (int i = 0; i < nwin; ++i) {
    int64_t c, cnt;
    left_range(a, wins[i], c, cnt);
    add(kTaskLeft, i, (cnt + NT - 1) / NT, 0, 0, cs.left);
  }
  *nL = (int)(out->size() - base);
  const size_t rn0 = out->size();
  for (int i = 0; i < nwin; ++i) {
    const int64_t w0 = wins[i].w0;
    if (sp < w0) add(kTaskRight, i, (w0 - sp + MT - 1) / MT, sp, w0, cs.near);
  }
  *nRn = (int)(out->size() - rn0);
  for (int i = 0; i < nnext; ++i) {
    Task T{};
    T.type = kTaskChase; T.win = i; T.ntiles = 0;
    out->push_back(T);
  }
  const size_t bulk0 = out->size();
  if (a.Z)
    for (int i = 0; i < nwin; ++i) add(kTaskZ, i, (a.zrows + MT - 1) / MT, 0, 0, cs.bulk);
  for (int i = 0; i < nwin; ++i) {
    const int64_t hi = std::min<int64_t>(sp, wins[i].w0);
    if (hi > 0) add(kTaskRight, i, (hi + MT - 1) / MT, 0, hi, cs.bulk);
  }
  // re-split the queue's last cs.tail tiles into small chunks (same order)
  int64_t acc = 0;
  size_t cut = out->size();
  while (cut > bulk0 && acc < cs.tail) acc += (*out)[--cut].ntiles;
  std::vector<Task> tail(out->begin() + cut, out->end());
  out->resize(cut);
  for (const Task& T : tail)
    for (int t0 = 0; t0 < T.ntiles; t0 += cs.tail_chunk) {
      Task U = T;
      U.tile0 = T.tile0 + t0;
      U.ntiles = std::min(cs.tail_chunk, T.ntiles - t0);
      out->push_back(U);
    }
}

}  // namespace hqr
