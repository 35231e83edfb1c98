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
// two-phase step of chase.cu with all of the CTA's warps.
#include <cuda_runtime.h>

#include <string>

#include <algorithm>
#ifdef HQR_PROGRESS  // debugging build only: per-warp progress in host-mapped memory, dumped on a hang
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <cstring>
#include <unistd.h>
#endif

#include "device_common.cuh"
#include "gemm_tile.cuh"
#include "kernels.hpp"
#include "plan.hpp"
#include "step.hpp"

namespace hqr {

namespace {

constexpr int kGroups = 3;  // consumer groups of 4 warps (one warp per SM sub-partition each): 3 groups fit
                            // the 128-register cap (4 warps on one sub-partition) without spills
constexpr int kProducerWarp = 4 * kGroups;
constexpr int kStepThreads = 32 * (4 * kGroups + 1);  // consumers + 1 producer warp; all chase
constexpr int kStepWarps = kStepThreads / 32;
static_assert(kStepWarps >= kChainCap, "one chase warp per bulge of a chain (plan.hpp kChainCap)");

__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;\n" ::: "memory"); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

#ifdef HQR_PROGRESS
__device__ int* g_prog;
// per-warp ring of the last 64 events: g_prog[((block * 16 + warp) * 65)] = count, then 64 slots
#define PROG(tag) do { if (lane == 0) { int* _b = g_prog + (blockIdx.x * 16 + warp) * 65; \
    const int _n = __ldcg(_b); __stcg(_b + 1 + (_n & 63), (tag)); __stcg(_b, _n + 1); } } while (0)
#else
#define PROG(tag) do { } while (0)
#endif

#ifdef HQR_TIMING  // debugging build only: per-step critical-path timestamps (globaltimer, ns)
__device__ unsigned long long g_tim[4096][4];  // min CTA start, min chase start, max chase end, max end
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_ctim[8];
__device__ unsigned long long g_wrec[8192][6];
__device__ unsigned long long g_trec[262144][8];  // per task: claim, deps met, tiles issued, done (max flush), type | win << 8, step  // per chased window: start, end (globaltimer ns), b0, step, claim, deps met
__device__ unsigned long long g_wait[12];  // [0..7] producer dependency spins per tag; [8] chase, [9] CTA, [10] consumer waits, [11] consumer K+epilogue  // chase: summed cycles per phase (all warps), windows
#define TIM_MIN(s, k) atomicMin(&g_tim[(s) & 4095][k], gtime())
#define TIM_MAX(s, k) atomicMax(&g_tim[(s) & 4095][k], gtime())
#else
#define TIM_MIN(s, k) do { } while (0)
#define TIM_MAX(s, k) do { } while (0)
#endif

// spin until *p >= target (acquire); the watchdog build reports a hang and traps
__device__ __forceinline__ void spin_until(const int* p, int target, int tag) {
#ifdef HQR_WATCHDOG
  long long it = 0;
#endif
  int v;
#ifdef HQR_TIMING
  const long long w0 = clock64();
  bool waited = false;
#endif
  while ((v = ld_acquire(p)) < target) {
#ifdef HQR_TIMING
    waited = true;
#endif
    __nanosleep(64);
#ifdef HQR_WATCHDOG
    if (++it == (1ll << (HQR_WD_LIMIT - 2))) {
#ifndef HQR_WD_NOPRINT
      printf("hqr watchdog: block %d spin tag %d value %d target %d\n", blockIdx.x, tag, v, target);
#endif
      __trap();
    }
#endif
  }
#ifdef HQR_TIMING
  if (waited) atomicAdd(&g_wait[tag & 7], (unsigned long long)(clock64() - w0));
#endif
}

// ---- chase of one window with all of the CTA's warps (same arithmetic as chase.cu) ------------------
struct ChaseSmem {
  double v1[kMaxChaseBulges], v2[kMaxChaseBulges], tau[kMaxChaseBulges];
  int pl[kMaxChaseBulges], m[kMaxChaseBulges];
};

__device__ void chase_window_9w(const StepArgs& a, const WindowDesc& W, int widx, double* sm, ChaseSmem& R) {
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
#ifdef HQR_TIMING
  long long c_p1 = 0, c_s1 = 0, c_p2 = 0, c_s2 = 0, c_pa = 0, c_pb = 0, c_t = clock64();
#define CTIM(acc) do { const long long _c = clock64(); acc += _c - c_t; c_t = _c; } while (0)
#else
#define CTIM(acc) do { } while (0)
#endif
  const int rmaxH = ihi - w0;
  for (int t = W.t0; t <= W.t1; ++t) {
    const int rQ = min(ilo - 1 + t - w0 + 3, kw - 1);
    // A warp's first bulge (jj = warp; every bulge when nbc <= kStepWarps, i.e. every multi-window
    // chain) keeps its reflector in registers across the barrier; further bulges of a warp (a block
    // that fits one window holds up to N/2 bulges) go through SMEM.
    double rv1 = 0.0, rv2 = 0.0, rtau = 0.0;  // the first bulge's reflector (tau = 0: none)
    for (int jj = warp; jj < nbc; jj += kStepWarps) {
      const int p = ilo - 1 + t - 3 * jj;
      if (p < ilo - 1 || p > ihi - 2) {
        if (jj >= kStepWarps && lane == 0) R.pl[jj] = INT_MIN;
        continue;
      }
      const int pl = p - w0;
      const int m = (p <= ihi - 3) ? 3 : 2;
      double x0, x1, x2;
      if (p == ilo - 1) {
        intro_vector(Hs, ldh, a.coef + 4 * (W.b0 + jj), x0, x1, x2);
      } else {
        const double* col = Hs + pl * ldh + pl;
        x0 = col[1];
        x1 = col[2];
        x2 = (m == 3) ? col[3] : 0.0;
      }
      double v1, v2, tau, beta;
      house(x0, x1, x2, v1, v2, tau, beta);
      CTIM(c_pa);
      __syncwarp();
      if (p >= ilo && lane < m) Hs[pl * ldh + pl + 1 + lane] = (lane == 0) ? beta : 0.0;  // beta, exact zeros
      if (jj < kStepWarps) {
        rv1 = v1; rv2 = v2; rtau = tau;
      } else if (lane == 0) {
        R.v1[jj] = v1; R.v2[jj] = v2; R.tau[jj] = tau; R.pl[jj] = (tau == 0.0) ? INT_MIN : pl; R.m[jj] = m;
      }
      CTIM(c_pb);
      if (tau == 0.0) continue;
      left_apply(Hs + (pl + 1), ldh, (p == ilo - 1) ? 0 : pl + 1, kw, m, v1, v2, tau, lane);
    }
    CTIM(c_p1);
    __syncthreads();
    CTIM(c_s1);
    for (int jj = warp; jj < nbc; jj += kStepWarps) {
      Refl r;
      if (jj < kStepWarps) {
        const int p = ilo - 1 + t - 3 * jj;
        r.pl = (rtau == 0.0 || p < ilo - 1 || p > ihi - 2) ? INT_MIN : p - w0;
        r.m = (p <= ihi - 3) ? 3 : 2;
        r.v1 = rv1; r.v2 = rv2; r.tau = rtau;
      } else {
        r.pl = R.pl[jj];
        r.v1 = R.v1[jj]; r.v2 = R.v2[jj]; r.tau = R.tau[jj]; r.m = R.m[jj];
      }
      if (r.pl == INT_MIN) continue;
      right_apply(Hs + (r.pl + 1) * ldh, ldh, min(r.pl + r.m + 1, rmaxH) + 1, r, lane);
      const int q0 = q_first_row(W, jj);
      right_apply(Qs + (r.pl + 1) * ldh + q0, ldh, rQ + 1 - q0, r, lane);
    }
    CTIM(c_p2);
    __syncthreads();
    CTIM(c_s2);
  }
#ifdef HQR_TIMING
  if (lane == 0) {
    atomicAdd(&g_ctim[0], (unsigned long long)c_p1);
    atomicAdd(&g_ctim[1], (unsigned long long)c_s1);
    atomicAdd(&g_ctim[2], (unsigned long long)c_p2);
    atomicAdd(&g_ctim[3], (unsigned long long)c_s2);
    atomicAdd(&g_ctim[6], (unsigned long long)c_pa);
    atomicAdd(&g_ctim[7], (unsigned long long)c_pb);
    if (warp == 0) atomicAdd(&g_ctim[4], 1ull);
    if (warp == 0) atomicAdd(&g_ctim[5], (unsigned long long)(W.t1 - W.t0 + 1));
  }
#endif
  aftermath_scan(Hs, ldh, W, a.aftermath, threadIdx.x, kStepThreads);  // a9 (check only)
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
  if (a.wstats) {
    __syncthreads();
    if (threadIdx.x == 0) a.wstats[widx] = band_units(Q, KP, QLD);
  }
}

// ---- streaming task pipeline ------------------------------------------------------------------
// The producer warp (warp 8, lane 0 acting) claims tasks, waits for their dependencies, loads Q_W
// when the window changes, and streams the tasks' panel tiles through the SMEM ring; every stage
// carries a descriptor.  The consumer groups take the ring's tiles in order (group q: tiles
// j = q mod 2) with no CTA-wide barrier between tasks.  Completion is counted per tile and warp
// (release adds) for the tasks other tasks depend on.  A chase task drains the ring (markers to
// every group), then all warps chase one window in the whole SMEM.
constexpr int kDescTile = 0, kDescChase = 1, kDescExit = 2;

struct StageDesc {
  int pos;     // ring position this descriptor belongs to (see the consumer's wait)
  int kind;    // kDescTile / kDescChase / kDescExit
  int left;    // tile: LEFT (1) or RIGHT/Z (0)
  int qe;      // tile: Q_W load epoch it multiplies with
  int cnt_add; // tile with ctr: tiles of the task this group has done (this warp adds them)
  int* ctr;    // tile: nullptr, or the counter the task's completion feeds (after the stores) ...
  int* ctr2;   // ... a second one (near tasks: their phase's step counter) or nullptr ...
  int* ctr_all;  // ... and the step's all-tiles counter
  TileRef t;
#ifdef HQR_TIMING
  int task;    // timing builds: the sweep task index
#endif
};

// One release fence, then relaxed adds: the release pattern for several counters at the cost of one
// membar (red.release costs a full MEMBAR.GPU + ERRBAR each).
__device__ __forceinline__ void fence_release_gpu() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_add(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

template <int KP, bool LEFT>
__device__ __forceinline__ TileRef make_tile_ref(const StepArgs& a, const WindowDesc& w, const Task& T, int i) {
  using G = Geom<KP, LEFT>;
  TileRef t;
  t.w0 = w.w0; t.kw = w.w1 - w.w0 + 1; t.nbc = w.nbc;
  if (LEFT) {
    int64_t c, c_al, cnt;
    left_range_al(a, w, c, c_al, cnt);
    t.M = a.H; t.c0 = c_al + (int64_t)(T.tile0 + i) * G::NT; t.lc1 = a.lc1; t.ld = a.n; t.cb = a.hcol0;
    t.isZ = false; t.r0 = t.r1 = 0; t.lcs = c;
  } else if (T.type == kTaskZ) {
    t.M = a.Z; t.r0 = (int64_t)(T.tile0 + i) * G::MT; t.r1 = a.zrows; t.ld = a.ldz; t.cb = 0;
    t.isZ = true; t.c0 = t.lc1 = t.lcs = 0;
  } else {
    t.M = a.H; t.r0 = T.r_lo + (int64_t)(T.tile0 + i) * G::MT; t.r1 = T.r_hi; t.ld = a.n;
    t.cb = a.hcol0; t.isZ = false; t.c0 = t.lc1 = t.lcs = 0;
  }
  return t;
}

// Per-task step arguments: the sweep-wide base with the task's step fields.
__device__ __forceinline__ StepArgs step_args(const StepArgs& base, const StepInfo* steps, int s, int nsteps) {
  StepArgs a = base;
  if (s < nsteps) {
    const StepInfo S = steps[s];
    a.win_begin = S.win_begin;
    a.win_count = S.win_count;
    a.slot_offset = S.slot_offset;
  }
  a.step = s;
  return a;
}

// The task list may span one step (a launch per step) or the whole sweep (one persistent launch):
// every dependency is a completion counter, so the same code serves both.  Dependencies of a task
// of step g (all on tasks earlier in the list; all CTAs resident, so no deadlock):
//   any GEMM task of window W    the chase of W (run while step g-1 was executing)
//   right (near and far), chase  every left tile of step g
//   chase (of step g+1)          every near-right tile of step g, and every tile of step g+1-kQSets
//                                (its Q slot set is reused)
//   far right of W               the far-right tiles of every step-(g-1) window whose columns meet W
//   Z of W                       the Z tiles of every step-(g-1) window whose columns meet W
// (the left update of W and the near-right updates of step g-1 are ordered through W's chase).
template <int KP>
__global__ void __launch_bounds__(kStepThreads, 1)
    step_kernel(StepArgs base, const StepInfo* __restrict__ steps, int nsteps, const Task* __restrict__ tasks,
                int ntasks, int task_base, const int32_t* __restrict__ dep_begin, const int2* __restrict__ deps,
                int* next_ctr, int* step_ctr, int* task_ctr,
                const int* __restrict__ up_flags, const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmR,
                const __grid_constant__ CUtensorMap tmZ, const int32_t* __restrict__ qidx, int ncrit, int crit_sms) {
  constexpr int NS = stages_of(KP);
  constexpr int QLD = pad_ld(KP);
  constexpr int SS = Geom<KP, true>::STAGE > Geom<KP, false>::STAGE ? Geom<KP, true>::STAGE
                                                                    : Geom<KP, false>::STAGE;
  extern __shared__ __align__(1024) double sm[];
#ifdef HQR_TIMING
  const long long k_start = clock64();
#endif
  __shared__ __align__(8) uint64_t full[NS], empty[NS], qfull;
  __shared__ StageDesc desc[NS];
  __shared__ WindowDesc cw;
  __shared__ int cwi;  // its plan index
  __shared__ StepArgs cargs;  // the chased window's step
  __shared__ ChaseSmem R;
  double* Qs = sm;
  double* Ps = sm + KP * QLD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    mbar_init(&qfull, 1);
  }
  if (tid < NS) desc[tid].pos = -1;
  fence_proxy_async();
  __syncthreads();

  if (warp == kProducerWarp) {
    // ================================ producer / scheduler ================================
    int j = 0;          // ring positions used (tiles + markers)
    int qe = -1;        // Q_W loads so far - 1
    int q_win = -1;     // plan window whose Q_W is resident (-1: none)
    // Producer-side waits are done by lane 0 alone, then __syncwarp: a lane that saw the phase
    // complete may publish the next position before its sibling lanes poll again, and the
    // consumers can complete one more phase in between -- a parity wait would then never return.
    auto wait_slot = [&](int jj) {  // stage of ring position jj free
      PROG(5000000 + jj);
      if (jj >= NS && lane == 0) mbar_wait(&empty[jj % NS], (unsigned)((jj / NS) - 1) & 1, 1000000 + jj);
      __syncwarp();
    };
    auto marker = [&](int kind) {   // one marker per consumer group
      for (int g = 0; g < kGroups; ++g, ++j) {
        wait_slot(j);
        if (lane == 0) {
          desc[j % NS].kind = kind;
          desc[j % NS].pos = j;
          mbar_arrive(&full[j % NS]);
        }
        __syncwarp();
      }
    };
    for (;;) {
      int t = 0;
      PROG(1000000 + j);
      if (lane == 0) {
        if (crit_sms == 0) {
          t = atomicAdd(next_ctr, 1);
        } else if ((int)blockIdx.x < crit_sms) {  // the critical queue
          const int i = atomicAdd(next_ctr, 1);
          t = i < ncrit ? qidx[i] : ntasks;
        } else {                                  // the bulk queue
          const int i = atomicAdd(next_ctr + 1, 1);
          t = i < ntasks - ncrit ? qidx[ncrit + i] : ntasks;
        }
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntasks) {
        marker(kDescExit);
        PROG(8000000 + j);
        break;
      }
      const Task T = tasks[t];
      const int g = T.step;
      const StepInfo S = steps[g];
      int* sc = step_ctr + 4 * g;
      const bool chase = T.type == kTaskChase;
      const int gw = chase ? -1 : S.win_begin + T.win;  // plan index of the task's window
      const int tg = task_base + t;                      // the task's index in the sweep
#ifdef HQR_TIMING
      const unsigned long long w_claim = gtime();
#endif
      if (lane == 0) {
        PROG(2000000 + t);
        if (up_flags) spin_until(up_flags + S.up_need, 1, 5);  // host-buffer sweep: rows / columns up
        if (chase) {  // the Q slot set is reused: every tile of step g+1-kQSets done
          const int g_old = g + 1 - kQSets;
          if (g_old >= 0) spin_until(step_ctr + 4 * g_old + 2, 4 * steps[g_old].ntiles, 3);
        }
      }
      {  // the last earlier task that touched each part of this task's rectangle, and (GEMM tasks)
         // the chase that produced the window's factor (hqr_api.cu build_task_deps): 32 counters
         // per round trip, one per lane
#ifdef HQR_TIMING
        const long long d0c = clock64();
        bool waited = false;
#endif
        const int dend = dep_begin[tg + 1];
        for (int d0 = dep_begin[tg]; d0 < dend; d0 += 32) {
          const int d = d0 + lane;
          int2 dp = make_int2(0, 0);
          if (d < dend) dp = deps[d];
          bool ok = d >= dend || ld_acquire(task_ctr + dp.x) >= dp.y;
          while (!__all_sync(0xffffffffu, ok)) {
#ifdef HQR_TIMING
            waited = true;
#endif
            __nanosleep(64);
            if (!ok) ok = ld_acquire(task_ctr + dp.x) >= dp.y;
          }
        }
#ifdef HQR_TIMING
        if (lane == 0 && waited) atomicAdd(&g_wait[1], (unsigned long long)(clock64() - d0c));
#endif
      }
      __syncwarp();  // the lanes' acquires before lane 0's async-proxy fence and TMA reads
      if (lane == 0) fence_proxy_async_all();  // other SMs' generic stores before this SM's TMA reads
      __syncwarp();
#ifdef HQR_TIMING
      if (lane == 0 && tg < 262144) {
        g_trec[tg][0] = w_claim;
        g_trec[tg][1] = gtime();
        g_trec[tg][4] = (unsigned long long)(T.type | (T.win << 8));
        g_trec[tg][5] = (unsigned long long)T.step | ((unsigned long long)T.ntiles << 32);
      }
#endif
      if (chase) {
#ifdef HQR_TIMING
        const unsigned long long w_depok = gtime();
#endif
        marker(kDescChase);
        PROG(7000000 + j);
        if (lane == 0) {
          cargs = step_args(base, steps, g + 1, nsteps);
          cw = cargs.wins[cargs.win_begin + T.win];
          cwi = cargs.win_begin + T.win;
        }
        __syncthreads();
        if (lane == 0) TIM_MIN(g, 1);
#ifdef HQR_TIMING
        const long long c_start = clock64();
#endif
#ifdef HQR_TIMING
        const unsigned long long w_start = gtime();
#endif
        chase_window_9w(cargs, cw, cwi, sm, R);
        __syncthreads();
#ifdef HQR_TIMING
        if (lane == 0) atomicAdd(&g_wait[8], (unsigned long long)(clock64() - c_start));
        if (lane == 0 && cwi < 8192) {
          g_wrec[cwi][0] = w_start;
          g_wrec[cwi][1] = gtime();
          g_wrec[cwi][2] = (unsigned long long)cw.b0;
          g_wrec[cwi][3] = (unsigned long long)(g + 1);
          g_wrec[cwi][4] = w_claim;
          g_wrec[cwi][5] = w_depok;
        }
#endif
        if (lane == 0) {
          TIM_MAX(g, 2);
          red_release_add(task_ctr + tg, 1);  // the CTA's stores are ordered by the barrier
#ifdef HQR_TIMING
          if (tg < 262144) g_trec[tg][3] = gtime();
#endif
        }
        q_win = -1;
        continue;
      }
      const StepArgs a = step_args(base, steps, g, nsteps);
      const WindowDesc w = a.wins[gw];
      // A new window needs its Q_W.  Its first NS-1 panel tiles are issued first (their stages free
      // up as the previous tiles are released); once every earlier position has been released --
      // no tile reads the old Q_W any more -- Q_W is loaded, so the panel loads overlap the drain.
#ifdef HQR_BENCH_NO_QSWITCH  // timing experiment only: keep the first Q_W (wrong results)
      const bool new_q = q_win < 0;
#else
      const bool new_q = gw != q_win;
#endif
      if (new_q) {
        ++qe;
        q_win = gw;
      }
      const int p0 = j;
      auto load_q = [&]() {
        PROG(4000000 + j);
        if (lane == 0)
          for (int jj = max(0, p0 - NS); jj < p0; ++jj)
            mbar_wait(&empty[jj % NS], (unsigned)(jj / NS) & 1, 2000000 + jj);
        __syncwarp();
        const double* Q = a.qslots + (size_t)(w.slot + a.slot_offset) * KP * QLD;
        constexpr unsigned qbytes = KP * QLD * 8, chunk = qbytes / 32;
        if (lane == 0) mbar_arrive_tx(&qfull, qbytes);
        __syncwarp();
        bulk_g2s(reinterpret_cast<char*>(Qs) + lane * chunk, reinterpret_cast<const char*>(Q) + lane * chunk,
                 chunk, &qfull);
      };
      const bool left = T.type == kTaskLeft || T.type == kTaskLeftNear;
      // the counters the task's completion feeds (tiles x 4 warps): its own, and the step's
      int* cnt = task_ctr + tg;
      int* cnt2 = nullptr;
      const int nq_pre = new_q ? min(T.ntiles, NS - 1) : 0;  // tiles issued before the Q_W load
      for (int i = 0; i < T.ntiles; ++i, ++j) {
        if (new_q && i == nq_pre) load_q();
        wait_slot(j);
        if (lane == 0) {
          StageDesc& d = desc[j % NS];
          d.pos = j; d.kind = kDescTile; d.left = left; d.qe = qe;
#ifdef HQR_TIMING
          d.task = tg;
#endif
          // completion counts: on each group's last tile of the task, that group's tile count
          // (the group of tile i takes the task's tiles i, i-G, ..., i.e. i/G + 1 of them)
          const bool last = i + kGroups >= T.ntiles;
          d.ctr = last ? cnt : nullptr;
          d.ctr2 = last ? cnt2 : nullptr;
          d.ctr_all = last ? sc + 2 : nullptr;
          d.cnt_add = i / kGroups + 1;
          if (left) {
            d.t = make_tile_ref<KP, true>(a, w, T, i);
            produce_tile<KP, true>(Ps + (j % NS) * SS, &full[j % NS], &tmL, &tmZ, d.t);
          } else {
            d.t = make_tile_ref<KP, false>(a, w, T, i);
            produce_tile<KP, false>(Ps + (j % NS) * SS, &full[j % NS], &tmR, &tmZ, d.t);
          }
        }
        __syncwarp();
      }
      if (new_q && nq_pre == T.ntiles) load_q();  // short task: the Q_W load after its tiles
#ifdef HQR_TIMING
      if (lane == 0 && tg < 262144) g_trec[tg][2] = gtime();
#endif
    }
  } else {
    // ================================ consumers ================================
    const int q = warp >> 2, i4 = warp & 3;  // group, sub-partition
    int last_qe = -1;
    // Completion counts (tiles x 4 warps) are published with release adds.  The release waits for
    // the warp's outstanding stores, so it is deferred: it is issued after the next tile's K loop
    // (the earlier stores have landed by then), or at once when the warp would otherwise wait
    // with counts pending (never sit on them: others may wait for them).
    int* pend_p = nullptr;
    int* pend_p2 = nullptr;
    int* pend_all = nullptr;
    int pend_n = 0;
    auto flush = [&]() {
      __syncwarp();
      if (lane == 0) {
        fence_release_gpu();  // the warp's stores (ordered by __syncwarp) before the three counts
        red_relaxed_add(pend_p, pend_n);
#ifdef HQR_TIMING
        if (pend_p - task_ctr >= 0 && pend_p - task_ctr < 262144) atomicMax(&g_trec[pend_p - task_ctr][3], gtime());
#endif
        if (pend_p2) red_relaxed_add(pend_p2, pend_n);
        red_relaxed_add(pend_all, pend_n);
      }
      pend_p = nullptr;
      pend_n = 0;
    };
    for (int j = q;; j += kGroups) {
      const int s = j % NS;
      PROG(11000000 + j);
      // The stage's previous phase belongs to the other group and may still be in flight; a parity
      // wait cannot tell phase p from p - 2, so first wait until the producer has published this
      // position (which it does only after the previous phase was consumed), then on the barrier.
      if (pend_p && *reinterpret_cast<volatile int*>(&desc[s].pos) != j) flush();
#ifdef HQR_TIMING
      const long long cw0 = clock64();
#endif
      while (*reinterpret_cast<volatile int*>(&desc[s].pos) != j) {
#ifdef HQR_EXP_DESC_SLEEP  // experiment: back off the consumers' descriptor spin
        __nanosleep(HQR_EXP_DESC_SLEEP);
#endif
      }
#ifdef HQR_TIMING
      const long long cw1 = clock64();
#endif
      mbar_wait(&full[s], (unsigned)(j / NS) & 1, 3000000 + j);
#ifdef HQR_TIMING
      if (lane == 0) {
        atomicAdd(&g_wait[10], (unsigned long long)(cw1 - cw0));
        atomicAdd(&g_wait[5], (unsigned long long)(clock64() - cw1));
      }
#endif
      const int kind = desc[s].kind;
      if (kind != kDescTile) {
        if (pend_p) flush();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (kind == kDescExit) {
          PROG(15000000 + j);
          break;
        }
        PROG(14000000 + j);
        __syncthreads();
        chase_window_9w(cargs, cw, cwi, sm, R);
        __syncthreads();
        continue;
      }
      const int qe = desc[s].qe, add = desc[s].cnt_add;
      int* const cp = desc[s].ctr;
      int* const cp2 = desc[s].ctr2;
      int* const call = desc[s].ctr_all;
      const bool left = desc[s].left;
      const TileRef t = desc[s].t;
      if (qe != last_qe) {
        if (pend_p && !mbar_test(&qfull, (unsigned)qe & 1)) flush();
        PROG(12000000 + qe);
#ifdef HQR_TIMING
        const long long cq0 = clock64();
#endif
        mbar_wait(&qfull, (unsigned)qe & 1, 4000000 + qe);
#ifdef HQR_TIMING
        if (lane == 0) {
          atomicAdd(&g_wait[7], (unsigned long long)(clock64() - cq0));
          atomicAdd(&g_wait[6], 1ull);
        }
#endif
        last_qe = qe;
      }
      PROG(13000000 + j);
      auto mid = [&]() {
        if (pend_p) flush();
      };
      // Q_W quarters: with two groups the warps of an SM sub-partition take opposite quarters (their
      // band shares add up to about half); otherwise the quarter rotates with the ring position
      const int qq = kGroups == 2 ? (i4 + 2 * q) & 3 : (i4 + j) & 3;
#ifdef HQR_TIMING
      const long long ck0 = clock64();
      const int ttask = desc[s].task;
      if (lane == 0 && ttask < 262144) atomicMin(&g_trec[ttask][6], gtime());
#endif
      if (left) consume_tile<KP, true>(Qs, Ps + s * SS, &empty[s], t, qq, lane, mid);
      else consume_tile<KP, false>(Qs, Ps + s * SS, &empty[s], t, qq, lane, mid);
#ifdef HQR_TIMING
      if (lane == 0) atomicAdd(&g_wait[11], (unsigned long long)(clock64() - ck0));
      if (lane == 0 && ttask < 262144) atomicMax(&g_trec[ttask][7], gtime());
#endif
      if (cp) {
        pend_p = cp;
        pend_p2 = cp2;
        pend_all = call;
        pend_n = add;
      }
    }
  }
#ifdef HQR_TIMING
  if (threadIdx.x == 0) atomicAdd(&g_wait[9], (unsigned long long)(clock64() - k_start));
#endif
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
cudaError_t launch_step_t(const StepArgs& base, const StepInfo* steps, int nsteps, const Task* tasks, int ntasks,
                          int task_base, const int32_t* dep_begin, const int2* deps, int* next_ctr, int* step_ctr,
                          int* task_ctr, const int* up_flags, const TensorMaps& tm, int max_kw, int num_sms,
                          cudaStream_t st, const int32_t* qidx, int ncrit, int crit_sms) {
  static size_t configured = 0;
  const size_t smem = step_smem<KP>(max_kw);
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(step_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int grid = std::max(1, std::min(ntasks, num_sms));
  if (crit_sms >= grid || ncrit <= 0 || ncrit >= ntasks) crit_sms = 0;  // both queues need CTAs and tasks
  step_kernel<KP><<<grid, kStepThreads, smem, st>>>(base, steps, nsteps, tasks, ntasks, task_base, dep_begin, deps,
                                                     next_ctr, step_ctr, task_ctr, up_flags, tm.left_H, tm.right_H,
                                                     tm.right_Z, qidx, ncrit, crit_sms);
  return cudaGetLastError();
}

}  // namespace

#ifdef HQR_TIMING
void debug_timing(int nsteps, bool reset) {
  static unsigned long long h[4096][4];
  if (reset) {
    for (int i = 0; i < 4096; ++i) { h[i][0] = h[i][1] = ~0ull; h[i][2] = h[i][3] = 0; }
    cudaMemcpyToSymbol(g_tim, h, sizeof(h));
    unsigned long long z[12] = {0};
    cudaMemcpyToSymbol(g_ctim, z, 8 * sizeof(unsigned long long));
    cudaMemcpyToSymbol(g_wait, z, sizeof(z));
    static unsigned long long wz[8192][6];
    cudaMemcpyToSymbol(g_wrec, wz, sizeof(wz));
    void* tz = nullptr;
    if (cudaGetSymbolAddress(&tz, g_trec) == cudaSuccess) {
      static unsigned long long tinit[262144][8];
      for (int i = 0; i < 262144; ++i) {
        for (int k = 0; k < 8; ++k) tinit[i][k] = 0;
        tinit[i][6] = ~0ull;
      }
      cudaMemcpy(tz, tinit, sizeof(tinit), cudaMemcpyHostToDevice);
    }
    return;
  }
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_tim, sizeof(h));
  double cs = 0, ce = 0, e = 0, gap = 0;
  int nc = 0;
  for (int s = 0; s < nsteps && s < 4096; ++s) {
    const double t0 = (double)h[s][0];
    e += (h[s][3] - t0) * 1e-3;
    if (s > 0) gap += ((double)h[s][0] - (double)h[s - 1][3]) * 1e-3;
    if (h[s][1] != ~0ull) {
      cs += (h[s][1] - t0) * 1e-3;
      ce += (h[s][2] - t0) * 1e-3;
      ++nc;
    }
  }
  unsigned long long ct[8], wt[12];
  cudaMemcpyFromSymbol(ct, g_ctim, sizeof(ct));
  cudaMemcpyFromSymbol(wt, g_wait, sizeof(wt));
  if (wt[9]) {
    const double T = (double)wt[9];  // summed CTA cycles
    fprintf(stderr, "hqr sm-time: chase %.3f | producer dep spins: chase-done %.3f left %.3f near-right %.3f "
            "qslot %.3f far/Z preds %.3f | consumer: pos %.3f data %.3f + Q_W %.3f (per warp, %.0f cycles "
            "per Q_W wait) busy %.3f (per warp)\n",
            wt[8] / T, wt[0] / T, wt[1] / T, wt[2] / T, wt[3] / T, wt[4] / T,
            wt[10] / T / (4.0 * kGroups), wt[5] / T / (4.0 * kGroups), wt[7] / T / (4.0 * kGroups), wt[6] ? (double)wt[7] / wt[6] : 0.0,
            wt[11] / T / (4.0 * kGroups));
  }
  if (ct[4]) {
    const double w = (double)ct[4] * kStepWarps, st = (double)ct[5] / (double)ct[4];
    fprintf(stderr, "hqr chase: %llu windows, %.1f steps each; cycles per step per warp: phase1 %.0f "
            "(vector load + house %.0f, beta / reflector stores %.0f, left application %.0f), "
            "sync1 %.0f, phase2 %.0f, sync2 %.0f\n", ct[4], st, (ct[0] + ct[6] + ct[7]) / w / st,
            ct[6] / w / st, ct[7] / w / st, ct[0] / w / st, ct[1] / w / st, ct[2] / w / st, ct[3] / w / st);
  }
  fprintf(stderr, "hqr timing: %d steps, mean launch %.1f us, chase start %.1f us, chase end %.1f us "
          "(%d steps with chases), mean gap between launches %.2f us\n", nsteps, e / nsteps,
          cs / std::max(nc, 1), ce / std::max(nc, 1), nc, gap / std::max(nsteps - 1, 1));
  if (const char* path = tuning_env("HQR_TIMING_WREC")) {  // per-window chase records for tools/
    static unsigned long long wr[8192][6];
    cudaMemcpyFromSymbol(wr, g_wrec, sizeof(wr));
    if (FILE* f = fopen(path, "w")) {
      fprintf(f, "window,start_ns,end_ns,b0,step,claim_ns,depok_ns\n");
      for (int i = 0; i < 8192; ++i)
        if (wr[i][1])
          fprintf(f, "%d,%llu,%llu,%llu,%llu,%llu,%llu\n", i, wr[i][0], wr[i][1], wr[i][2], wr[i][3], wr[i][4], wr[i][5]);
      fclose(f);
    }
    static unsigned long long tr[262144][8];
    cudaMemcpyFromSymbol(tr, g_trec, sizeof(tr));
    std::string tp = std::string(path) + ".tasks";
    if (FILE* f = fopen(tp.c_str(), "w")) {
      fprintf(f, "task,claim_ns,depok_ns,issued_ns,done_ns,type,win,step,cstart_ns,cend_ns,ntiles\n");
      for (int i = 0; i < 262144; ++i)
        if (tr[i][0])
          fprintf(f, "%d,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%llu\n", i, tr[i][0], tr[i][1], tr[i][2], tr[i][3],
                  tr[i][4] & 255, tr[i][4] >> 8, tr[i][5] & 0xffffffffull, tr[i][6], tr[i][7], tr[i][5] >> 32);
      fclose(f);
    }
  }
  for (int s = 0; s < nsteps && s < 4096; s += std::max(1, nsteps / 12)) {
    const double t0 = (double)h[s][0];
    fprintf(stderr, "  step %4d: launch %.1f us, chase %.1f .. %.1f us\n", s, (h[s][3] - t0) * 1e-3,
            h[s][1] != ~0ull ? (h[s][1] - t0) * 1e-3 : -1.0, h[s][2] ? (h[s][2] - t0) * 1e-3 : -1.0);
  }
}
#else
void debug_timing(int, bool) {}
#endif

#ifdef HQR_PROGRESS
void debug_progress_init() {
  static int* d = nullptr;
  if (d) return;
  const size_t count = 1024 * 16 * 65, bytes = count * sizeof(int);
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0, bytes);
  cudaMemcpyToSymbol(g_prog, &d, sizeof(d));
  int dev = 0;
  cudaGetDevice(&dev);
  const char* e = tuning_env("HQR_PROGRESS_SECS");
  const int secs = e ? atoi(e) : 20;
  std::thread([secs, dev, bytes, count] {
    std::this_thread::sleep_for(std::chrono::seconds(secs));
    cudaSetDevice(dev);
    int* h = (int*)malloc(bytes);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaError_t err = cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    fprintf(stderr, "hqr progress dump (%s): blocks whose producer did not exit, last events per warp\n",
            cudaGetErrorString(err));
    for (int b = 0; b < 148; ++b) {
      const int* pw = h + (b * 16 + kProducerWarp) * 65;
      const int last = pw[1 + ((pw[0] - 1) & 63)];
      if (last / 1000000 == 8) continue;
      for (int w = 0; w < kStepWarps; ++w) {
        const int* r = h + (b * 16 + w) * 65;
        fprintf(stderr, "b%d w%d n=%d:", b, w, r[0]);
        for (int k = r[0] > 40 ? r[0] - 40 : 0; k < r[0]; ++k) fprintf(stderr, " %d", r[1 + (k & 63)]);
        fprintf(stderr, "\n");
      }
    }
    fflush(stderr);
    _exit(3);
  }).detach();
}
#else
void debug_progress_init() {}
#endif

cudaError_t launch_step(const StepArgs& base, const StepInfo* steps, int nsteps, const Task* tasks, int ntasks,
                        int task_base, const int32_t* dep_begin, const int2* deps, int* next_ctr, int* step_ctr,
                        int* task_ctr, const int* up_flags, const TensorMaps& tm, int max_kw, int num_sms,
                        cudaStream_t st, const int32_t* qidx, int ncrit, int crit_sms) {
  if (!tm.valid) return cudaErrorNotSupported;
  if (!qidx) crit_sms = 0;
#define HQR_LS(K) return launch_step_t<K>(base, steps, nsteps, tasks, ntasks, task_base, dep_begin, deps, next_ctr, \
                                          step_ctr, task_ctr, up_flags, tm, max_kw, num_sms, st, qidx, ncrit, crit_sms)
  switch (base.KP) {
    case 32: HQR_LS(32);
    case 64: HQR_LS(64);
    case 96: HQR_LS(96);
    case 128: HQR_LS(128);
  }
#undef HQR_LS
  return cudaErrorInvalidValue;
}

// Host: the task queue of one step (L, Rn, C, Z, Rf).  Chunk sizes (tiles per task) per phase:
// cs.left, cs.near for L / Rn (they gate the next chase: small), cs.bulk for Z / Rf; the last
// cs.tail tiles of the queue use chunks of cs.tail_chunk so the CTAs finish together.
void build_step_tasks(const StepArgs& a, const WindowDesc* wins, int nwin, const WindowDesc* next_wins,
                      int nnext, int64_t sp, const ChunkSizes& cs, const int* lnear, const int64_t* rnear,
                      std::vector<Task>* out, int* nL, int* nRn) {
  const int NT = left_cols(a.KP), MT = right_rows(a.KP);
  // tiles [t_begin, t_end) of window `win` in tasks of `chunk` tiles
  auto add = [&](int type, int win, int64_t t_begin, int64_t t_end, int64_t r_lo, int64_t r_hi, int chunk) {
    for (int64_t t0 = t_begin; t0 < t_end; t0 += chunk) {
      Task T{};
      T.type = type; T.win = win; T.tile0 = (int32_t)t0; T.step = a.step;
      T.ntiles = (int32_t)std::min<int64_t>(chunk, t_end - t0);
      T.r_lo = r_lo; T.r_hi = r_hi;
      out->push_back(T);
    }
  };
  // re-split the last `tiles` tiles of the queue from index `from` on into chunks of `chunk` (same
  // order): the phase's end -- which the next phase waits for -- is then not one long task
  auto resplit = [&](size_t from, int tiles, int chunk) {
    int64_t acc = 0;
    size_t cut = out->size();
    while (cut > from && acc < tiles) acc += (*out)[--cut].ntiles;
    std::vector<Task> tail(out->begin() + cut, out->end());
    out->resize(cut);
    for (const Task& T : tail)
      for (int t0 = 0; t0 < T.ntiles; t0 += chunk) {
        Task U = T;
        U.tile0 = T.tile0 + t0;
        U.ntiles = std::min(chunk, T.ntiles - t0);
        out->push_back(U);
      }
  };
  const size_t base = out->size();
  // what the next step's chases read first: LeftNear, RightNear, then the chases themselves
  for (int i = 0; i < nwin; ++i) add(kTaskLeftNear, i, 0, lnear[i], 0, 0, cs.near_task);
  for (int i = 0; i < nwin; ++i) {
    const int64_t w0 = wins[i].w0;
    if (rnear[i] < w0) add(kTaskRightNear, i, 0, (w0 - rnear[i] + MT - 1) / MT, rnear[i], w0, cs.near_task);
  }
  auto chases = [&]() {
    for (int i = 0; i < nnext; ++i) {
      Task T{};
      T.type = kTaskChase; T.win = i; T.ntiles = 0; T.step = a.step;
      out->push_back(T);
    }
  };
  // the chases after the left tasks (their near inputs are done by then; a chase claimed right after
  // the near tasks idles its SM until they finish): measured 0.2-0.3 ms better at configs[2] / [3].
  // HQR_CHASE_POS=0: right after the near tasks (A/B knob, tuning builds only)
  static const int chase_pos = tuning_env("HQR_CHASE_POS") ? atoi(tuning_env("HQR_CHASE_POS")) : 1;
  if (chase_pos == 0) chases();
  const size_t l0 = out->size();
  for (int i = 0; i < nwin; ++i) {
    int64_t c, c_al, cnt;
    left_range_al(a, wins[i], c, c_al, cnt);
    add(kTaskLeft, i, lnear[i], (cnt + NT - 1) / NT, 0, 0, cs.left);
  }
  if (cs.ltail > 0) resplit(l0, cs.ltail, cs.phase_chunk);
  if (chase_pos == 1) chases();
  const size_t rn0 = out->size();
  for (int i = 0; i < nwin; ++i) {
    const int64_t hi = std::min<int64_t>(wins[i].w0, rnear[i]);
    if (sp < hi) add(kTaskRight, i, 0, (hi - sp + MT - 1) / MT, sp, hi, cs.near);
  }
  if (cs.ntail > 0) resplit(rn0, cs.ntail, cs.phase_chunk);
  *nL = *nRn = 0;
  for (size_t i = base; i < out->size(); ++i) {
    const int ty = (*out)[i].type;
    *nL += ty == kTaskLeft || ty == kTaskLeftNear;
    *nRn += ty == kTaskRight || ty == kTaskRightNear;
  }
  const size_t bulk0 = out->size();
  if (a.Z)
    for (int i = 0; i < nwin; ++i) add(kTaskZ, i, 0, (a.zrows + MT - 1) / MT, 0, 0, cs.bulk);
  for (int i = 0; i < nwin; ++i) {
    const int64_t hi = std::min<int64_t>(sp, wins[i].w0);
    if (hi > 0) add(kTaskRightFar, i, 0, (hi + MT - 1) / MT, 0, hi, cs.bulk);
  }
  if (cs.tail > 0) resplit(bulk0, cs.tail, cs.tail_chunk);  // the queue's last tiles
  for (size_t i = base; i < out->size(); ++i) (*out)[i].idx = (int32_t)(i - base);
}

}  // namespace hqr
