// hqr_api.cu -- the C ABI (include/hqr.h): validation, planning, workspace, kernel orchestration.
//
// Orchestration of one sweep:
//   a1  validate + pair shifts on the host (sigma_j = s + s', pi_j = s s'), upload 2*nb doubles;
//   a7  plan the wavefront (plan.hpp) and upload the window table once per distinct plan;
//   per wavefront step g:  chase(g)  ->  left(g)  ->  right+Z(g)   (one stream, in order)
//       chase  one CTA per window (a2 introduction + a3 in-window chase, chase.cu)
//       left   a4 Q^T H(W, right of W) for every window of the step (update.cu)
//       right  a5 H(above W, W) Q and a6 Z(:, W) Q for every window of the step (update.cu)
//   The step sequence is captured once into a CUDA graph per (plan, pointers) and replayed
//   (HQR_FLAG_NO_GRAPH launches directly; HQR_FLAG_PROFILE times each kernel with events).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include <nccl.h>

#include "../../include/hqr.h"
#include "dist.hpp"
#include "kernels.hpp"
#include "plan.hpp"
#include "step.hpp"

using hqr::Plan;
using hqr::StepArgs;
using hqr::WindowDesc;

namespace {

// Q slot sets of the sharded sweep: its deferred far-right / Z updates (low-priority stream) may
// trail the chases by up to kQSetsDist - 1 steps
constexpr int kQSetsDist = 32;

// (n, window, then ilo, ihi, nshifts of every block)
typedef std::vector<int64_t> PlanKey;

struct Blocks {
  std::vector<int64_t> ilo, ihi;
  std::vector<int> nshifts;
  bool sweeps = false;  // entries are successive sweeps of ONE block (hqr_sweeps), not disjoint blocks
  int count() const { return (int)ilo.size(); }
};

PlanKey plan_key(int64_t n, const Blocks& b, int window) {
  PlanKey k{n, window, b.sweeps ? -1 : 0};
  for (int i = 0; i < b.count(); ++i) {
    k.push_back(b.ilo[i]);
    k.push_back(b.ihi[i]);
    k.push_back(b.nshifts[i]);
  }
  return k;
}

struct GraphKey {
  PlanKey pk;   // plan key
  const double* H;
  const double* Z;
  bool operator<(const GraphKey& o) const {
    return std::tie(pk, H, Z) < std::tie(o.pk, o.H, o.Z);
  }
};

struct CachedGraph {
  cudaGraphExec_t exec;
  hqr_stats stats;
};

struct FusedTasks {            // task queues of every step for the fused step kernel
  std::vector<hqr::Task> tasks;          // all steps, in queue order
  std::vector<int32_t> begin;            // step g's tasks: [begin[g], begin[g+1])
  std::vector<hqr::StepInfo> steps;
  std::vector<hqr::WinDeps> wdeps;
  hqr::Task* d_tasks = nullptr;
  hqr::StepInfo* d_steps = nullptr;
  hqr::WinDeps* d_wdeps = nullptr;
  int* d_ctr = nullptr;                  // [8 claim counters][4 per step][kWinCtr per window][1 per task]
  size_t nctr = 0;
  std::vector<int32_t> dep_begin;        // task t's dependencies: deps[dep_begin[t] .. dep_begin[t+1])
  std::vector<int2> deps;                // (task index, completion count to wait for)
  int32_t* d_dep_begin = nullptr;
  int2* d_deps = nullptr;
  // two claim queues (DESIGN.md §6 "Critical SMs"): the chases and the near tasks the next chases
  // read (LeftNear, RightNear) in list order, then every other task in list order
  std::vector<int32_t> qidx;
  int32_t ncrit = 0;
  int32_t* d_qidx = nullptr;
  double chase_path_us = 0.0;            // estimated chase critical path of one chain (us)
  double flops = 0, bytes = 0;
};

// Precise task dependencies (DESIGN.md §6 "Task dependencies"): every update task and chase
// reads and writes one rectangle of H or Z (a left task: the window's rows x its column tiles; a
// right task: its row tiles x the window's columns; Z likewise; a chase: H(W, W)).  The task list is
// a valid sequential order (steps in order; within a step LeftNear, RightNear, Left, chases, Right,
// Z, far-right), so a task only has to wait for the last earlier task that touched each part of its
// rectangle.  Parts = square cells of c x c elements; a shared cell without a shared element only
// adds a wait (correct, but it can chain independent tasks: the windows of one wavefront step are
// only lag*s - k rows / columns apart -- 16 at k = 96 -- so the cell side is the largest power of
// two <= min(8, that gap)).  GEMM tasks also wait for their window's chase (the Q_W slot).
int build_task_deps(const Plan& P, int KP, int64_t n, int64_t zrows, bool has_z, FusedTasks* f) {
  int64_t gap = 8;
  for (int g = 0; g < P.nsteps; ++g)
    for (int i = P.step_begin[g] + 1; i < P.step_begin[g + 1]; ++i)
      gap = std::min<int64_t>(gap, (int64_t)P.windows[i].w0 - P.windows[i - 1].w1 - 1);
  int cell = 8;
  while (cell > 1 && cell > gap) cell >>= 1;
  const int kDepRows = cell, kDepCols = cell;
  const int64_t rc = (n + kDepRows - 1) / kDepRows, cc = (n + kDepCols - 1) / kDepCols;
  const int64_t zrc = (zrows + kDepRows - 1) / kDepRows;
  std::vector<int32_t> lastH((size_t)(rc * cc), -1), lastZ(has_z ? (size_t)(zrc * cc) : 0, -1);
  std::vector<int32_t> chase_task(P.windows.size(), -1);  // window -> its chase task
  const int NT = hqr::left_cols(KP), MT = hqr::right_rows(KP);
  f->dep_begin.assign(f->tasks.size() + 1, 0);
  f->deps.clear();
  std::vector<int32_t> seen;
  StepArgs a{};
  a.n = n; a.lc0 = 0; a.lc1 = n;
  auto target = [&](int32_t d) {
    const hqr::Task& D = f->tasks[d];
    return D.type == hqr::kTaskChase ? 1 : 4 * D.ntiles;
  };
  for (int g = 0; g < P.nsteps; ++g) {
    for (int32_t t = f->begin[g]; t < f->begin[g + 1]; ++t) {
      const hqr::Task& T = f->tasks[t];
      f->dep_begin[t] = (int32_t)f->deps.size();
      seen.clear();
      std::vector<int32_t>* grid = &lastH;
      int64_t r0, r1, c0, c1;  // rectangle [r0, r1) x [c0, c1)
      if (T.type == hqr::kTaskChase) {
        const int wi = P.step_begin[g + 1] + T.win;
        const WindowDesc& w = P.windows[wi];
        chase_task[wi] = t;
        r0 = c0 = w.w0;
        r1 = c1 = (int64_t)w.w1 + 1;
      } else {
        const int wi = P.step_begin[g] + T.win;
        const WindowDesc& w = P.windows[wi];
        if (chase_task[wi] >= 0) seen.push_back(chase_task[wi]);  // the Q_W slot (step 0: own launch)
        if (T.type == hqr::kTaskLeft || T.type == hqr::kTaskLeftNear) {
          int64_t c, c_al, cnt;  // (the columns the tiles store: from c on)
          hqr::left_range_al(a, w, c, c_al, cnt);
          r0 = w.w0; r1 = (int64_t)w.w1 + 1;
          c0 = std::max<int64_t>(c, c_al + (int64_t)NT * T.tile0);
          c1 = std::min<int64_t>(c_al + (int64_t)NT * (T.tile0 + T.ntiles), n);
        } else if (T.type == hqr::kTaskZ) {
          grid = &lastZ;
          r0 = (int64_t)MT * T.tile0;
          r1 = std::min<int64_t>((int64_t)MT * (T.tile0 + T.ntiles), zrows);
          c0 = w.w0; c1 = (int64_t)w.w1 + 1;
        } else {  // right (near / rest / far)
          r0 = T.r_lo + (int64_t)MT * T.tile0;
          r1 = std::min<int64_t>(T.r_lo + (int64_t)MT * (T.tile0 + T.ntiles), T.r_hi);
          c0 = w.w0; c1 = (int64_t)w.w1 + 1;
        }
      }
      if (r1 > r0 && c1 > c0) {
        for (int64_t cj = c0 / kDepCols; cj <= (c1 - 1) / kDepCols; ++cj)
          for (int64_t ri = r0 / kDepRows; ri <= (r1 - 1) / kDepRows; ++ri) {
            int32_t& cell = (*grid)[(size_t)(cj * (grid == &lastZ ? zrc : rc) + ri)];
            if (cell >= 0 && (seen.empty() || seen.back() != cell)) seen.push_back(cell);
            cell = t;
          }
      }
      std::sort(seen.begin(), seen.end());
      seen.erase(std::unique(seen.begin(), seen.end()), seen.end());
      for (int32_t d : seen) f->deps.push_back(make_int2(d, target(d)));
    }
  }
  f->dep_begin[f->tasks.size()] = (int32_t)f->deps.size();
  return 0;
}

struct CachedPlan {
  Plan plan;
  WindowDesc* d_wins = nullptr;
  int KP = 0;
  double flops_chase = -1.0;  // in-window chase flops (computed once per plan)
  std::unique_ptr<FusedTasks> fused[2];  // [Z absent, Z present]
};

struct State {
  bool ready = false;
  int device = 0, rank = 0, world = 1, flags = 0, num_sms = 0;
  cudaStream_t stream = nullptr;   // stream A: chase -> left -> right (high priority)
  cudaStream_t zstream = nullptr;  // stream B: Z updates (low priority)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_in = nullptr;     // entry: the library stream waits for the caller's legacy stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_q[hqr::kQSets] = {}, ev_z[hqr::kQSets] = {};
  cudaStream_t cstream = nullptr;  // sharded sweep: NCCL broadcasts (comm stream)
  cudaStream_t qzs[3] = {};        // QZ sweep: the step's four update launches side by side
  cudaEvent_t qz_fork = nullptr, qz_join[3] = {};
  cudaEvent_t dev_chase[kQSetsDist] = {}, dev_bc[kQSetsDist] = {}, dev_bulk[kQSetsDist] = {};
  double* d_coef = nullptr;
  size_t coef_cap = 0;
  double* d_aft = nullptr;       // aftermath flags of the last single-GPU sweep (int8 per row)
  size_t aft_cap = 0;            // (in doubles)
  int64_t aft_n = 0;             // n of the sweep that wrote them (0: none)
  std::vector<int64_t> user_cb, user_rb;  // hqr_config shard bounds (empty: sqrt-balanced default)
  int64_t user_n = 0;            // the n they are for
  int window_max = 0;            // hqr_config window cap (0: HQR_MAX_WINDOW)
  double* d_q = nullptr;
  size_t q_cap = 0;
  int* d_upflags = nullptr;      // host-buffer sweeps: per upload chunk, 1 once on the device
  size_t upflags_cap = 0;
  double* d_wstats = nullptr;    // per plan window: executed DMMA work units (record_band)
  size_t wstats_cap = 0;
  const void* wstats_plan = nullptr;  // plan (CachedPlan) the last single-GPU sweep recorded
  int64_t wstats_n = 0;
  bool wstats_z = false;
  double* d_hstage = nullptr;
  double* d_zstage = nullptr;
  size_t stage_cap = 0;
  int64_t hstage_zero_n = -1;  // d_hstage is zero below the subdiagonal of the n x n layout (overlapped uploads)
  std::map<PlanKey, std::unique_ptr<CachedPlan>> plans;
  std::map<GraphKey, CachedGraph> graphs;
  std::vector<cudaEvent_t> prof_events;
  cudaStream_t cin = nullptr, cout = nullptr;  // host-buffer sweeps: copies in / out
  std::vector<cudaEvent_t> io_events;          // their synchronisation (no timing)
  hqr_stats stats{};
  ncclComm_t comm = nullptr;       // world > 1
  // virtual shards (hqr_sweep_virtual): library-owned per-rank buffers on this one GPU
  std::vector<double*> vH, vZ;
  std::vector<size_t> vH_cap, vZ_cap;
};

State g;

int cuerr(cudaError_t e) { return e == cudaSuccess ? 0 : 1000 + (int)e; }
int ncclerr(ncclResult_t e) { return e == ncclSuccess ? 0 : 2000 + (int)e; }
#define NK(x)                                   \
  do {                                          \
    ncclResult_t e_ = (x);                      \
    if (e_ != ncclSuccess) return ncclerr(e_);  \
  } while (0)
#define CK(x)                                   \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return cuerr(e_);    \
  } while (0)

// a1: argument validation that does not touch matrix values (shared by the sweeps / plan queries)
int validate_block(int64_t n, int64_t ilo, int64_t ihi, const double* sr, const double* si,
                   int nshifts, bool check_shifts) {
  if (ilo < 0 || ilo > ihi) return -4;
  if (ihi >= n || ihi - ilo + 1 < 3) return -5;
  const int64_t N = ihi - ilo + 1;
  if (nshifts < 2 || (nshifts & 1) || nshifts > N) return -8;
  if (check_shifts) {
    if (!sr) return -6;
    if (!si) return -7;
    for (int i = 0; i < nshifts; ++i)
      if (!std::isfinite(sr[i]) || !std::isfinite(si[i])) return -6;
    for (int j = 0; j < nshifts / 2; ++j) {
      double r0 = sr[2 * j], r1 = sr[2 * j + 1], i0 = si[2 * j], i1 = si[2 * j + 1];
      bool real_pair = (i0 == 0.0 && i1 == 0.0);
      bool conj_pair = (i0 != 0.0 && r0 == r1 && i0 == -i1);
      if (!real_pair && !conj_pair) return -7;
    }
  }
  return 0;
}

int validate_blocks(int64_t n, const Blocks& b, const double* sr, const double* si, int window,
                    bool check_shifts) {
  if (n < 1) return -3;
  if (b.count() < 1) return -4;
  int64_t off = 0;
  for (int i = 0; i < b.count(); ++i) {
    if (i > 0 && !b.sweeps && b.ilo[i] <= b.ihi[i - 1]) return -4;  // ascending, disjoint
    int rc = validate_block(n, b.ilo[i], b.ihi[i], sr ? sr + off : nullptr, si ? si + off : nullptr,
                            b.nshifts[i], check_shifts);
    if (rc) return rc;
    off += b.nshifts[i];
  }
  if (window <= 0) return -9;
  return 0;
}

int get_plan(int64_t n, const Blocks& b, int window, CachedPlan** out, bool upload) {
  PlanKey key = plan_key(n, b, window);
  auto it = g.plans.find(key);
  if (it == g.plans.end()) {
    auto cp = std::make_unique<CachedPlan>();
    const int kmax = g.window_max > 0 ? g.window_max : hqr::kMaxWindow;
    int rc = b.sweeps ? hqr::make_plan_sweeps(n, b.ilo[0], b.ihi[0], b.count(), b.nshifts.data(), window,
                                              kmax, &cp->plan)
                      : hqr::make_plan_multi(n, b.count(), b.ilo.data(), b.ihi.data(), b.nshifts.data(),
                                             window, kmax, &cp->plan);
    if (rc) return rc;
    cp->KP = hqr::padded_kp(cp->plan.max_kw);
    it = g.plans.emplace(key, std::move(cp)).first;
  }
  CachedPlan* cp = it->second.get();
  if (upload && !cp->d_wins) {
    size_t bytes = cp->plan.windows.size() * sizeof(WindowDesc);
    CK(cudaMalloc(&cp->d_wins, bytes));
    CK(cudaMemcpy(cp->d_wins, cp->plan.windows.data(), bytes, cudaMemcpyHostToDevice));
  }
  *out = cp;
  return 0;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int ensure(double** p, size_t* cap, size_t count) {
  if (*cap >= count) return 0;
  // captured graphs hold the old pointer: drop them (after the stream has drained)
  if (*p) {
    CK(cudaStreamSynchronize(g.stream));
    for (auto& kv : g.graphs) cudaGraphExecDestroy(kv.second.exec);
    g.graphs.clear();
  }
  if (*p) CK(cudaFree(*p));
  *p = nullptr;
  *cap = 0;
  CK(cudaMalloc(p, count * sizeof(double)));
  *cap = count;
  return 0;
}

// a1: the shift pairs go to the device as they are -- coef[4j..4j+3] = (re_2j, re_2j+1, im_2j,
// im_2j+1); the chase forms sigma = s + s' and pi = s s' from them on scaled inputs (R1, R3, R15)
int upload_coef(const double* sr, const double* si, int nb) {
  std::vector<double> coef(4 * (size_t)nb);
  for (int j = 0; j < nb; ++j) {
    coef[4 * j] = sr[2 * j];
    coef[4 * j + 1] = sr[2 * j + 1];
    coef[4 * j + 2] = si[2 * j];
    coef[4 * j + 3] = si[2 * j + 1];
  }
  int rc = ensure(&g.d_coef, &g.coef_cap, coef.size());
  if (rc) return rc;
  CK(cudaMemcpyAsync(g.d_coef, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice, g.stream));
  return 0;
}

// Entry of every sweep: the library stream (non-blocking) waits for the work the caller has
// queued on the legacy default stream (e.g. torch's default stream still writing H or Z).
int wait_for_caller() {
  CK(cudaEventRecord(g.ev_in, cudaStreamLegacy));
  CK(cudaStreamWaitEvent(g.stream, g.ev_in, 0));
  return 0;
}

cudaEvent_t prof_event(size_t i) {
  while (g.prof_events.size() <= i) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g.prof_events.push_back(e);
  }
  return g.prof_events[i];
}

// Enqueue every step of the sweep.  Stream A (high priority) carries the chain of dependent work
// chase(g) -> left(g) -> right(g); the Z update, which nothing else reads ("a completely
// separate subgraph"), runs on stream B (low priority, "min_prio") as soon as chase(g) has
// produced the step's factors, overlapping the next steps.  kQSets rotating Q slot sets let Z trail
// the chase by up to kQSets-1 steps.  prof: one stream, events around every launch.
int enqueue_sweep(const CachedPlan& cp, double* H, double* Z, int64_t n, bool prof,
                  std::vector<int>* classes, hqr_stats* st) {
  const Plan& P = cp.plan;
  const bool split = (Z != nullptr) && !prof;
  cudaStream_t A = g.stream, B = split ? g.zstream : g.stream;
  StepArgs a{};
  a.H = H; a.Z = Z; a.n = n; a.ilo = P.ilo; a.ihi = P.ihi;
  a.hcol0 = 0; a.lc0 = 0; a.lc1 = n; a.zrows = n; a.ldz = n;
  a.wins = cp.d_wins; a.coef = g.d_coef; a.qslots = g.d_q; a.KP = cp.KP; a.wstats = g.d_wstats;
  a.QLD = hqr::pad_ld(cp.KP);
  a.aftermath = reinterpret_cast<signed char*>(g.d_aft);
  size_t ev = 0;
  static const bool dbg_sync = hqr::tuning_env("HQR_DEBUG_SYNC") != nullptr;  // debugging builds: sync after launches
  auto mark = [&](int cls) {
    if (dbg_sync) {
      cudaError_t e = cudaStreamSynchronize(A);
      if (e != cudaSuccess) fprintf(stderr, "hqr: CUDA error %d before mark class %d\n", (int)e, cls);
    }
    if (!prof) return;
    cudaEventRecord(prof_event(ev++), A);
    if (classes) classes->push_back(cls);
  };
  hqr::TensorMaps tm;
  CK(hqr::make_tensor_maps(&tm, H, n, Z, n, n, n, cp.KP));
  if (dbg_sync) {
    const unsigned long long* q = reinterpret_cast<const unsigned long long*>(&tm.left_H);
    fprintf(stderr, "hqr: tensor maps valid=%d KP=%d H=%p map@%p %llx %llx %llx\n", (int)tm.valid, cp.KP,
            (const void*)H, (const void*)&tm.left_H, q[0], q[1], q[2]);
  }
  if (split) {
    CK(cudaEventRecord(g.ev_fork, A));
    CK(cudaStreamWaitEvent(B, g.ev_fork, 0));
  }
  for (int s = 0; s < P.nsteps; ++s) {
    const int set = s % hqr::kQSets;
    a.win_begin = P.step_begin[s];
    a.win_count = P.step_begin[s + 1] - P.step_begin[s];
    a.slot_offset = set * P.nchains;
    const WindowDesc* hw = P.windows.data() + a.win_begin;
    if (split && s >= hqr::kQSets) CK(cudaStreamWaitEvent(A, g.ev_z[set], 0));
    mark(0);
    CK(hqr::launch_chase(a, P.max_kw, P.max_nbc, A));
    mark(-1);
    st->launches_chase++;
    int64_t items;
    double fl, by;
    if (split) {
      CK(cudaEventRecord(g.ev_q[set], A));
      CK(cudaStreamWaitEvent(B, g.ev_q[set], 0));
      StepArgs az = a;
      az.right_mode = 2;
      CK(hqr::launch_right(az, hw, g.num_sms, tm, B, &items, &fl, &by));
      if (items) st->launches_right++;
      st->flops_update += fl;
      st->bytes_update += by;
      CK(cudaEventRecord(g.ev_z[set], B));
    }
    mark(1);
    CK(hqr::launch_left(a, hw, g.num_sms, tm, A, &items, &fl, &by));
    mark(-1);
    if (items) st->launches_left++;
    st->flops_update += fl;
    st->bytes_update += by;
    mark(2);
    StepArgs ar = a;
    ar.right_mode = split ? 1 : 0;
    CK(hqr::launch_right(ar, hw, g.num_sms, tm, A, &items, &fl, &by));
    mark(-1);
    if (items) st->launches_right++;
    st->flops_update += fl;
    st->bytes_update += by;
  }
  if (split) {
    CK(cudaEventRecord(g.ev_join, B));
    CK(cudaStreamWaitEvent(A, g.ev_join, 0));
  }
  st->steps = P.nsteps;
  st->windows = (int64_t)P.windows.size();
  st->kernels_launched = st->launches_chase + st->launches_left + st->launches_right;
  return 0;
}

// Fused path (single GPU, TMA-capable layout): chase(0), then one step-kernel launch per step that
// runs the step's updates and the next step's chase from a prioritised task queue (step.cu).
// Task chunk sizes; HQR_CHUNK="left,near,bulk,tail,tail_chunk" overrides them (tuning builds only).
hqr::ChunkSizes chunk_sizes() {
  hqr::ChunkSizes cs;
  if (const char* e = hqr::tuning_env("HQR_CHUNK")) {
    int v[5];
    if (sscanf(e, "%d,%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3], &v[4]) == 5 && v[0] > 0 && v[1] > 0 &&
        v[2] > 0 && v[3] >= 0 && v[4] > 0) {
      cs.left = v[0]; cs.near = v[1]; cs.bulk = v[2]; cs.tail = v[3]; cs.tail_chunk = v[4];
    }
  }
  if (const char* e = hqr::tuning_env("HQR_NEAR_TASK")) cs.near_task = std::max(1, atoi(e));  // tuning builds
  if (const char* e = hqr::tuning_env("HQR_PHASE_TAIL")) {  // tuning builds: "ltail,ntail,chunk"
    int v[3];
    if (sscanf(e, "%d,%d,%d", &v[0], &v[1], &v[2]) == 3 && v[0] >= 0 && v[1] >= 0 && v[2] > 0) {
      cs.ltail = v[0]; cs.ntail = v[1]; cs.phase_chunk = v[2];
    }
  }
  return cs;
}

int get_fused(CachedPlan& cp, bool has_z, int64_t n, FusedTasks** out) {
  auto& slot = cp.fused[has_z ? 1 : 0];
  if (!slot) {
    auto f = std::make_unique<FusedTasks>();
    const Plan& P = cp.plan;
    // sp(g): smallest first row of any window of a later step (suffix minimum), rounded down to a
    // multiple of 8 like the RightNear rows below: the right tiles (MT rows from these starts) then
    // keep to the 8-row cells of the dependency grid (see left_range_al)
    std::vector<int64_t> sp(P.nsteps, INT64_MAX);
    int64_t run = INT64_MAX;
    for (int g = P.nsteps - 1; g >= 0; --g) {
      sp[g] = (run == INT64_MAX) ? run : (run & ~(int64_t)7);
      for (int i = P.step_begin[g]; i < P.step_begin[g + 1]; ++i) run = std::min<int64_t>(run, P.windows[i].w0);
    }
    StepArgs a{};
    a.n = n; a.hcol0 = 0; a.lc0 = 0; a.lc1 = n; a.zrows = n; a.ldz = n; a.KP = cp.KP;
    a.Z = has_z ? reinterpret_cast<double*>(1) : nullptr;  // only tested for presence
    const int nwin_all = (int)P.windows.size();
    f->wdeps.assign(nwin_all, hqr::WinDeps{{-1, -1, -1}, 0, 0, 0, 0, -1, -1, -1, {0, 0}});
    const int NT = hqr::left_cols(cp.KP);
    for (int g = 0; g < P.nsteps; ++g) {
      f->begin.push_back((int32_t)f->tasks.size());
      const int b0 = P.step_begin[g];
      const WindowDesc* w = P.windows.data() + b0;
      const int nw = P.step_begin[g + 1] - b0;
      const WindowDesc* wn = (g + 1 < P.nsteps) ? P.windows.data() + P.step_begin[g + 1] : nullptr;
      const int nn = (g + 1 < P.nsteps) ? P.step_begin[g + 2] - P.step_begin[g + 1] : 0;
      // near tasks (step.hpp): for every window W' of step g+1, the step-g windows meeting it
      std::vector<int64_t> xcol(nw), rnear(nw, INT64_MAX);
      std::vector<int> lnear(nw, 0);
      for (int i = 0; i < nw; ++i) xcol[i] = w[i].w1;
      for (int j = 0; j < nn; ++j) {
        const WindowDesc& W2 = wn[j];
        hqr::WinDeps& D2 = f->wdeps[P.step_begin[g + 1] + j];
        for (int i = 0; i < nw; ++i) {
          if (!(w[i].w0 <= W2.w1 && W2.w0 <= w[i].w1)) continue;
          if (w[i].w0 <= W2.w0) {
            if (D2.c_pred >= 0) return -103;
            D2.c_pred = b0 + i;
            xcol[i] = std::max<int64_t>(xcol[i], W2.w1);
          } else {
            if (D2.c_below >= 0) return -103;
            D2.c_below = b0 + i;
            rnear[i] = std::min<int64_t>(rnear[i], std::max<int64_t>((int64_t)W2.w0 & ~(int64_t)7, sp[g]));
          }
        }
      }
      for (int i = 0; i < nw; ++i) {
        if (rnear[i] >= w[i].w0) continue;
        for (int k = 0; k < nw; ++k)  // the window whose rows meet the RightNear rows
          if (k != i && w[k].w0 < w[i].w0 && w[k].w1 >= rnear[i]) {
            if (f->wdeps[b0 + i].rn_over >= 0) return -103;
            f->wdeps[b0 + i].rn_over = b0 + k;
            xcol[k] = std::max<int64_t>(xcol[k], w[i].w1);
          }
      }
      for (int i = 0; i < nw; ++i) {
        int64_t c, c_al, cnt;
        hqr::left_range_al(a, w[i], c, c_al, cnt);
        const int64_t tiles = (cnt + NT - 1) / NT;
        lnear[i] = (int)std::min<int64_t>(tiles, (xcol[i] + 1 - c_al + NT - 1) / NT);
      }
      int nl, nrn;
      a.step = g;
      hqr::build_step_tasks(a, w, nw, wn, nn, sp[g], chunk_sizes(), lnear.data(), rnear.data(), &f->tasks,
                            &nl, &nrn);
      hqr::StepInfo S{};
      S.win_begin = P.step_begin[g];
      S.win_count = nw;
      S.slot_offset = (g % hqr::kQSets) * P.nchains;
      S.nL = nl;
      S.nRn = nrn;
      for (int i = f->begin.back(); i < (int)f->tasks.size(); ++i) {
        const hqr::Task& T = f->tasks[i];
        if (T.type == hqr::kTaskChase) continue;
        hqr::WinDeps& D = f->wdeps[S.win_begin + T.win];
        S.ntiles += T.ntiles;
        if (T.type == hqr::kTaskLeft || T.type == hqr::kTaskLeftNear) S.nLt += T.ntiles;
        if (T.type == hqr::kTaskRight || T.type == hqr::kTaskRightNear) S.nRnt += T.ntiles;
        if (T.type == hqr::kTaskLeftNear) D.lnear += T.ntiles;
        if (T.type == hqr::kTaskRightNear) D.rnear += T.ntiles;
        if (T.type == hqr::kTaskRightFar) D.rftiles += T.ntiles;
        if (T.type == hqr::kTaskZ) D.ztiles += T.ntiles;
      }
      f->steps.push_back(S);
      for (int i = 0; i < nw; ++i) {
        const double kw = w[i].w1 - w[i].w0 + 1;
        const double rows = (double)(n - 1 - w[i].w1) + (double)w[i].w0 + (has_z ? (double)n : 0.0);
        f->flops += 2.0 * kw * kw * rows;
        f->bytes += 16.0 * kw * rows;
        // windows of the previous step whose columns meet this one (far-right / Z ordering)
        if (g > 0) {
          int np = 0;
          for (int k = P.step_begin[g - 1]; k < P.step_begin[g]; ++k)
            if (P.windows[k].w0 <= w[i].w1 && w[i].w0 <= P.windows[k].w1) {
              if (np == 3) return -102;  // cannot happen for planner windows (checked)
              f->wdeps[P.step_begin[g] + i].pred[np++] = k;
            }
        }
      }
    }
    f->begin.push_back((int32_t)f->tasks.size());
    // host-buffer sweeps: the last upload chunk (H rows / Z columns) step g's tasks and the chase
    // of step g+1 touch: max w1 over the windows of steps g and g+1 (cumulative)
    {
      int64_t reach = 0;
      for (int g2 = 0; g2 < P.nsteps; ++g2) {
        for (int s2 = g2; s2 <= std::min(g2 + 1, P.nsteps - 1); ++s2)
          for (int i = P.step_begin[s2]; i < P.step_begin[s2 + 1]; ++i) reach = std::max<int64_t>(reach, P.windows[i].w1);
        f->steps[g2].up_need = (int32_t)(reach / hqr::kUploadChunk);
      }
    }
    {
      int rcd = build_task_deps(P, cp.KP, n, n, has_z, f.get());
      if (rcd) return rcd;
      if (const char* path = hqr::tuning_env("HQR_DUMP_DEPS")) {  // tuning builds: the task graph for tools/
        if (FILE* fd = fopen(path, "w")) {
          fprintf(fd, "task,type,step,win,ntiles,deps\n");
          for (size_t t = 0; t < f->tasks.size(); ++t) {
            const hqr::Task& T = f->tasks[t];
            fprintf(fd, "%zu,%d,%d,%d,%d,", t, T.type, T.step, T.win, T.ntiles);
            for (int d = f->dep_begin[t]; d < f->dep_begin[t + 1]; ++d) fprintf(fd, "%d:%d ", f->deps[d].x, f->deps[d].y);
            fprintf(fd, "\n");
          }
          fclose(fd);
        }
      }
      CK(cudaMalloc(&f->d_dep_begin, f->dep_begin.size() * sizeof(int32_t)));
      CK(cudaMemcpy(f->d_dep_begin, f->dep_begin.data(), f->dep_begin.size() * sizeof(int32_t),
                    cudaMemcpyHostToDevice));
      CK(cudaMalloc(&f->d_deps, std::max<size_t>(f->deps.size(), 1) * sizeof(int2)));
      if (!f->deps.empty())
        CK(cudaMemcpy(f->d_deps, f->deps.data(), f->deps.size() * sizeof(int2), cudaMemcpyHostToDevice));
    }
    CK(cudaMalloc(&f->d_tasks, f->tasks.size() * sizeof(hqr::Task)));
    CK(cudaMemcpy(f->d_tasks, f->tasks.data(), f->tasks.size() * sizeof(hqr::Task), cudaMemcpyHostToDevice));
    {  // the critical queue (chases, LeftNear, RightNear) and the bulk queue, each in list order
      f->qidx.clear();
      for (int pass = 0; pass < 2; ++pass)
        for (int32_t i = 0; i < (int32_t)f->tasks.size(); ++i) {
          const int ty = f->tasks[i].type;
          const bool crit = ty == hqr::kTaskChase || ty == hqr::kTaskLeftNear || ty == hqr::kTaskRightNear;
          if (crit == (pass == 0)) f->qidx.push_back(i);
          if (pass == 0 && crit) ++f->ncrit;
        }
      CK(cudaMalloc(&f->d_qidx, f->qidx.size() * sizeof(int32_t)));
      CK(cudaMemcpy(f->d_qidx, f->qidx.data(), f->qidx.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      // one chain's chase path: its windows' steps back to back (~2700 cycles per step)
      double steps = 0.0;
      for (const WindowDesc& w : P.windows) steps += (double)(w.t1 - w.t0 + 1);
      f->chase_path_us = steps / std::max(1, P.nchains) * 1.4;
    }
    CK(cudaMalloc(&f->d_steps, f->steps.size() * sizeof(hqr::StepInfo)));
    CK(cudaMemcpy(f->d_steps, f->steps.data(), f->steps.size() * sizeof(hqr::StepInfo), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&f->d_wdeps, f->wdeps.size() * sizeof(hqr::WinDeps)));
    CK(cudaMemcpy(f->d_wdeps, f->wdeps.data(), f->wdeps.size() * sizeof(hqr::WinDeps), cudaMemcpyHostToDevice));
    f->nctr = 8 + 4 * (size_t)P.nsteps + hqr::kWinCtr * (size_t)nwin_all + f->tasks.size();  // + per task
    CK(cudaMalloc(&f->d_ctr, f->nctr * sizeof(int)));
    slot = std::move(f);
  }
  *out = slot.get();
  return 0;
}

cudaEvent_t io_event(size_t i) {
  while (g.io_events.size() <= i) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    g.io_events.push_back(e);
  }
  return g.io_events[i];
}

// Stream memory operations (driver API, fetched through the runtime): a copy stream tells the
// persistent kernel which chunks have arrived, and waits for the kernel's step counters before
// copying finished columns back.
typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
int stream_value_fns(StreamValueFn* wr, StreamValueFn* wt) {
  static StreamValueFn w = nullptr, t = nullptr;
  if (!w || !t) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return 1000 + (int)cudaErrorNotSupported;
    w = reinterpret_cast<StreamValueFn>(p);
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return 1000 + (int)cudaErrorNotSupported;
    t = reinterpret_cast<StreamValueFn>(p);
  }
  *wr = w;
  *wt = t;
  return 0;
}
#define CU(call) do { CUresult r_ = (call); if (r_ != CUDA_SUCCESS) return 1000 + (int)cudaErrorUnknown; } while (0)

// Host-buffer sweep (the e2e path): the copies overlap the persistent sweep kernel instead of
// bracketing it.  Windows move down the diagonal, so step s touches H only in rows [0, max w1 + 1)
// of its windows (left updates: window rows, all columns right; right updates: rows above; chase:
// the window) and Z only in columns [0, max w1 + 1).  Chunk k (H rows and Z columns
// [512 k, 512 k + 512)) goes up on one copy stream, then a flag is written (cuStreamWriteValue32);
// the kernel's producer waits for the flag of the last chunk a task's step needs
// (StepInfo::up_need).  Column c of H and Z is final once every step that touches it is done (every
// later window starts below c), so a second copy stream waits for the steps' completion counters
// (cuStreamWaitValue32) and copies finished column chunks down during the sweep; of H only the
// rows [0, c1 + 1) of a column chunk [c0, c1) come back, and of a row chunk [r, r + 512) only the
// columns [r - 1, n) go up (below the subdiagonal H is zero in and out: those entries are zeroed on
// the device, never read from the caller's buffer).
struct IoPlan {
  double* Hh = nullptr;  // caller's host H (nullptr: H is device-resident)
  double* Zh = nullptr;  // caller's host Z (nullptr: device-resident or absent)
  double* dH = nullptr;
  double* dZ = nullptr;
  int64_t n = 0;
  int* d_flags = nullptr;   // per chunk: 1 once it is on the device
  std::vector<int64_t> fin;  // after step s (and every earlier step), columns [0, fin[s]) are final
  int64_t chunk = hqr::kUploadChunk;
  int64_t h2d = 0, d2h = 0;
  StreamValueFn write_value = nullptr, wait_value = nullptr;

  int64_t nchunks() const { return (n + chunk - 1) / chunk; }
  void plan(const Plan& P) {
    fin.assign(P.nsteps, n);
    int64_t run = n;
    for (int s = P.nsteps - 1; s >= 0; --s) {
      fin[s] = run;  // min w0 over the windows of later steps
      for (int i = P.step_begin[s]; i < P.step_begin[s + 1]; ++i) run = std::min<int64_t>(run, P.windows[i].w0);
    }
  }
  int upload(cudaStream_t A, int64_t first_rows) {  // before chase(0); A waits for its rows
    int rc = stream_value_fns(&write_value, &wait_value);
    if (rc) return rc;
    const size_t col = (size_t)n * sizeof(double);
    CK(cudaStreamWaitEvent(g.cin, g.ev0, 0));
    CK(cudaMemsetAsync(d_flags, 0, (size_t)nchunks() * sizeof(int), g.cin));
    h2d = 0;
    // zeros below the subdiagonal of the staging buffer: set once per (buffer, n) and kept (the sweep
    // writes exact zeros there), all before the first copy -- a memset is a kernel, and a kernel
    // queued behind the copies the running sweep waits for could not find an SM
    if (Hh && g.hstage_zero_n != n) {
      for (int64_t k = 1; k < nchunks(); ++k) {
        const int64_t c = k * chunk, w = std::min(chunk, n - c);
        CK(cudaMemset2DAsync(dH + c, col, 0, (size_t)w * sizeof(double), (size_t)(c - 1), g.cin));
      }
      g.hstage_zero_n = n;
    }
    for (int64_t k = 0; k < nchunks(); ++k) {
      const int64_t c = k * chunk, w = std::min(chunk, n - c);
      if (Hh) {  // rows [c, c + w): columns [c - 1, n) up (below them: the zeros above)
        const int64_t j0 = std::max<int64_t>(c - 1, 0);
        CK(cudaMemcpy2DAsync(dH + c + j0 * n, col, Hh + c + j0 * n, col, (size_t)w * sizeof(double),
                             (size_t)(n - j0), cudaMemcpyHostToDevice, g.cin));
        h2d += w * (n - j0) * (int64_t)sizeof(double);
      }
      if (Zh) {
        CK(cudaMemcpyAsync(dZ + c * n, Zh + c * n, col * w, cudaMemcpyHostToDevice, g.cin));
        h2d += (int64_t)(col * w);
      }
      CU(write_value((CUstream)g.cin, (CUdeviceptr)(d_flags + k), 1, 0));
      if (c <= first_rows && first_rows < c + w) {  // chase(0) is a separate launch: an event
        cudaEvent_t e = io_event(0);
        CK(cudaEventRecord(e, g.cin));
        CK(cudaStreamWaitEvent(A, e, 0));
      }
    }
    return 0;
  }
  int down(int64_t c0, int64_t c1) {  // finished columns [c0, c1) to the host (on cout)
    const size_t col = (size_t)n * sizeof(double);
    const int64_t rows = std::min(n, c1 + 1);  // H rows the sweep may have changed
    const int64_t kmax = std::max((rows - 1) / chunk, (c1 - 1) / chunk);
    CU(wait_value((CUstream)g.cout, (CUdeviceptr)(d_flags + kmax), 1, CU_STREAM_WAIT_VALUE_GEQ));
    if (Hh)
      CK(cudaMemcpy2DAsync(Hh + c0 * n, col, dH + c0 * n, col, (size_t)rows * sizeof(double), (size_t)(c1 - c0),
                           cudaMemcpyDeviceToHost, g.cout));
    if (Zh) CK(cudaMemcpyAsync(Zh + c0 * n, dZ + c0 * n, col * (c1 - c0), cudaMemcpyDeviceToHost, g.cout));
    d2h += (int64_t)(c1 - c0) * (Hh ? rows : 0) * 8 + (Zh ? (int64_t)(col * (c1 - c0)) : 0);
    return 0;
  }
  // all downloads, enqueued before the kernel finishes: chunk by chunk behind the step counters,
  // the rest after the kernel (event `kernel_done` recorded on A)
  int download(cudaStream_t A, const int* step_ctr, const std::vector<hqr::StepInfo>& steps,
               cudaEvent_t kernel_done) {
    int64_t done = 0;
    for (size_t s = 0; s < fin.size(); ++s) {
      if (steps[s].ntiles > 0)
        CU(wait_value((CUstream)g.cout, (CUdeviceptr)(step_ctr + 4 * s + 2), (cuuint32_t)(4 * steps[s].ntiles),
                      CU_STREAM_WAIT_VALUE_GEQ));
      if (fin[s] - done >= chunk) {
        int rc = down(done, fin[s]);
        if (rc) return rc;
        done = fin[s];
      }
    }
    CK(cudaStreamWaitEvent(g.cout, kernel_done, 0));
    if (done < n) {
      int rc = down(done, n);
      if (rc) return rc;
    }
    cudaEvent_t e = io_event(1);
    CK(cudaEventRecord(e, g.cout));
    CK(cudaStreamWaitEvent(A, e, 0));
    return 0;
  }
};

// Critical SMs: when one chain's chase path (its windows' chases back to back) is
// comparable to the sweep's GEMM time, `2 nchains + 2` CTAs serve only the critical queue (chases and
// the near tasks the next chases read), so a chase is claimed as soon as its inputs are ready instead
// of behind the previous step's bulk tiles, and runs on an SM whose ring holds no bulk tiles to drain.
// GEMM-bound sweeps (the chase path well below the GEMM time) keep one queue (0).
int crit_sms(const Plan& P, const FusedTasks& f) {
  if (const char* e = hqr::tuning_env("HQR_CRIT_SMS")) return std::max(0, atoi(e));  // tuning builds
  const double gemm_us = f.flops / (g.num_sms * 0.19e12) * 1e6;  // ~0.75 of the per-SM DMMA peak
  if (f.chase_path_us < 0.5 * gemm_us) return 0;
  const int c = 2 * P.nchains + 2;  // a chase and its near tiles per chain at once, plus two
  return c <= g.num_sms / 4 ? c : 0;
}

int enqueue_fused(CachedPlan& cp, double* H, double* Z, int64_t n, const hqr::TensorMaps& tm,
                  hqr_stats* st, bool prof = false, std::vector<int>* classes = nullptr,
                  IoPlan* io = nullptr) {
  const Plan& P = cp.plan;
  FusedTasks* f = nullptr;
  int rc = get_fused(cp, Z != nullptr, n, &f);
  if (rc) return rc;
  cudaStream_t A = g.stream;
  CK(cudaMemsetAsync(f->d_ctr, 0, f->nctr * sizeof(int), A));
  auto args = [&](int s) {
    StepArgs a{};
    a.H = H; a.Z = Z; a.n = n; a.ilo = P.ilo; a.ihi = P.ihi;
    a.hcol0 = 0; a.lc0 = 0; a.lc1 = n; a.zrows = n; a.ldz = n;
    a.wins = cp.d_wins; a.coef = g.d_coef; a.qslots = g.d_q; a.KP = cp.KP; a.QLD = hqr::pad_ld(cp.KP);
    a.wstats = g.d_wstats;
    a.aftermath = reinterpret_cast<signed char*>(g.d_aft);
    if (s < P.nsteps) {
      a.win_begin = P.step_begin[s];
      a.win_count = P.step_begin[s + 1] - P.step_begin[s];
      a.slot_offset = (s % hqr::kQSets) * P.nchains;
    }
    a.step = s;
    return a;
  };
  size_t ev = 0;
  auto mark = [&](int cls) {  // prof: events around every launch (class 0 chase, 3 fused step)
    if (!prof) return;
    cudaEventRecord(prof_event(ev++), A);
    if (classes) classes->push_back(cls);
  };
  if (io) {
    io->plan(P);
    int64_t first_rows = 0;
    for (int i = P.step_begin[0]; i < P.step_begin[1]; ++i) first_rows = std::max<int64_t>(first_rows, P.windows[i].w1);
    if ((rc = io->upload(A, first_rows))) return rc;
  }
  mark(0);
  CK(hqr::launch_chase(args(0), P.max_kw, P.max_nbc, A));
  mark(-1);
  st->launches_chase++;
  int* step_ctr = f->d_ctr + 8;
  int* win_ctr = step_ctr + 4 * (size_t)P.nsteps;
  int* task_ctr = win_ctr + hqr::kWinCtr * P.windows.size();  // per task: completion count
  // (step 0's chases ran in their own launch: step-0 tasks do not wait for them)
  const StepArgs base = args(0);
  static const bool per_step = hqr::tuning_env("HQR_PER_STEP") != nullptr;  // A/B knob (tuning builds): a launch per step
  if (!per_step || io) {
    // one persistent launch for the whole sweep: step g+1's work starts as soon as its own
    // dependencies are met (no launch boundary, no end-of-step tail)
    mark(3);
    int csms = crit_sms(P, *f);
    if (csms >= std::max(1, std::min((int)f->tasks.size(), g.num_sms)) || f->ncrit <= 0 ||
        f->ncrit >= (int)f->tasks.size())
      csms = 0;  // (launch_step's own rule: both queues need CTAs and tasks)
    st->crit_sms = csms;
    CK(hqr::launch_step(base, f->d_steps, P.nsteps, f->d_tasks, (int)f->tasks.size(), 0, f->d_dep_begin,
                        f->d_deps, f->d_ctr, step_ctr, task_ctr, io ? io->d_flags : nullptr, tm, P.max_kw,
                        g.num_sms, A, f->d_qidx, f->ncrit, csms));
    mark(-1);
    st->launches_left++;
    if (io) {
      cudaEvent_t kd = io_event(2);
      CK(cudaEventRecord(kd, A));
      if ((rc = io->download(A, step_ctr, f->steps, kd))) return rc;
    }
  } else {
    for (int s = 0; s < P.nsteps; ++s) {
      const int nt = f->begin[s + 1] - f->begin[s];
      mark(3);
      CK(hqr::launch_step(base, f->d_steps, P.nsteps, f->d_tasks + f->begin[s], nt, f->begin[s], f->d_dep_begin,
                          f->d_deps, step_ctr + 4 * s + 3, step_ctr, task_ctr, nullptr, tm, P.max_kw, g.num_sms, A,
                          nullptr, 0, 0));
      mark(-1);
      st->launches_left++;  // one fused launch per step (counted once)
    }
  }
  if (io) {
    st->h2d_bytes = io->h2d;
    st->d2h_bytes = io->d2h;
  }
  st->flops_update = f->flops;
  st->bytes_update = f->bytes;
  st->steps = P.nsteps;
  st->windows = (int64_t)P.windows.size();
  st->kernels_launched = st->launches_chase + st->launches_left;
  return 0;
}

}  // namespace

extern "C" {

int hqr_setup(const hqr_config* cfg) {
  if (!cfg) return -1;
  if (g.ready) hqr_teardown();
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return -1;
  if (cfg->world > 1 && !cfg->nccl_id) return -1;
  if (cfg->window_max < 0 || cfg->window_max > hqr::kMaxWindow) return -1;
  if ((cfg->col_bounds || cfg->row_bounds) && cfg->world > 1) {
    // explicit shard bounds (for n = n_max): both given, 0 = b[0] < ... < b[world] = n_max, even
    // (16-byte TMA strides), H shards >= HQR_MAX_WINDOW + 8 columns wide (a window meets <= 2 ranks)
    if (!cfg->col_bounds || !cfg->row_bounds || cfg->n_max < 1) return -1;
    const int64_t* cb = cfg->col_bounds;
    const int64_t* rb = cfg->row_bounds;
    if (cb[0] != 0 || rb[0] != 0 || cb[cfg->world] != cfg->n_max || rb[cfg->world] != cfg->n_max) return -1;
    for (int r = 0; r < cfg->world; ++r) {
      if (cb[r + 1] - cb[r] < hqr::kMaxWindow + 8 || rb[r + 1] - rb[r] < 2) return -1;
      if ((r > 0 && ((cb[r] | rb[r]) & 1))) return -1;
    }
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= cfg->device || cfg->device < 0) {
    cudaGetLastError();
    return -101;
  }
  CK(cudaSetDevice(cfg->device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, cfg->device));
  if (prop.major != 10) return -101;  // built for sm_100a only
  g.device = cfg->device;
  g.window_max = cfg->window_max;
  g.user_cb.clear();
  g.user_rb.clear();
  g.user_n = 0;
  if (cfg->col_bounds && cfg->world > 1) {
    g.user_cb.assign(cfg->col_bounds, cfg->col_bounds + cfg->world + 1);
    g.user_rb.assign(cfg->row_bounds, cfg->row_bounds + cfg->world + 1);
    g.user_n = cfg->n_max;
  }
  g.rank = cfg->rank;
  g.world = cfg->world;
  g.flags = cfg->flags;
  g.num_sms = prop.multiProcessorCount;
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CK(cudaStreamCreateWithPriority(&g.stream, cudaStreamNonBlocking, prio_hi));
  CK(cudaStreamCreateWithPriority(&g.zstream, cudaStreamNonBlocking, prio_lo));
  CK(cudaStreamCreateWithFlags(&g.cin, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&g.cout, cudaStreamNonBlocking));
  CK(cudaEventCreate(&g.ev0));
  CK(cudaEventCreate(&g.ev1));
  CK(cudaEventCreateWithFlags(&g.ev_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&g.ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&g.ev_join, cudaEventDisableTiming));
  CK(cudaStreamCreateWithPriority(&g.cstream, cudaStreamNonBlocking, prio_hi));
  CK(cudaEventCreateWithFlags(&g.qz_fork, cudaEventDisableTiming));
  for (int i = 0; i < 3; ++i) {
    CK(cudaStreamCreateWithPriority(&g.qzs[i], cudaStreamNonBlocking, prio_hi));
    CK(cudaEventCreateWithFlags(&g.qz_join[i], cudaEventDisableTiming));
  }
  for (int i = 0; i < kQSetsDist; ++i) {
    CK(cudaEventCreateWithFlags(&g.dev_chase[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g.dev_bc[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g.dev_bulk[i], cudaEventDisableTiming));
  }
  for (int i = 0; i < hqr::kQSets; ++i) {
    CK(cudaEventCreateWithFlags(&g.ev_q[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g.ev_z[i], cudaEventDisableTiming));
  }
  if (g.world > 1) {
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof(id));
    NK(ncclCommInitRank(&g.comm, g.world, id, g.rank));
  } else if (g.flags & HQR_FLAG_NCCL_SELF) {  // one-rank communicator: the NCCL transport on one GPU
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    NK(ncclCommInitRank(&g.comm, 1, id, 0));
  }
  if (hqr::tuning_env("HQR_PROGRESS_SECS")) hqr::debug_progress_init();
  g.ready = true;
  return 0;
}

int hqr_teardown(void) {
  if (!g.ready) return 0;
  cudaSetDevice(g.device);
  cudaStreamSynchronize(g.stream);
  for (auto& kv : g.graphs) cudaGraphExecDestroy(kv.second.exec);
  g.graphs.clear();
  for (auto& kv : g.plans) {
    if (kv.second->d_wins) cudaFree(kv.second->d_wins);
    for (auto& f : kv.second->fused)
      if (f) {
        if (f->d_tasks) cudaFree(f->d_tasks);
        if (f->d_ctr) cudaFree(f->d_ctr);
        if (f->d_steps) cudaFree(f->d_steps);
        if (f->d_wdeps) cudaFree(f->d_wdeps);
        if (f->d_dep_begin) cudaFree(f->d_dep_begin);
        if (f->d_deps) cudaFree(f->d_deps);
        if (f->d_qidx) cudaFree(f->d_qidx);
      }
  }
  g.plans.clear();
  for (auto e : g.prof_events) cudaEventDestroy(e);
  g.prof_events.clear();
  if (g.d_coef) cudaFree(g.d_coef);
  if (g.d_aft) cudaFree(g.d_aft);
  g.d_aft = nullptr;
  g.aft_cap = 0;
  g.aft_n = 0;
  if (g.d_wstats) cudaFree(g.d_wstats);
  if (g.d_upflags) cudaFree(g.d_upflags);
  g.d_upflags = nullptr;
  g.upflags_cap = 0;
  g.d_wstats = nullptr;
  g.wstats_cap = 0;
  g.wstats_plan = nullptr;
  if (g.d_q) cudaFree(g.d_q);
  if (g.d_hstage) cudaFree(g.d_hstage);
  if (g.d_zstage) cudaFree(g.d_zstage);
  g.d_coef = g.d_q = g.d_hstage = g.d_zstage = nullptr;
  g.coef_cap = g.q_cap = g.stage_cap = 0;
  g.hstage_zero_n = -1;
  cudaEventDestroy(g.ev0);
  cudaEventDestroy(g.ev1);
  cudaEventDestroy(g.ev_in);
  cudaEventDestroy(g.ev_fork);
  cudaEventDestroy(g.ev_join);
  for (int i = 0; i < kQSetsDist; ++i) {
    cudaEventDestroy(g.dev_chase[i]);
    cudaEventDestroy(g.dev_bc[i]);
    cudaEventDestroy(g.dev_bulk[i]);
  }
  if (g.cstream) cudaStreamDestroy(g.cstream);
  g.cstream = nullptr;
  if (g.qz_fork) cudaEventDestroy(g.qz_fork);
  g.qz_fork = nullptr;
  for (int i = 0; i < 3; ++i) {
    if (g.qzs[i]) cudaStreamDestroy(g.qzs[i]);
    if (g.qz_join[i]) cudaEventDestroy(g.qz_join[i]);
    g.qzs[i] = nullptr;
    g.qz_join[i] = nullptr;
  }
  for (int i = 0; i < hqr::kQSets; ++i) {
    cudaEventDestroy(g.ev_q[i]);
    cudaEventDestroy(g.ev_z[i]);
  }
  cudaStreamDestroy(g.zstream);
  cudaStreamDestroy(g.cin);
  cudaStreamDestroy(g.cout);
  for (cudaEvent_t e : g.io_events) cudaEventDestroy(e);
  g.io_events.clear();
  cudaStreamDestroy(g.stream);
  if (g.comm) {
    ncclCommDestroy(g.comm);
    g.comm = nullptr;
  }
  for (auto p : g.vH) if (p) cudaFree(p);
  for (auto p : g.vZ) if (p) cudaFree(p);
  g.vH.clear(); g.vZ.clear(); g.vH_cap.clear(); g.vZ_cap.clear();
  g.ready = false;
  cudaError_t e = cudaGetLastError();
  return cuerr(e);
}

}  // extern "C"

namespace {

// F_alg of nb bulges on [ilo, ihi]: per reflector 10 (6 for the final 2-reflector)
// x (left columns + right rows + n Z rows)
double falg_block(int64_t n, int64_t ilo, int64_t ihi, int nb, bool with_z) {
  double f = 0.0;
  for (int64_t p = ilo - 1; p <= ihi - 2; ++p) {
    const int m = (p <= ihi - 3) ? 3 : 2;
    const int64_t c0 = (p == ilo - 1) ? ilo : p + 1;
    const int64_t r1 = std::min<int64_t>(p + m + 1, ihi);
    f += (m == 3 ? 10.0 : 6.0) * ((double)(n - c0) + (double)(r1 + 1) + (with_z ? (double)n : 0.0));
  }
  return f * nb;
}

int sweep_impl(double* H, double* Z, int64_t n, const Blocks& blocks, const double* shifts_re,
               const double* shifts_im, int window) {
  if (!H) return -1;
  int rc = validate_blocks(n, blocks, shifts_re, shifts_im, window, true);
  if (rc) return rc;
  CachedPlan* cp = nullptr;
  rc = get_plan(n, blocks, window, &cp, false);  // a7 plan (host only, cached; validates the window)
  if (rc) return rc;
  if (!g.ready) return -100;
  CK(cudaSetDevice(g.device));
  rc = get_plan(n, blocks, window, &cp, true);
  if (rc) return rc;

  hqr_stats st{};
  st.window_eff = cp->plan.k;
  const bool h_dev = is_device_ptr(H);
  const bool z_dev = Z ? is_device_ptr(Z) : true;

  // decoupling check (-10): two scalars per block
  for (int i = 0; i < blocks.count(); ++i) {
    const int64_t ilo = blocks.ilo[i], ihi = blocks.ihi[i];
    double sub[2] = {0.0, 0.0};
    if (ilo > 0 || ihi < n - 1) {
      const double* p0 = H + ilo + (ilo - 1) * n;
      const double* p1 = H + (ihi + 1) + ihi * n;
      if (h_dev) {
        if (ilo > 0) CK(cudaMemcpy(&sub[0], p0, sizeof(double), cudaMemcpyDeviceToHost));
        if (ihi < n - 1) CK(cudaMemcpy(&sub[1], p1, sizeof(double), cudaMemcpyDeviceToHost));
      } else {
        if (ilo > 0) sub[0] = *p0;
        if (ihi < n - 1) sub[1] = *p1;
      }
      if (sub[0] != 0.0 || sub[1] != 0.0) return -10;
    }
  }

  rc = wait_for_caller();
  if (rc) return rc;
  // a1 the shift pairs of all blocks' bulges (sigma, pi are formed in the chase: R1/R3/R15)
  rc = upload_coef(shifts_re, shifts_im, cp->plan.nb);
  if (rc) return rc;
  // a9 aftermath flags: -1 (not scanned) everywhere, then the chases of each block's last chain
  rc = ensure(&g.d_aft, &g.aft_cap, (size_t)(n + 7) / 8);
  if (rc) return rc;
  CK(cudaMemsetAsync(g.d_aft, 0xff, (size_t)n, g.stream));
  g.aft_n = 0;
  rc = ensure(&g.d_q, &g.q_cap, (size_t)hqr::kQSets * cp->plan.nchains * cp->KP * hqr::pad_ld(cp->KP));
  if (rc) return rc;
  rc = ensure(&g.d_wstats, &g.wstats_cap, cp->plan.windows.size());
  if (rc) return rc;
  g.wstats_plan = cp;
  g.wstats_n = n;
  g.wstats_z = Z != nullptr;

  // host buffers: stage through library-owned device memory
  const size_t nn = (size_t)n * (size_t)n;
  double* dH = H;
  double* dZ = Z;
  CK(cudaEventRecord(g.ev0, g.stream));
  if (!h_dev || !z_dev) {
    size_t need = nn;
    if (g.stage_cap < need) {
      if (g.d_hstage) CK(cudaFree(g.d_hstage));
      if (g.d_zstage) CK(cudaFree(g.d_zstage));
      g.d_hstage = g.d_zstage = nullptr;
      g.stage_cap = 0;
      g.hstage_zero_n = -1;
      CK(cudaMalloc(&g.d_hstage, need * sizeof(double)));
      CK(cudaMalloc(&g.d_zstage, need * sizeof(double)));
      g.stage_cap = need;
    }
    if (!h_dev) dH = g.d_hstage;
    if (Z && !z_dev) dZ = g.d_zstage;
  }

  const bool prof = (g.flags & HQR_FLAG_PROFILE) != 0;
  const bool use_graph = !prof && !(g.flags & HQR_FLAG_NO_GRAPH);
  std::vector<int> classes;
  hqr::TensorMaps tmf;
  CK(hqr::make_tensor_maps(&tmf, dH, n, dZ, n, n, n, cp->KP));
  const bool fused = tmf.valid && !(g.flags & HQR_FLAG_NO_FUSE) &&
                     cp->plan.max_nbc <= hqr::kMaxChaseBulges;
  if (fused) {  // build / upload the task queues outside any stream capture
    FusedTasks* f = nullptr;
    rc = get_fused(*cp, dZ != nullptr, n, &f);
    if (rc) return rc;
  }
  // host buffers with the fused path: copies overlapped with the steps (IoPlan); otherwise the
  // whole matrices are staged before and after the sweep
  const bool host_io = (!h_dev || (Z && !z_dev));
  const bool overlap = host_io && fused && !prof;
  if (host_io && !overlap) {
    if (!h_dev) {
      CK(cudaMemcpyAsync(dH, H, nn * sizeof(double), cudaMemcpyHostToDevice, g.stream));
      st.h2d_bytes += nn * sizeof(double);
      g.hstage_zero_n = -1;  // the caller's entries below the subdiagonal are in the buffer now
    }
    if (Z && !z_dev) {
      CK(cudaMemcpyAsync(dZ, Z, nn * sizeof(double), cudaMemcpyHostToDevice, g.stream));
      st.h2d_bytes += nn * sizeof(double);
    }
  }
  static const bool timing = hqr::tuning_env("HQR_TIMING_DUMP") != nullptr;  // -DHQR_TIMING -DHQR_TUNING builds
  if (timing && fused) hqr::debug_timing(0, true);
  if (overlap) {
    IoPlan io;
    io.Hh = h_dev ? nullptr : H;
    io.Zh = (Z && !z_dev) ? Z : nullptr;
    io.dH = dH;
    io.dZ = dZ;
    io.n = n;
    const size_t nch = (size_t)((n + hqr::kUploadChunk - 1) / hqr::kUploadChunk);
    if (g.upflags_cap < nch) {
      if (g.d_upflags) CK(cudaFree(g.d_upflags));
      g.d_upflags = nullptr;
      g.upflags_cap = 0;
      CK(cudaMalloc(&g.d_upflags, nch * sizeof(int)));
      g.upflags_cap = nch;
    }
    io.d_flags = g.d_upflags;
    rc = enqueue_fused(*cp, dH, dZ, n, tmf, &st, false, nullptr, &io);
    if (rc) return rc;
  } else if (use_graph) {
    GraphKey gk{plan_key(n, blocks, window), dH, dZ};
    auto it = g.graphs.find(gk);
    if (it == g.graphs.end()) {
      cudaGraph_t graph;
      CK(cudaStreamBeginCapture(g.stream, cudaStreamCaptureModeThreadLocal));
      hqr_stats cap{};
      int rc2 = fused ? enqueue_fused(*cp, dH, dZ, n, tmf, &cap)
                      : enqueue_sweep(*cp, dH, dZ, n, false, nullptr, &cap);
      cudaError_t ec = cudaStreamEndCapture(g.stream, &graph);
      if (rc2) return rc2;
      CK(ec);
      cudaGraphExec_t exec;
      CK(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      it = g.graphs.emplace(gk, CachedGraph{exec, cap}).first;
    }
    CK(cudaGraphLaunch(it->second.exec, g.stream));
    const hqr_stats& c = it->second.stats;  // launches / flops of the captured sequence
    st.flops_update = c.flops_update;
    st.bytes_update = c.bytes_update;
    st.launches_chase = c.launches_chase;
    st.launches_left = c.launches_left;
    st.launches_right = c.launches_right;
    st.steps = c.steps;
    st.windows = c.windows;
    st.kernels_launched = c.kernels_launched;
    st.crit_sms = c.crit_sms;
  } else if (fused) {
    rc = enqueue_fused(*cp, dH, dZ, n, tmf, &st, prof, &classes);
    if (rc) return rc;
  } else {
    rc = enqueue_sweep(*cp, dH, dZ, n, prof, &classes, &st);
    if (rc) return rc;
  }

  if (!h_dev && !overlap) {
    CK(cudaMemcpyAsync(H, dH, nn * sizeof(double), cudaMemcpyDeviceToHost, g.stream));
    st.d2h_bytes += nn * sizeof(double);
  }
  if (Z && !z_dev && !overlap) {
    CK(cudaMemcpyAsync(Z, dZ, nn * sizeof(double), cudaMemcpyDeviceToHost, g.stream));
    st.d2h_bytes += nn * sizeof(double);
  }
  CK(cudaEventRecord(g.ev1, g.stream));
  CK(cudaStreamSynchronize(g.stream));
  CK(cudaGetLastError());
  g.aft_n = n;
  if (timing && fused) hqr::debug_timing(cp->plan.nsteps, false);
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, g.ev0, g.ev1));
  st.ms_total = ms;
  if (prof) {
    // events come in (start, end) pairs; classes[2i] is the kernel class of pair i
    for (size_t i = 0; i + 1 < classes.size(); i += 2) {
      float e = 0;
      cudaEventElapsedTime(&e, g.prof_events[i], g.prof_events[i + 1]);
      if (classes[i] == 0) st.ms_chase += e;
      else if (classes[i] == 1) st.ms_left += e;
      else if (classes[i] == 2) st.ms_right += e;
      else st.ms_step += e;
    }
  }
  // in-window chase flops (per 3-reflector: 10 flops x (left cols + right rows + Q rows)),
  // once per plan (a host loop over every reflector)
  if (cp->flops_chase < 0) {
    const Plan& P = cp->plan;
    double f = 0;
    for (const WindowDesc& w : P.windows) {
      for (int t = w.t0; t <= w.t1; ++t)
        for (int jj = 0; jj < w.nbc; ++jj) {
          int64_t p = w.ilo - 1 + t - 3 * (int64_t)jj;
          if (p < w.ilo - 1 || p > w.ihi - 2) continue;
          int m = (p <= w.ihi - 3) ? 3 : 2;
          int64_t pl = p - w.w0;
          double cnt = (double)(w.w1 - std::max<int64_t>(pl, 0) - w.w0) + (double)(pl + m + 2) +
                       (double)std::min<int64_t>(pl + m + 3, w.w1 - w.w0 + 1);
          f += (m == 3 ? 10.0 : 6.0) * cnt;
        }
    }
    cp->flops_chase = f;
  }
  st.flops_chase = cp->flops_chase;
  st.flops_alg = 0.0;  // F_alg of every block of this call
  for (int i = 0; i < blocks.count(); ++i) st.flops_alg += falg_block(n, blocks.ilo[i], blocks.ihi[i], blocks.nshifts[i] / 2, Z != nullptr);
  g.stats = st;
  return 0;
}

int plan_query_impl(int64_t n, const Blocks& b, int window, int32_t* info, int32_t* windows,
                    int64_t cap) {
  int rc = validate_blocks(n, b, nullptr, nullptr, window, false);
  if (rc) return rc;
  Plan P;
  rc = b.sweeps ? hqr::make_plan_sweeps(n, b.ilo[0], b.ihi[0], b.count(), b.nshifts.data(), window,
                                        hqr::kMaxWindow, &P)
                : hqr::make_plan_multi(n, b.count(), b.ilo.data(), b.ihi.data(), b.nshifts.data(), window,
                                       hqr::kMaxWindow, &P);
  if (rc) return rc;
  if (info) {
    int32_t v[10] = {P.k, P.nbc_max, P.s, P.lag, P.nchains, P.nsteps, (int32_t)P.windows.size(),
                     P.max_kw, P.max_nbc, P.nb};
    std::memcpy(info, v, sizeof(v));
  }
  if (windows && cap >= (int64_t)P.windows.size()) {
    for (int s = 0; s < P.nsteps; ++s)
      for (int i = P.step_begin[s]; i < P.step_begin[s + 1]; ++i) {
        const WindowDesc& w = P.windows[i];
        int32_t* r = windows + 12 * (int64_t)i;
        r[0] = s; r[1] = w.chain; r[2] = w.w0; r[3] = w.w1; r[4] = w.t0; r[5] = w.t1;
        r[6] = w.b0; r[7] = w.nbc; r[8] = w.slot; r[9] = w.last; r[10] = w.ilo; r[11] = w.ihi;
      }
  }
  return 0;
}

// ================================================================================================
// Sharded sweep (dist.hpp).  One executor for both transports:
//   NCCL     one rank per process / GPU: ncclSend/Recv for the lent column slabs, ncclBroadcast of
//            every window's factor from its owner (grouped per step);
//   VIRTUAL  every rank's shard lives on this one GPU (hqr_sweep_virtual, for tests): the slabs move
//            with device-to-device copies and all ranks share one Q slot array, so the broadcast is a
//            no-op.  The per-rank kernel sequence is identical.
// Per step: (1) lend straddling slabs, (2) chase owned windows, (3) broadcast factors, (4) left
// update of every window on the held columns, (5) right update of owned windows, Z update of every
// window on the local rows, (6) return the slabs.
// ================================================================================================
struct RankCtx {
  int rank;
  double* H;                      // local columns [cb[r], cb[r+1] + halo), ld n
  double* Z;                      // local rows [rb[r], rb[r+1]), ld = rows, or nullptr
  int64_t hcols, zrows;
  std::vector<hqr::RankStep> steps;
  std::vector<WindowDesc> owned;  // owned windows of all steps, grouped by step
  std::vector<int32_t> owned_begin;
  WindowDesc* d_owned = nullptr;
  hqr::TensorMaps tm;
};

int prepare_rank(const CachedPlan& cp, const hqr::DistLayout& L, RankCtx* rc) {
  const Plan& P = cp.plan;
  rc->steps.resize(P.nsteps);
  rc->owned.clear();
  rc->owned_begin.assign(1, 0);
  for (int s = 0; s < P.nsteps; ++s) {
    hqr::rank_step(P, L, rc->rank, s, &rc->steps[s]);
    for (int32_t i : rc->steps[s].owned) rc->owned.push_back(P.windows[i]);
    rc->owned_begin.push_back((int32_t)rc->owned.size());
  }
  if (!rc->owned.empty()) {
    CK(cudaMalloc(&rc->d_owned, rc->owned.size() * sizeof(WindowDesc)));
    CK(cudaMemcpy(rc->d_owned, rc->owned.data(), rc->owned.size() * sizeof(WindowDesc),
                  cudaMemcpyHostToDevice));
  }
  return 0;
}

int run_dist(const CachedPlan& cp, const hqr::DistLayout& L, std::vector<RankCtx>& ranks, bool nccl,
             hqr_stats* st) {
  const Plan& P = cp.plan;
  const int64_t n = P.n;
  // A (high priority): lend, chase, left updates, near-right updates, return -- the chain that
  //   feeds the next chases; C: the grouped broadcast of each step's factors (NCCL);
  // B (low priority): the updates nothing later in the sweep reads before they are done -- Z(local
  //   rows, W) Q_W for every window and the far-right rows [0, sp) of the owned windows (P:713,
  //   P:758-765) -- trailing A by up to kQSetsDist - 1 steps (the Q slot sets rotate).
  // sp(s) = the smallest first row of any later window, even: later left / near-right / chase work
  // touches only rows >= sp(s), so the far-right rows never meet it.  Straddling windows keep their
  // far-right on A (their lent columns go back at the end of the step), and a rank drains B before
  // it lends or borrows columns (B may still be updating the lent ones; the borrower's whole right
  // update of the straddling window must follow its earlier deferred far-right rows).
  cudaStream_t A = g.stream, B = g.zstream, C = nccl ? g.cstream : g.stream;
  // Per-rank busy time (tuning builds, virtual ranks: HQR_DIST_PROFILE=file): every launch on one
  // stream, bracketed by events, written as (step, rank, class, ms) -- each rank's kernels as they
  // would run on its own GPU, for tools/dist_balance_measured.py.  Classes: 0 chase, 1 left,
  // 2 near-right, 3 far-right, 4 Z, 5 slab copies.
  const char* prof_path = nccl ? nullptr : hqr::tuning_env("HQR_DIST_PROFILE");
  struct ProfRec { int step, rank, cls; cudaEvent_t e0, e1; };
  std::vector<ProfRec> prof;
  if (prof_path) B = A;
  auto pbeg = [&](int s, int r, int cls) -> int {
    if (!prof_path) return -1;
    ProfRec pr{s, r, cls, nullptr, nullptr};
    cudaEventCreate(&pr.e0);
    cudaEventCreate(&pr.e1);
    cudaEventRecord(pr.e0, A);
    prof.push_back(pr);
    return (int)prof.size() - 1;
  };
  auto pend = [&](int i) {
    if (i >= 0) cudaEventRecord(prof[i].e1, A);
  };
  for (auto& rc : ranks) {
    CK(hqr::make_tensor_maps(&rc.tm, rc.H, rc.hcols, rc.Z, rc.zrows, rc.zrows, n, cp.KP));
  }
  std::vector<int64_t> sp(P.nsteps, 0);
  {
    int64_t run = n;
    for (int s = P.nsteps - 1; s >= 0; --s) {
      sp[s] = run & ~(int64_t)1;
      for (int i = P.step_begin[s]; i < P.step_begin[s + 1]; ++i) run = std::min<int64_t>(run, P.windows[i].w0);
    }
  }
  CK(cudaEventRecord(g.ev_fork, A));
  CK(cudaStreamWaitEvent(B, g.ev_fork, 0));
  if (nccl) CK(cudaStreamWaitEvent(C, g.ev_fork, 0));
  const size_t qsz = (size_t)cp.KP * hqr::pad_ld(cp.KP);
  auto args = [&](const RankCtx& rc, int s, int so) {
    StepArgs a{};
    a.H = rc.H; a.Z = rc.Z; a.n = n; a.hcol0 = L.cb[rc.rank];
    a.lc0 = rc.steps[s].lc0; a.lc1 = rc.steps[s].lc1; a.zrows = rc.zrows; a.ldz = rc.zrows;
    a.wins = cp.d_wins; a.win_begin = P.step_begin[s]; a.win_count = P.step_begin[s + 1] - P.step_begin[s];
    a.coef = g.d_coef; a.qslots = g.d_q; a.KP = cp.KP; a.QLD = hqr::pad_ld(cp.KP); a.slot_offset = so;
    a.step = s;
    return a;
  };
  auto account = [&](int64_t items, double fl, double by, int* launches) {
    if (items) (*launches)++;
    st->flops_update += fl;
    st->bytes_update += by;
  };
  for (int s = 0; s < P.nsteps; ++s) {
    const int set = s % kQSetsDist;
    const int so = set * P.nchains;
    if (s >= kQSetsDist) CK(cudaStreamWaitEvent(A, g.dev_bulk[set], 0));  // B is done with this slot set
    // (1) lend: rank r+1's leading columns -> rank r's halo (the lender's B drained first)
    // (the borrower applies its straddling window's whole right update on A: after its earlier
    // deferred far-right rows on those columns)
    bool lends = false;
    for (auto& rc : ranks) lends |= rc.steps[s].lend_out > 0 || rc.steps[s].lend_in > 0;
    if (lends && s > 0) {
      CK(cudaEventRecord(g.ev_join, B));
      CK(cudaStreamWaitEvent(A, g.ev_join, 0));
    }
    if (nccl) {
      RankCtx& rc = ranks[0];
      const hqr::RankStep& rs = rc.steps[s];
      if (rs.lend_out || rs.lend_in) {
        NK(ncclGroupStart());
        if (rs.lend_out) NK(ncclSend(rc.H, (size_t)rs.lend_out * n, ncclDouble, rc.rank - 1, g.comm, A));
        if (rs.lend_in)
          NK(ncclRecv(rc.H + (L.cb[rc.rank + 1] - L.cb[rc.rank]) * n, (size_t)rs.lend_in * n, ncclDouble,
                      rc.rank + 1, g.comm, A));
        NK(ncclGroupEnd());
      }
    } else {
      for (size_t r = 0; r + 1 < ranks.size(); ++r) {
        const int64_t cnt = ranks[r].steps[s].lend_in;
        if (cnt) {
          const int pi = pbeg(s, (int)r, 5);
          CK(cudaMemcpyAsync(ranks[r].H + (L.cb[r + 1] - L.cb[r]) * n, ranks[r + 1].H,
                             (size_t)cnt * n * sizeof(double), cudaMemcpyDeviceToDevice, A));
          pend(pi);
        }
      }
    }
    // (2) chase owned windows
    for (auto& rc : ranks) {
      const int nown = rc.owned_begin[s + 1] - rc.owned_begin[s];
      if (!nown) continue;
      StepArgs a = args(rc, s, so);
      a.wins = rc.d_owned; a.win_begin = rc.owned_begin[s]; a.win_count = nown;
      const int pi = pbeg(s, rc.rank, 0);
      CK(hqr::launch_chase(a, P.max_kw, P.max_nbc, A));
      pend(pi);
      st->launches_chase++;
    }
    CK(cudaEventRecord(g.dev_chase[set], A));
    // (3) broadcast every window's factor from its owner (comm stream), A and B wait for it
    cudaEvent_t qready = g.dev_chase[set];
    if (nccl) {
      CK(cudaStreamWaitEvent(C, g.dev_chase[set], 0));
      NK(ncclGroupStart());
      for (int i = P.step_begin[s]; i < P.step_begin[s + 1]; ++i) {
        const WindowDesc& w = P.windows[i];
        double* q = g.d_q + (size_t)(w.slot + so) * qsz;
        NK(ncclBroadcast(q, q, qsz, ncclDouble, hqr::owner_of_col(L, w.w0), g.comm, C));
      }
      NK(ncclGroupEnd());
      CK(cudaEventRecord(g.dev_bc[set], C));
      CK(cudaStreamWaitEvent(A, g.dev_bc[set], 0));
      qready = g.dev_bc[set];
    }
    (void)qready;
    // (4) A: left update of every window on the held columns
    for (auto& rc : ranks) {
      StepArgs a = args(rc, s, so);
      const WindowDesc* hw = P.windows.data() + a.win_begin;
      int64_t items;
      double fl, by;
      const int pi = pbeg(s, rc.rank, 1);
      CK(hqr::launch_left(a, hw, g.num_sms, rc.tm, A, &items, &fl, &by));
      pend(pi);
      account(items, fl, by, &st->launches_left);
    }
    // B starts the step's deferred work only after the step's left updates: the far-right rows
    // of a window meet the left update of a window above it in the same step (rows < sp) -- the
    // two commute but must not run concurrently
    CK(cudaEventRecord(g.dev_chase[set], A));
    CK(cudaStreamWaitEvent(B, g.dev_chase[set], 0));
    // (4) A: near-right of the owned windows (all rows if the rank straddles: its lent columns
    //     return below); (5) B: their far-right rows [0, sp) and Z(local rows, W) Q_W
    for (auto& rc : ranks) {
      StepArgs a = args(rc, s, so);
      const WindowDesc* hw = P.windows.data() + a.win_begin;
      int64_t items;
      double fl, by;
      const int nown = rc.owned_begin[s + 1] - rc.owned_begin[s];
      if (nown) {
        StepArgs ar = a;
        ar.wins = rc.d_owned; ar.win_begin = rc.owned_begin[s]; ar.win_count = nown;
        ar.right_mode = 1;
        const bool straddle = rc.steps[s].lend_in > 0;
        ar.rrow_lo = straddle ? 0 : sp[s];
        ar.rrow_hi = n;  // rows [rrow_lo, w0)
        int pi = pbeg(s, rc.rank, 2);
        CK(hqr::launch_right(ar, rc.owned.data() + rc.owned_begin[s], g.num_sms, rc.tm, A, &items, &fl, &by));
        pend(pi);
        account(items, fl, by, &st->launches_right);
        if (!straddle && sp[s] > 0) {
          StepArgs af = ar;
          af.rrow_lo = 0;
          af.rrow_hi = sp[s];
          pi = pbeg(s, rc.rank, 3);
          CK(hqr::launch_right(af, rc.owned.data() + rc.owned_begin[s], g.num_sms, rc.tm, B, &items, &fl, &by));
          pend(pi);
          account(items, fl, by, &st->launches_right);
        }
      }
      if (rc.Z) {
        StepArgs az = a;
        az.right_mode = 2;
        const int pi = pbeg(s, rc.rank, 4);
        CK(hqr::launch_right(az, hw, g.num_sms, rc.tm, B, &items, &fl, &by));
        pend(pi);
        account(items, fl, by, &st->launches_right);
      }
    }
    CK(cudaEventRecord(g.dev_bulk[set], B));
    // (6) return the lent slabs
    if (nccl) {
      RankCtx& rc = ranks[0];
      const hqr::RankStep& rs = rc.steps[s];
      if (rs.lend_out || rs.lend_in) {
        NK(ncclGroupStart());
        if (rs.lend_in)
          NK(ncclSend(rc.H + (L.cb[rc.rank + 1] - L.cb[rc.rank]) * n, (size_t)rs.lend_in * n, ncclDouble,
                      rc.rank + 1, g.comm, A));
        if (rs.lend_out) NK(ncclRecv(rc.H, (size_t)rs.lend_out * n, ncclDouble, rc.rank - 1, g.comm, A));
        NK(ncclGroupEnd());
      }
    } else {
      for (size_t r = 0; r + 1 < ranks.size(); ++r) {
        const int64_t cnt = ranks[r].steps[s].lend_in;
        if (cnt) {
          const int pi = pbeg(s, (int)r, 5);
          CK(cudaMemcpyAsync(ranks[r + 1].H, ranks[r].H + (L.cb[r + 1] - L.cb[r]) * n,
                             (size_t)cnt * n * sizeof(double), cudaMemcpyDeviceToDevice, A));
          pend(pi);
        }
      }
    }
  }
  CK(cudaEventRecord(g.ev_join, B));
  CK(cudaStreamWaitEvent(A, g.ev_join, 0));
  if (nccl) {
    CK(cudaEventRecord(g.ev_join, C));
    CK(cudaStreamWaitEvent(A, g.ev_join, 0));
  }
  if (prof_path) {
    CK(cudaStreamSynchronize(A));
    if (FILE* fp = fopen(prof_path, "w")) {
      fprintf(fp, "step,rank,cls,ms\n");
      for (auto& pr : prof) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pr.e0, pr.e1);
        fprintf(fp, "%d,%d,%d,%.6f\n", pr.step, pr.rank, pr.cls, ms);
      }
      fclose(fp);
    }
    for (auto& pr : prof) {
      cudaEventDestroy(pr.e0);
      cudaEventDestroy(pr.e1);
    }
  }
  st->steps = P.nsteps;
  st->windows = (int64_t)P.windows.size();
  st->kernels_launched = st->launches_chase + st->launches_left + st->launches_right;
  return 0;
}

// common validation + shift upload for the sharded entry points
int dist_prepare(int64_t n, const Blocks& b, const double* sr, const double* si, int window, int world,
                 CachedPlan** cpo, hqr::DistLayout* L) {
  int rc = validate_blocks(n, b, sr, si, window, true);
  if (rc) return rc;
  if (!g.user_cb.empty() && world == g.world) {  // hqr_config shard bounds (for n = n_max only)
    if (n != g.user_n) return -11;
    L->world = world;
    L->halo = hqr::kMaxWindow;
    L->cb = g.user_cb;
    L->rb = g.user_rb;
  } else {
    rc = hqr::make_layout(n, world, hqr::kMaxWindow, L);
    if (rc) return rc;
  }
  if (!g.ready) return -100;
  CK(cudaSetDevice(g.device));
  rc = get_plan(n, b, window, cpo, true);
  if (rc) return rc;
  CachedPlan* cp = *cpo;
  rc = wait_for_caller();
  if (rc) return rc;
  rc = upload_coef(sr, si, cp->plan.nb);
  if (rc) return rc;
  rc = ensure(&g.d_q, &g.q_cap, (size_t)kQSetsDist * cp->plan.nchains * cp->KP * hqr::pad_ld(cp->KP));
  return rc;
}

Blocks make_blocks(int nblocks, const int64_t* ilo, const int64_t* ihi, const int* nshifts) {
  Blocks b;
  for (int i = 0; i < nblocks; ++i) {
    b.ilo.push_back(ilo[i]);
    b.ihi.push_back(ihi[i]);
    b.nshifts.push_back(nshifts[i]);
  }
  return b;
}

}  // namespace

extern "C" {

int hqr_sweep(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, const double* shifts_re,
              const double* shifts_im, int nshifts, int window) {
  // world > 1: a collective on this rank's local shards -- the sharded executor
  if (g.ready && g.world > 1) return hqr_sweep_dist(H, Z, n, ilo, ihi, shifts_re, shifts_im, nshifts, window);
  return sweep_impl(H, Z, n, make_blocks(1, &ilo, &ihi, &nshifts), shifts_re, shifts_im, window);
}

int hqr_sweep_multi(double* H, double* Z, int64_t n, int nblocks, const int64_t* ilo,
                    const int64_t* ihi, const double* shifts_re, const double* shifts_im,
                    const int* nshifts, int window) {
  if (!H) return -1;
  if (nblocks < 1 || !ilo || !ihi || !nshifts) return -4;
  if (g.ready && g.world > 1)  // world > 1: the collective on local shards (as hqr_sweep)
    return hqr_sweep_dist_multi(H, Z, n, nblocks, ilo, ihi, shifts_re, shifts_im, nshifts, window);
  return sweep_impl(H, Z, n, make_blocks(nblocks, ilo, ihi, nshifts), shifts_re, shifts_im, window);
}

int hqr_sweeps(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, int nsweeps,
               const double* shifts_re, const double* shifts_im, const int* nshifts, int window) {
  if (!H) return -1;
  if (nsweeps < 1 || !nshifts) return -8;
  if (g.ready && g.world > 1) return -1;  // single GPU (the sharded executor runs one sweep)
  Blocks b;
  b.sweeps = true;
  for (int i = 0; i < nsweeps; ++i) {
    b.ilo.push_back(ilo);
    b.ihi.push_back(ihi);
    b.nshifts.push_back(nshifts[i]);
  }
  return sweep_impl(H, Z, n, b, shifts_re, shifts_im, window);
}

int hqr_plan_query_sweeps(int64_t n, int64_t ilo, int64_t ihi, int nsweeps, const int* nshifts, int window,
                          int32_t* info, int32_t* windows, int64_t cap) {
  if (nsweeps < 1 || !nshifts) return -8;
  Blocks b;
  b.sweeps = true;
  for (int i = 0; i < nsweeps; ++i) {
    b.ilo.push_back(ilo);
    b.ihi.push_back(ihi);
    b.nshifts.push_back(nshifts[i]);
  }
  return plan_query_impl(n, b, window, info, windows, cap);
}

int hqr_plan_query(int64_t n, int64_t ilo, int64_t ihi, int nshifts, int window, int32_t* info,
                   int32_t* windows, int64_t cap) {
  return plan_query_impl(n, make_blocks(1, &ilo, &ihi, &nshifts), window, info, windows, cap);
}

int hqr_plan_query_multi(int64_t n, int nblocks, const int64_t* ilo, const int64_t* ihi,
                         const int* nshifts, int window, int32_t* info, int32_t* windows,
                         int64_t cap) {
  if (nblocks < 1 || !ilo || !ihi || !nshifts) return -4;
  return plan_query_impl(n, make_blocks(nblocks, ilo, ihi, nshifts), window, info, windows, cap);
}

int hqr_dist_layout(int64_t n, int world, int64_t* col_bounds, int64_t* row_bounds, int* halo) {
  if (n < 1) return -1;
  if (world < 1) return -2;
  hqr::DistLayout L;
  int rc = hqr::make_layout(n, world, hqr::kMaxWindow, &L);
  if (rc) return rc;
  for (int r = 0; r <= world; ++r) {
    if (col_bounds) col_bounds[r] = L.cb[r];
    if (row_bounds) row_bounds[r] = L.rb[r];
  }
  if (halo) *halo = L.halo;
  return 0;
}

int hqr_dist_query(int64_t n, int64_t ilo, int64_t ihi, int nshifts, int window, int world, int rank,
                   int64_t* out, int64_t cap) {
  Blocks b;
  b.ilo = {ilo}; b.ihi = {ihi}; b.nshifts = {nshifts};
  int rc = validate_blocks(n, b, nullptr, nullptr, window, false);
  if (rc) return rc;
  if (world < 1 || rank < 0 || rank >= world) return -7;
  hqr::DistLayout L;
  rc = hqr::make_layout(n, world, hqr::kMaxWindow, &L);
  if (rc) return rc;
  Plan P;
  rc = hqr::make_plan(n, ilo, ihi, nshifts, window, hqr::kMaxWindow, &P);
  if (rc) return rc;
  if (!out || cap < P.nsteps) return P.nsteps;
  for (int s = 0; s < P.nsteps; ++s) {
    hqr::RankStep rs;
    hqr::rank_step(P, L, rank, s, &rs);
    int64_t* row = out + 6 * (int64_t)s;
    row[0] = s; row[1] = rs.lend_out; row[2] = rs.lend_in; row[3] = rs.lc0; row[4] = rs.lc1;
    row[5] = (int64_t)rs.owned.size();
  }
  return 0;
}

int hqr_nccl_unique_id(void* out) {
  if (!out) return -1;
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

static int dist_impl(double* H_local, double* Z_local, int64_t n, const Blocks& blocks, const double* shifts_re,
                     const double* shifts_im, int window) {
  if (!H_local) return -1;
  CachedPlan* cp = nullptr;
  hqr::DistLayout L;
  int rc = dist_prepare(n, blocks, shifts_re, shifts_im, window, g.world, &cp, &L);
  if (rc) return rc;
  if (g.world > 1 && !g.comm) return -100;
  {  // -10: H[ilo, ilo-1] on the rank owning column ilo-1, H[ihi+1, ihi] on the owner of column ihi,
     // every block; the verdict is agreed over all ranks (max), so every rank returns the same code
    const int64_t c0 = L.cb[g.rank], c1 = L.cb[g.rank + 1];
    int bad = 0;
    double v = 0.0;
    for (int i = 0; i < blocks.count(); ++i) {
      const int64_t ilo = blocks.ilo[i], ihi = blocks.ihi[i];
      if (ilo > 0 && ilo - 1 >= c0 && ilo - 1 < c1) {
        CK(cudaMemcpy(&v, H_local + ilo + (ilo - 1 - c0) * n, sizeof(double), cudaMemcpyDeviceToHost));
        bad |= v != 0.0;
      }
      if (ihi < n - 1 && ihi >= c0 && ihi < c1) {
        CK(cudaMemcpy(&v, H_local + (ihi + 1) + (ihi - c0) * n, sizeof(double), cudaMemcpyDeviceToHost));
        bad |= v != 0.0;
      }
    }
    if (g.world > 1) {
      int* d_bad = reinterpret_cast<int*>(g.d_q);  // workspace scratch (Q slots are rewritten below)
      CK(cudaMemcpyAsync(d_bad, &bad, sizeof(int), cudaMemcpyHostToDevice, g.stream));
      NK(ncclAllReduce(d_bad, d_bad, 1, ncclInt32, ncclMax, g.comm, g.stream));
      CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, g.stream));
      CK(cudaStreamSynchronize(g.stream));
    }
    if (bad) return -10;
  }
  hqr_stats st{};
  st.window_eff = cp->plan.k;
  std::vector<RankCtx> ranks(1);
  RankCtx& r = ranks[0];
  r.rank = g.rank;
  r.H = H_local;
  r.Z = Z_local;
  r.hcols = L.cb[g.rank + 1] - L.cb[g.rank] + L.halo;
  r.zrows = L.rb[g.rank + 1] - L.rb[g.rank];
  rc = prepare_rank(*cp, L, &r);
  if (rc) return rc;
  CK(cudaEventRecord(g.ev0, g.stream));
  rc = run_dist(*cp, L, ranks, g.comm != nullptr, &st);
  if (rc) return rc;
  CK(cudaEventRecord(g.ev1, g.stream));
  CK(cudaStreamSynchronize(g.stream));
  if (r.d_owned) cudaFree(r.d_owned);
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, g.ev0, g.ev1));
  st.ms_total = ms;
  g.stats = st;
  return 0;
}

static int virtual_impl(double* H, double* Z, int64_t n, const Blocks& blocks, const double* shifts_re,
                        const double* shifts_im, int window, int vworld) {
  if (!H) return -1;
  if (vworld < 1) return -10;
  CachedPlan* cp = nullptr;
  hqr::DistLayout L;
  int rc = dist_prepare(n, blocks, shifts_re, shifts_im, window, vworld, &cp, &L);
  if (rc) return rc;
  if (!is_device_ptr(H) || (Z && !is_device_ptr(Z))) return -1;
  for (int i = 0; i < blocks.count(); ++i) {  // -10 (as hqr_sweep)
    const int64_t ilo = blocks.ilo[i], ihi = blocks.ihi[i];
    double v[2] = {0.0, 0.0};
    if (ilo > 0) CK(cudaMemcpy(&v[0], H + ilo + (ilo - 1) * n, sizeof(double), cudaMemcpyDeviceToHost));
    if (ihi < n - 1) CK(cudaMemcpy(&v[1], H + (ihi + 1) + ihi * n, sizeof(double), cudaMemcpyDeviceToHost));
    if (v[0] != 0.0 || v[1] != 0.0) return -10;
  }
  hqr_stats st{};
  st.window_eff = cp->plan.k;
  g.vH.resize(vworld, nullptr); g.vZ.resize(vworld, nullptr);
  g.vH_cap.resize(vworld, 0); g.vZ_cap.resize(vworld, 0);
  std::vector<RankCtx> ranks(vworld);
  for (int r = 0; r < vworld; ++r) {
    RankCtx& rc_ = ranks[r];
    rc_.rank = r;
    rc_.hcols = L.cb[r + 1] - L.cb[r] + L.halo;
    rc_.zrows = L.rb[r + 1] - L.rb[r];
    rc = ensure(&g.vH[r], &g.vH_cap[r], (size_t)n * rc_.hcols);
    if (rc) return rc;
    rc_.H = g.vH[r];
    // scatter: owned columns (contiguous), Z rows (strided)
    CK(cudaMemcpyAsync(rc_.H, H + L.cb[r] * n, (size_t)(L.cb[r + 1] - L.cb[r]) * n * sizeof(double),
                       cudaMemcpyDeviceToDevice, g.stream));
    rc_.Z = nullptr;
    if (Z) {
      rc = ensure(&g.vZ[r], &g.vZ_cap[r], (size_t)rc_.zrows * n);
      if (rc) return rc;
      rc_.Z = g.vZ[r];
      CK(cudaMemcpy2DAsync(rc_.Z, rc_.zrows * sizeof(double), Z + L.rb[r], n * sizeof(double),
                           rc_.zrows * sizeof(double), n, cudaMemcpyDeviceToDevice, g.stream));
    }
    rc = prepare_rank(*cp, L, &rc_);
    if (rc) return rc;
  }
  CK(cudaEventRecord(g.ev0, g.stream));
  rc = run_dist(*cp, L, ranks, false, &st);
  if (rc) return rc;
  CK(cudaEventRecord(g.ev1, g.stream));
  for (int r = 0; r < vworld; ++r) {  // gather
    RankCtx& rc_ = ranks[r];
    CK(cudaMemcpyAsync(H + L.cb[r] * n, rc_.H, (size_t)(L.cb[r + 1] - L.cb[r]) * n * sizeof(double),
                       cudaMemcpyDeviceToDevice, g.stream));
    if (Z)
      CK(cudaMemcpy2DAsync(Z + L.rb[r], n * sizeof(double), rc_.Z, rc_.zrows * sizeof(double),
                           rc_.zrows * sizeof(double), n, cudaMemcpyDeviceToDevice, g.stream));
  }
  CK(cudaStreamSynchronize(g.stream));
  for (auto& rc_ : ranks)
    if (rc_.d_owned) cudaFree(rc_.d_owned);
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, g.ev0, g.ev1));
  st.ms_total = ms;
  g.stats = st;
  return 0;
}

// ================================================================================================
// Generalized (QZ) sweep (qz.cu).  Per wavefront step: the QZ chase of every
// window (H, T windows + Q_W, Z_W in SMEM), then the DMMA update kernels of update.cu, each twice:
// left  Q_W^T on the rows of W right of it in H and in T;
// right Z_W on the columns of W above it in H and in T;
// accumulate Qacc(:, W) Q_W and Zacc(:, W) Z_W.
// One stream, in order (a step's left updates before its right updates: they meet in the blocks
// H(W_c, W_c') / T(W_c, W_c')).
// ================================================================================================
int hqr_qz_sweep(double* H, double* T, double* Q, double* Z, int64_t n, int64_t ilo, int64_t ihi,
                 const double* shifts_re, const double* shifts_im, int nshifts, int window) {
  if (!H) return -1;
  if (!T) return -2;
  Blocks b;
  b.ilo = {ilo}; b.ihi = {ihi}; b.nshifts = {nshifts};
  int rc = validate_blocks(n, b, shifts_re, shifts_im, window, true);
  if (rc) return rc;
  const int kmax = std::min(g.window_max > 0 ? g.window_max : hqr::kMaxWindowQZ, hqr::kMaxWindowQZ);
  Plan P0;
  rc = hqr::make_plan(n, ilo, ihi, nshifts, window, kmax, &P0);  // validates the window (-9)
  if (rc) return rc;
  if (!g.ready) return -100;
  if (g.world > 1) return -1;
  CK(cudaSetDevice(g.device));
  if (!is_device_ptr(H) || !is_device_ptr(T) || (Q && !is_device_ptr(Q)) || (Z && !is_device_ptr(Z))) return -1;
  {  // -10 (H decoupled at the block ends); T's leading diagonal entries divide the bulge vector (-2)
    double v[4] = {0.0, 0.0, 1.0, 1.0};
    if (ilo > 0) CK(cudaMemcpy(&v[0], H + ilo + (ilo - 1) * n, sizeof(double), cudaMemcpyDeviceToHost));
    if (ihi < n - 1) CK(cudaMemcpy(&v[1], H + (ihi + 1) + ihi * n, sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[2], T + ilo + ilo * n, sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[3], T + (ilo + 1) + (ilo + 1) * n, sizeof(double), cudaMemcpyDeviceToHost));
    if (v[0] != 0.0 || v[1] != 0.0) return -10;
    if (v[2] == 0.0 || v[3] == 0.0) return -2;
  }
  // the plan (cached like the QR sweep's, key marked as QZ: its window cap differs)
  PlanKey key = plan_key(n, b, window);
  key.push_back(-2);
  key.push_back(kmax);
  auto it = g.plans.find(key);
  if (it == g.plans.end()) {
    auto cp = std::make_unique<CachedPlan>();
    cp->plan = std::move(P0);
    cp->KP = hqr::padded_kp(cp->plan.max_kw);
    it = g.plans.emplace(key, std::move(cp)).first;
  }
  CachedPlan* cp = it->second.get();
  const Plan& P = cp->plan;
  if (!cp->d_wins) {
    CK(cudaMalloc(&cp->d_wins, P.windows.size() * sizeof(WindowDesc)));
    CK(cudaMemcpy(cp->d_wins, P.windows.data(), P.windows.size() * sizeof(WindowDesc), cudaMemcpyHostToDevice));
  }
  rc = wait_for_caller();
  if (rc) return rc;
  rc = upload_coef(shifts_re, shifts_im, P.nb);
  if (rc) return rc;
  const int KP = cp->KP, QLD = hqr::pad_ld(KP);
  const size_t slots = (size_t)hqr::kQSets * P.nchains * KP * QLD;
  rc = ensure(&g.d_q, &g.q_cap, 2 * slots);  // Q_W slots, then Z_W slots
  if (rc) return rc;
  double* zslots = g.d_q + slots;
  hqr::TensorMaps tmA, tmB;  // (H, Qacc) and (T, Zacc)
  CK(hqr::make_tensor_maps(&tmA, H, n, Q, n, n, n, KP));
  CK(hqr::make_tensor_maps(&tmB, T, n, Z, n, n, n, KP));
  hqr_stats st{};
  st.window_eff = P.k;
  // Stream A: chase -> left (H, T) -> near-right (H, T: rows [sp, w0)) per step (the next chase
  // reads their results); stream B (low priority): the far-right rows [0, sp) of H and T, Qacc Q_W
  // and Zacc Z_W, which no later chase, left or near-right update reads,
  // started after the step's left updates (a far-right block of W meets the left update of a window
  // above it in the same step) and trailing A by up to kQSets - 1 steps (rotating slot sets).
  // sp(s) = the smallest first row of any later window, even (as the fused QR kernel's split).
  // Captured once per (plan, pointers) into a CUDA graph and replayed.
  std::vector<int64_t> sp(P.nsteps, 0);
  {
    int64_t run = n;
    for (int s = P.nsteps - 1; s >= 0; --s) {
      sp[s] = run & ~(int64_t)1;
      for (int i = P.step_begin[s]; i < P.step_begin[s + 1]; ++i) run = std::min<int64_t>(run, P.windows[i].w0);
    }
  }
  auto enqueue = [&](hqr_stats* sts) -> int {
    cudaStream_t A = g.stream, Bs = g.zstream;
    CK(cudaEventRecord(g.ev_fork, A));
    CK(cudaStreamWaitEvent(Bs, g.ev_fork, 0));
    for (int s = 0; s < P.nsteps; ++s) {
      const int set = s % hqr::kQSets;
      if (s >= hqr::kQSets) CK(cudaStreamWaitEvent(A, g.ev_z[set], 0));
      StepArgs a{};
      a.n = n; a.ilo = ilo; a.ihi = ihi; a.hcol0 = 0; a.lc0 = 0; a.lc1 = n; a.zrows = n; a.ldz = n;
      a.wins = cp->d_wins; a.win_begin = P.step_begin[s]; a.win_count = P.step_begin[s + 1] - P.step_begin[s];
      a.coef = g.d_coef; a.KP = KP; a.QLD = QLD; a.slot_offset = set * P.nchains; a.step = s;
      const WindowDesc* hw = P.windows.data() + a.win_begin;
      StepArgs aH = a, aHz = a, aT = a, aTz = a;
      aH.H = H; aH.Z = Q; aH.qslots = g.d_q;             // left on H; Qacc Q_W
      aHz.H = H; aHz.Z = nullptr; aHz.qslots = zslots;   // right on H rows above W with Z_W
      aT.H = T; aT.Z = nullptr; aT.qslots = g.d_q;       // left on T
      aTz.H = T; aTz.Z = Z; aTz.qslots = zslots;         // right on T rows above W; Zacc Z_W
      CK(hqr::launch_qz_chase(aH, T, zslots, P.max_kw, A));
      sts->launches_chase++;
      int64_t items;
      double fl, by;
      auto acc = [&](int* l) { *l += items > 0; sts->flops_update += fl; sts->bytes_update += by; };
      // H's and T's updates side by side (two streams, joined before the next chase); on one matrix
      // the left update precedes the right one (a step's windows share blocks H(W1 rows, W2 cols))
      CK(cudaEventRecord(g.qz_fork, A));
      CK(cudaStreamWaitEvent(g.qzs[0], g.qz_fork, 0));
      CK(hqr::launch_left(aH, hw, g.num_sms, tmA, A, &items, &fl, &by)); acc(&sts->launches_left);
      CK(hqr::launch_left(aT, hw, g.num_sms, tmB, g.qzs[0], &items, &fl, &by)); acc(&sts->launches_left);
      CK(cudaEventRecord(g.qz_join[1], g.qzs[0]));  // the step's left updates, for B
      CK(cudaEventRecord(g.ev_q[set], A));
      StepArgs aHn = aHz, aTn = aTz;
      aHn.right_mode = 1; aHn.rrow_lo = sp[s]; aHn.rrow_hi = n;  // rows [sp, w0)
      CK(hqr::launch_right(aHn, hw, g.num_sms, tmA, A, &items, &fl, &by)); acc(&sts->launches_right);
      aTn.right_mode = 1; aTn.rrow_lo = sp[s]; aTn.rrow_hi = n;
      CK(hqr::launch_right(aTn, hw, g.num_sms, tmB, g.qzs[0], &items, &fl, &by)); acc(&sts->launches_right);
      CK(cudaEventRecord(g.qz_join[0], g.qzs[0]));
      CK(cudaStreamWaitEvent(A, g.qz_join[0], 0));
      CK(cudaStreamWaitEvent(Bs, g.ev_q[set], 0));
      CK(cudaStreamWaitEvent(Bs, g.qz_join[1], 0));
      if (sp[s] > 0) {  // far-right rows [0, sp) (rrow_hi = 0 would mean all rows)
        aHz.right_mode = 1; aHz.rrow_lo = 0; aHz.rrow_hi = sp[s];
        CK(hqr::launch_right(aHz, hw, g.num_sms, tmA, Bs, &items, &fl, &by)); acc(&sts->launches_right);
        StepArgs aTf = aTz;
        aTf.Z = nullptr; aTf.right_mode = 1; aTf.rrow_lo = 0; aTf.rrow_hi = sp[s];
        CK(hqr::launch_right(aTf, hw, g.num_sms, tmB, Bs, &items, &fl, &by)); acc(&sts->launches_right);
      }
      if (Q) {
        aH.right_mode = 2;
        CK(hqr::launch_right(aH, hw, g.num_sms, tmA, Bs, &items, &fl, &by)); acc(&sts->launches_right);
      }
      if (Z) {
        aTz.right_mode = 2;
        CK(hqr::launch_right(aTz, hw, g.num_sms, tmB, Bs, &items, &fl, &by)); acc(&sts->launches_right);
      }
      CK(cudaEventRecord(g.ev_z[set], Bs));
    }
    CK(cudaEventRecord(g.ev_join, Bs));
    CK(cudaStreamWaitEvent(A, g.ev_join, 0));
    sts->steps = P.nsteps;
    sts->windows = (int64_t)P.windows.size();
    sts->kernels_launched = sts->launches_chase + sts->launches_left + sts->launches_right;
    return 0;
  };
  CK(cudaEventRecord(g.ev0, g.stream));
  if (g.flags & (HQR_FLAG_NO_GRAPH | HQR_FLAG_PROFILE)) {
    rc = enqueue(&st);
    if (rc) return rc;
  } else {
    GraphKey gk{key, H, T};
    gk.pk.push_back((int64_t)(uintptr_t)Q);
    gk.pk.push_back((int64_t)(uintptr_t)Z);
    auto git = g.graphs.find(gk);
    if (git == g.graphs.end()) {
      cudaGraph_t graph;
      hqr_stats cap{};
      CK(cudaStreamBeginCapture(g.stream, cudaStreamCaptureModeThreadLocal));
      const int rc2 = enqueue(&cap);
      const cudaError_t ec = cudaStreamEndCapture(g.stream, &graph);
      if (rc2) return rc2;
      CK(ec);
      cudaGraphExec_t exec;
      CK(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      git = g.graphs.emplace(gk, CachedGraph{exec, cap}).first;
    }
    CK(cudaGraphLaunch(git->second.exec, g.stream));
    const hqr_stats& c = git->second.stats;
    st.flops_update = c.flops_update; st.bytes_update = c.bytes_update;
    st.launches_chase = c.launches_chase; st.launches_left = c.launches_left; st.launches_right = c.launches_right;
    st.steps = c.steps; st.windows = c.windows; st.kernels_launched = c.kernels_launched;
  }
  CK(cudaEventRecord(g.ev1, g.stream));
  CK(cudaStreamSynchronize(g.stream));
  CK(cudaGetLastError());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, g.ev0, g.ev1));
  st.ms_total = ms;
  g.stats = st;
  g.wstats_plan = nullptr;  // flops_dmma is not tracked for the QZ sweep
  return 0;
}

// ================================================================================================
// QR iteration (partial, reading R21): sweeps of the bottom unreduced block
// with the eigenvalues of its trailing nshifts x nshifts block as shifts, deflation after each
// sweep, small blocks solved by the one-CTA Francis QR (qriter.cu).  The sweep is hqr_sweep's
// product path (fused persistent kernel).  The host only orchestrates (finds the block from the
// subdiagonal, pairs the shifts, loops).
// ================================================================================================
namespace {
int make_shifts_host(const double* wr, const double* wi, int m, int ns, double* sr, double* si) {
  int k = 0;  // complex pairs in the order found, then the reals paired in the order found (R21)
  for (int j = 0; j < m && k + 1 < ns; ++j)
    if (wi[j] > 0.0) {
      sr[k] = wr[j]; si[k] = wi[j]; sr[k + 1] = wr[j]; si[k + 1] = -wi[j];
      k += 2;
    }
  int pending = -1;
  for (int j = 0; j < m && k + 1 < ns; ++j)
    if (wi[j] == 0.0) {
      if (pending < 0) {
        pending = j;
      } else {
        sr[k] = wr[pending]; si[k] = 0.0; sr[k + 1] = wr[j]; si[k + 1] = 0.0;
        k += 2;
        pending = -1;
      }
    }
  return k;
}

// One AED step on the window [k0, k0+nwin) (the trailing rows of the unreduced block [l, hi]):
// the one-CTA kernel (Schur form, spike, deflation with reordering, Hessenberg re-reduction), then,
// when something deflated, the window factor U applied to the rest of H and to Z by the DMMA update
// kernels (left: H(window, right of it); right: H(above, window), Z(:, window)).  ewr / ewi (host,
// nwin) receive the eigenvalues of the final window blocks in window order; *nd / *m the deflated /
// undeflated counts (*nd < 0: the window's Schur iteration did not converge, nothing changed).
cudaError_t aed_step(double* H, double* Z, int64_t n, int64_t l, int64_t hi, int nwin, double thr,
                     double* d_uslot, int KPa, int QLDa, double* d_ew, double* d_ei, int* d_res, WindowDesc* d_wd,
                     const hqr::TensorMaps& tma, double* ewr, double* ewi, int* nd, int* m) {
  const int64_t k0 = hi - nwin + 1;
  int res[2] = {0, 0};
  cudaError_t e = hqr::launch_aed(H, n, l, k0, nwin, thr, d_uslot, KPa, QLDa, d_ew, d_ei, d_res, g.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(res, d_res, 2 * sizeof(int), cudaMemcpyDeviceToHost, g.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ewr, d_ew, nwin * sizeof(double), cudaMemcpyDeviceToHost, g.stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ewi, d_ei, nwin * sizeof(double), cudaMemcpyDeviceToHost, g.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g.stream);
  if (e != cudaSuccess) return e;
  *nd = res[0];
  *m = res[1];
  if (res[0] <= 0) return cudaSuccess;
  WindowDesc wd{};
  wd.w0 = (int32_t)k0; wd.w1 = (int32_t)(k0 + nwin - 1); wd.slot = 0; wd.nbc = 0;
  wd.ilo = (int32_t)l; wd.ihi = (int32_t)hi; wd.scan_lo = 0; wd.scan_hi = -1;
  e = cudaMemcpyAsync(d_wd, &wd, sizeof(wd), cudaMemcpyHostToDevice, g.stream);
  if (e != cudaSuccess) return e;
  StepArgs a{};
  a.H = H; a.Z = Z; a.n = n; a.ilo = l; a.ihi = hi; a.hcol0 = 0; a.lc0 = 0; a.lc1 = n; a.zrows = n; a.ldz = n;
  a.wins = d_wd; a.win_begin = 0; a.win_count = 1; a.qslots = d_uslot; a.KP = KPa; a.QLD = QLDa;
  a.slot_offset = 0; a.right_mode = 0;
  int64_t items;
  double fl, by;
  e = hqr::launch_left(a, &wd, g.num_sms, tma, g.stream, &items, &fl, &by);
  if (e == cudaSuccess) e = hqr::launch_right(a, &wd, g.num_sms, tma, g.stream, &items, &fl, &by);
  return e;
}
}  // namespace

int hqr_qr_iterate(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, int nshifts, int window,
                   int nmin, int aed_window, int max_sweeps, double* wr, double* wi, int* sweeps_out) {
  if (!H) return -1;
  if (n < 1) return -3;
  if (ilo < 0 || ilo > ihi) return -4;
  if (ihi >= n) return -5;
  if (nshifts < 2 || (nshifts & 1) || nshifts > hqr::small_eig_max()) return -6;
  if (window < 1) return -7;
  if (nmin < 2 || nmin > hqr::small_eig_max()) return -8;
  if (aed_window < 0 || aed_window == 1 || aed_window > hqr::kMaxWindow) return -9;
  if (!wr || !wi) return -10;
  if (!g.ready) return -100;
  if (g.world > 1) return -1;
  CK(cudaSetDevice(g.device));
  if (!is_device_ptr(H) || (Z && !is_device_ptr(Z))) return -1;
  const int SM = hqr::small_eig_max();
  // the AED factor slot also serves the small blocks left at the end (R24: up to kMaxWindow rows)
  const int KPa = hqr::padded_kp(std::max({aed_window, std::min(nmin, hqr::kMaxWindow), 2})),
            QLDa = hqr::pad_ld(KPa);
  // scratch: eigenvalues (2 SM), AED eigenvalues (2 kMaxWindow), ||H||^2, ints, the AED factor slot,
  // the AED window descriptor
  const size_t nscr = 2 * (size_t)SM + 2 * (size_t)hqr::kMaxWindow + 8 + (size_t)KPa * QLDa + 16;
  double* d_w = nullptr;
  CK(cudaMalloc(&d_w, nscr * sizeof(double)));
  double* d_ew = d_w + 2 * SM;
  double* d_ei = d_ew + hqr::kMaxWindow;
  double* d_fro = d_ei + hqr::kMaxWindow;
  int* d_info = reinterpret_cast<int*>(d_fro + 1);   // [0] info, [1] deflate count, [2..3] AED res
  double* d_uslot = d_fro + 8;
  WindowDesc* d_wd = reinterpret_cast<WindowDesc*>(d_uslot + (size_t)KPa * QLDa);
  std::vector<double> sub((size_t)std::max<int64_t>(n - 1, 1)), ewr(std::max(nshifts, hqr::kMaxWindow)),
      ewi(ewr.size()), sr(nshifts), si(nshifts);
  int sweeps = 0, rc = 0, naed = 0, ndefl = 0;
  int64_t hi = ihi;
  double falg = 0.0, thr = 0.0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventRecord(t0, g.stream));
  auto fail = [&](int code) { cudaFree(d_w); cudaEventDestroy(t0); cudaEventDestroy(t1); return code; };
  if (aed_window > 0) {  // deflation threshold u ||H||_F (the paper's default norm-stable condition, R22)
    double fro2 = 0.0;
    cudaError_t e = hqr::launch_fro2(H, n * n, d_fro, g.num_sms, g.stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&fro2, d_fro, sizeof(double), cudaMemcpyDeviceToHost, g.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g.stream);
    if (e != cudaSuccess) return fail(cuerr(e));
    thr = 0x1p-53 * std::sqrt(fro2);
  }
  hqr::TensorMaps tma;
  {
    cudaError_t e = hqr::make_tensor_maps(&tma, H, n, Z, n, n, n, KPa);
    if (e != cudaSuccess) return fail(cuerr(e));
  }
  while (hi >= ilo) {
    // the bottom unreduced block [l, hi]: the subdiagonal h(k, k-1), k = ilo+1 .. hi (stride n+1)
    int64_t l = hi;
    if (hi > ilo) {
      const int64_t cnt = hi - ilo;
      cudaError_t e = cudaMemcpy2D(sub.data(), sizeof(double), H + (ilo + 1) + ilo * n, (n + 1) * sizeof(double),
                                   sizeof(double), (size_t)cnt, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return fail(cuerr(e));
      while (l > ilo && sub[(size_t)(l - 1 - ilo)] != 0.0) --l;
    }
    const int64_t N = hi - l + 1;
    if (N <= nmin) {  // small block: real Schur form (R24), its eigenvalues from the diagonal blocks
      if (N == 1) {
        cudaError_t e = cudaMemcpy(wr + l, H + l + l * n, sizeof(double), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return fail(cuerr(e));
        wi[l] = 0.0;
        hi = l - 1;
        continue;
      }
      if (N <= hqr::kMaxWindow) {
        // the AED window machinery with the block's first row as the window start: the spike is
        // zero, every block deflates (threshold 0), T and U are applied to the rest of H and to Z
        int nd = 0, m = 0;
        cudaError_t e = aed_step(H, Z, n, l, hi, (int)N, 0.0, d_uslot, KPa, QLDa, d_ew, d_ei, d_info + 2, d_wd, tma,
                                 ewr.data(), ewi.data(), &nd, &m);
        if (e != cudaSuccess) return fail(cuerr(e));
        if (nd == N) {
          for (int j = 0; j < N; ++j) {
            wr[l + j] = ewr[j];
            wi[l + j] = ewi[j];
          }
          hi = l - 1;
          continue;
        }
        // (not converged: H unchanged, the eigenvalue-only solver below)
      }
      cudaError_t e = hqr::launch_small_eig(H, n, l, (int)N, d_w, d_w + SM, d_info, g.stream);
      if (e == cudaSuccess) e = cudaMemcpyAsync(wr + l, d_w, N * sizeof(double), cudaMemcpyDeviceToHost, g.stream);
      if (e == cudaSuccess) e = cudaMemcpyAsync(wi + l, d_w + SM, N * sizeof(double), cudaMemcpyDeviceToHost, g.stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(g.stream);
      if (e != cudaSuccess) return fail(cuerr(e));
      hi = l - 1;
      continue;
    }
    if (sweeps >= max_sweeps) {
      rc = (int)(hi + 1);  // LAPACK-style: the eigenvalues of rows ilo..hi were not found
      break;
    }
    int k = 0;  // shifts found
    if (aed_window > 0) {
      // AED on the trailing window (R22): Schur form, spike, deflation, Hessenberg re-reduction,
      // then the window's factor U propagated by the DMMA update kernels
      const int nwin = (int)std::min<int64_t>(aed_window, N);
      const int64_t k0 = hi - nwin + 1;
      int nd = 0, m = 0;
      cudaError_t e = aed_step(H, Z, n, l, hi, nwin, thr, d_uslot, KPa, QLDa, d_ew, d_ei, d_info + 2, d_wd, tma,
                               ewr.data(), ewi.data(), &nd, &m);
      if (e != cudaSuccess) return fail(cuerr(e));
      ++naed;
      if (nd < 0) {  // the window's Schur iteration did not converge: plain shifts below
        k = 0;
      } else {
        if (nd > 0) {
          for (int j = m; j < nwin; ++j) {
            wr[k0 + j] = ewr[j];
            wi[k0 + j] = ewi[j];
          }
          ndefl += nd;
          hi -= nd;
          if (100 * nd > 14 * nwin) continue;  // many deflations: another AED before a sweep
          if (hi - l + 1 <= nmin) continue;
        }
        // the bottom-most undeflated candidates (the failed ones) as shifts
        const int want = std::min(nshifts, m);
        k = make_shifts_host(ewr.data() + (m - want), ewi.data() + (m - want), want, want, sr.data(), si.data());
        if (k > hi - l + 1) k = (int)((hi - l + 1) & ~(int64_t)1);
      }
    }
    if (k < 2) {  // shifts: the eigenvalues of the trailing nshifts x nshifts block
      const int64_t Nb = hi - l + 1;
      int ns = (int)std::min<int64_t>(nshifts, (Nb - 2) & ~(int64_t)1);
      if (ns < 2) ns = 2;
      cudaError_t e = hqr::launch_small_eig(H, n, hi - ns + 1, ns, d_w, d_w + SM, d_info, g.stream);
      if (e == cudaSuccess) e = cudaMemcpyAsync(ewr.data(), d_w, ns * sizeof(double), cudaMemcpyDeviceToHost, g.stream);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(ewi.data(), d_w + SM, ns * sizeof(double), cudaMemcpyDeviceToHost, g.stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(g.stream);
      if (e != cudaSuccess) return fail(cuerr(e));
      k = make_shifts_host(ewr.data(), ewi.data(), ns, ns, sr.data(), si.data());
      if (k < 2) {
        rc = (int)(hi + 1);
        break;
      }
    }
    const int src = sweep_impl(H, Z, n, make_blocks(1, &l, &hi, &k), sr.data(), si.data(), window);
    if (src) return fail(src);
    falg += g.stats.flops_alg;
    ++sweeps;
    CK(cudaMemsetAsync(d_info + 1, 0, sizeof(int), g.stream));
    cudaError_t e = hqr::launch_deflate(H, n, l, hi, d_info + 1, g.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g.stream);
    if (e != cudaSuccess) return fail(cuerr(e));
  }
  CK(cudaEventRecord(t1, g.stream));
  CK(cudaEventSynchronize(t1));
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaFree(d_w);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  g.stats.ms_total = ms;  // the whole iteration (device time of the library stream)
  g.stats.flops_alg = falg;
  g.stats.steps = sweeps;
  g.stats.launches_chase = naed;    // (re-used: AED steps)
  g.stats.window_eff = ndefl;       // (re-used: eigenvalues deflated by AED)
  if (sweeps_out) *sweeps_out = sweeps;
  return rc;
}

int hqr_aed(double* H, double* Z, int64_t n, int64_t ilo, int64_t k0, int nw, double thr, double* ew, double* ei,
            int* nd_out, int* nund_out) {
  if (!H) return -1;
  if (n < 1) return -3;
  if (ilo < 0 || k0 < ilo || k0 + nw > n) return -4;
  if (nw < 2 || nw > hqr::kMaxWindow) return -9;
  if (!ew || !ei || !nd_out || !nund_out) return -10;
  if (!g.ready) return -100;
  if (g.world > 1) return -1;
  CK(cudaSetDevice(g.device));
  if (!is_device_ptr(H) || (Z && !is_device_ptr(Z))) return -1;
  const int KPa = hqr::padded_kp(nw), QLDa = hqr::pad_ld(KPa);
  const size_t nscr = 2 * (size_t)hqr::kMaxWindow + 8 + (size_t)KPa * QLDa + 16;
  double* d_w = nullptr;
  CK(cudaMalloc(&d_w, nscr * sizeof(double)));
  double* d_ew = d_w;
  double* d_ei = d_ew + hqr::kMaxWindow;
  int* d_res = reinterpret_cast<int*>(d_ei + hqr::kMaxWindow);
  double* d_uslot = d_ei + hqr::kMaxWindow + 8;
  WindowDesc* d_wd = reinterpret_cast<WindowDesc*>(d_uslot + (size_t)KPa * QLDa);
  hqr::TensorMaps tma;
  cudaError_t e = hqr::make_tensor_maps(&tma, H, n, Z, n, n, n, KPa);
  int nd = 0, m = 0;
  if (e == cudaSuccess)
    e = aed_step(H, Z, n, ilo, k0 + nw - 1, nw, thr, d_uslot, KPa, QLDa, d_ew, d_ei, d_res, d_wd, tma, ew, ei, &nd, &m);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g.stream);
  cudaFree(d_w);
  if (e != cudaSuccess) return cuerr(e);
  *nd_out = nd;
  *nund_out = m;
  return 0;
}

int hqr_get_aftermath(signed char* flags, int64_t n) {
  if (!flags) return -1;
  if (!g.ready || g.aft_n == 0) return -100;
  if (n != g.aft_n) return -3;
  CK(cudaSetDevice(g.device));
  CK(cudaMemcpy(flags, g.d_aft, (size_t)n, cudaMemcpyDeviceToHost));
  return 0;
}

int hqr_sweep_dist(double* H_local, double* Z_local, int64_t n, int64_t ilo, int64_t ihi,
                   const double* shifts_re, const double* shifts_im, int nshifts, int window) {
  return dist_impl(H_local, Z_local, n, make_blocks(1, &ilo, &ihi, &nshifts), shifts_re, shifts_im, window);
}

int hqr_sweep_dist_multi(double* H_local, double* Z_local, int64_t n, int nblocks, const int64_t* ilo,
                         const int64_t* ihi, const double* shifts_re, const double* shifts_im,
                         const int* nshifts, int window) {
  if (!H_local) return -1;
  if (nblocks < 1 || !ilo || !ihi || !nshifts) return -4;
  return dist_impl(H_local, Z_local, n, make_blocks(nblocks, ilo, ihi, nshifts), shifts_re, shifts_im, window);
}

int hqr_sweep_virtual(double* H, double* Z, int64_t n, int64_t ilo, int64_t ihi, const double* shifts_re,
                      const double* shifts_im, int nshifts, int window, int vworld) {
  return virtual_impl(H, Z, n, make_blocks(1, &ilo, &ihi, &nshifts), shifts_re, shifts_im, window, vworld);
}

int hqr_sweep_virtual_multi(double* H, double* Z, int64_t n, int nblocks, const int64_t* ilo,
                            const int64_t* ihi, const double* shifts_re, const double* shifts_im,
                            const int* nshifts, int window, int vworld) {
  if (!H) return -1;
  if (nblocks < 1 || !ilo || !ihi || !nshifts) return -4;
  return virtual_impl(H, Z, n, make_blocks(nblocks, ilo, ihi, nshifts), shifts_re, shifts_im, window, vworld);
}

int hqr_get_stats(hqr_stats* out) {
  if (!out) return -1;
  *out = g.stats;
  out->flops_dmma = 0.0;
  // executed DMMA flops of the last single-GPU sweep: per window 2 U (n - w1 - 1 + w0 + zrows),
  // U recorded by the chase from the factor's band extents (TMA path; the cp.async path for odd n
  // multiplies full K and is not counted)
  if (g.wstats_plan && g.d_wstats && g.ready) {
    const CachedPlan* cp = static_cast<const CachedPlan*>(g.wstats_plan);
    const auto& W = cp->plan.windows;
    std::vector<double> u(W.size());
    if (cudaMemcpy(u.data(), g.d_wstats, u.size() * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess) {
      double f = 0.0;
      for (size_t i = 0; i < W.size(); ++i)
        f += 2.0 * u[i] * ((double)(g.wstats_n - 1 - W[i].w1) + (double)W[i].w0 + (g.wstats_z ? (double)g.wstats_n : 0.0));
      out->flops_dmma = f;
    }
  }
  return 0;
}

const char* hqr_error_string(int code) {
  switch (code) {
    case 0: return "ok";
    case -1: return "H is NULL / invalid config";
    case -2: return "T is NULL or T[ilo,ilo] / T[ilo+1,ilo+1] is zero (QZ)";
    case -3: return "n < 1";
    case -4: return "ilo < 0 or ilo > ihi";
    case -5: return "ihi >= n or active block shorter than 3";
    case -6: return "non-finite shift (or shifts_re NULL)";
    case -7: return "shift pair is neither two reals nor an exact conjugate pair (or shifts_im NULL)";
    case -8: return "nshifts odd, < 2 or larger than the active block";
    case -9: return "window out of range";
    case -10: return "active block not decoupled (H[ilo,ilo-1] or H[ihi+1,ihi] nonzero)";
    case -100: return "library not set up (call hqr_setup)";
    case -101: return "no usable sm_100 CUDA device";
    case -11: return "matrix too small for the number of shards (each needs >= HQR_MAX_WINDOW + 8 columns)";
  }
  if (code >= 2000) return "NCCL error (code - 2000 = ncclResult_t)";
  if (code >= 1000) return "CUDA error (code - 1000 = cudaError_t)";
  return "unknown error";
}

}  // extern "C"
