// step.hpp -- the fused wavefront-step kernel (step.cu): task queue types and launcher.
#pragma once
#include <cstdint>
#include <vector>

#include "kernels.hpp"

namespace hqr {

// Task types.  Left / RightNear-rest / RightFar / Z: GEMM tiles of one window; Chase: the chase of a
// window of the next step.  LeftNear / RightNear: the few tiles the next step's chases read (below).
constexpr int kTaskLeft = 0, kTaskRight = 1, kTaskZ = 2, kTaskChase = 3, kTaskLeftNear = 4,
              kTaskRightNear = 5, kTaskRightFar = 6;
constexpr int kMaxChaseBulges = 64;  // bulges per window the fused chase handles

struct Task {       // one claimable unit of work of a wavefront step
  int32_t type;     // kTask*
  int32_t win;      // window index within the step (kTaskChase: within the next step)
  int32_t tile0, ntiles;
  int32_t step;     // wavefront step
  int32_t idx;      // index within the step's queue
  int64_t r_lo, r_hi;  // right tasks: H rows [r_lo, r_hi), tiles of right_rows(KP) from r_lo
};

struct StepInfo {   // per wavefront step (device array)
  int32_t win_begin, win_count, slot_offset;
  int32_t nL, nRn;          // tasks of the left / near-right phases (near parts included)
  int32_t nLt, nRnt;        // their tiles
  int32_t ntiles;           // all GEMM tiles of the step
  int32_t up_need;          // host-buffer sweeps: the last upload chunk its tasks (and the chase of
                            // step g+1) need (chunks of kUploadChunk H rows / Z columns)
};

constexpr int kUploadChunk = 512;

struct WinDeps {    // per plan window (device array)
  int32_t pred[3];          // windows of the previous step whose columns meet this one (-1: none)
  int32_t ztiles, rftiles;  // its Z / far-right tiles
  int32_t lnear, rnear;     // its LeftNear / RightNear tiles
  int32_t rn_over;          // RightNear: the window of its step whose rows meet those rows (-1: none)
  int32_t c_pred, c_below;  // its chase: the previous step's windows meeting it from above / below
  int32_t pad[2];
};

// The chase of window W' (step g+1) reads H(W', W'); at step g only these tasks write there: the
// chases of the step-g windows meeting W' -- the predecessor X (w0_X <= w0') and the window Y
// below -- X's left tiles on columns (w1_X, w1'] and Y's right tiles on rows [w0', w0_Y).  Those
// tiles form the LeftNear task of X and the RightNear task of Y; the chase waits for them (and for
// step g-1's left / near-right phases) instead of for the whole left / near-right phases of step g,
// so it overlaps them.  A RightNear task of Y also waits for the LeftNear task of the window whose
// rows meet its rows (they update the same block H(rows, Y) from the two sides); LeftNear covers
// those columns too.  Every left / near-right task of step g waits for step g-1's left and
// near-right phases (previously implied by waiting for the chase).

// Completion counters (device, zeroed per sweep):
//   step_ctr[4 g + 0]  left tiles of step g done x 4 (one release add per consumer warp)
//   step_ctr[4 g + 1]  near-right tiles x 4
//   step_ctr[4 g + 2]  all GEMM tiles x 4
//   win_ctr[kWinCtr w + 0]   chase of plan window w done (1)
//   win_ctr[kWinCtr w + 1]   Z tiles of w x 4;  + 2  far-right tiles of w x 4
//   win_ctr[kWinCtr w + 3]   LeftNear tiles of w x 4;  + 4  RightNear tiles of w x 4
constexpr int kWinCtr = 8;

struct ChunkSizes {   // tiles per task, per phase
  int left = 24, near = 48, bulk = 48;  // tuned for the persistent sweep (configs[3], tools/tune_chunks.sh)
  int tail = 0, tail_chunk = 8;  // the queue's last `tail` tiles in chunks of `tail_chunk`
  int ltail = 300, ntail = 0, phase_chunk = 2;  // the left phase's last tiles in small chunks (tools/tune_phase_tail.sh)
  int near_task = 1;  // tiles per LeftNear / RightNear task: the next chase waits for these (one tile
                      // each: the tiles of one window run on several SMs at once)
};

// Tasks of one step in queue order (LeftNear, RightNear, C, L, Rn, Z, Rf).
// lnear[i]: LeftNear tiles of window i; rnear[i]: first row of its RightNear rows (>= w0: none).
void build_step_tasks(const StepArgs& a, const WindowDesc* wins, int nwin, const WindowDesc* next_wins,
                      int nnext, int64_t sp, const ChunkSizes& cs, const int* lnear, const int64_t* rnear,
                      std::vector<Task>* out, int* nL, int* nRn);

// One persistent launch (one CTA per SM) running `ntasks` tasks -- one step's queue, or the whole
// sweep's -- claimed through *next_ctr.  base: the sweep's StepArgs (per-step fields come from
// steps[]).  Task i of `tasks` is task task_base + i of the sweep; its dependencies are
// deps[dep_begin[t] .. dep_begin[t+1]) (t the sweep index): (task, count) pairs, wait until
// task_ctr[task] >= count (per-task completion counts: 4 per GEMM tile -- one per consumer warp --,
// 1 per chase).  Needs the TMA path.
// up_flags (nullable): per upload chunk, nonzero once on the device (host-buffer sweeps).
// crit_sms > 0: CTAs 0 .. crit_sms-1 claim tasks qidx[0 .. ncrit) through next_ctr[0], the others
// qidx[ncrit .. ntasks) through next_ctr[1] (two queues, each in list order); 0: one queue in list
// order through next_ctr[0] (qidx unused).
cudaError_t launch_step(const StepArgs& base, const StepInfo* steps, int nsteps, const Task* tasks, int ntasks,
                        int task_base, const int32_t* dep_begin, const int2* deps, int* next_ctr, int* step_ctr,
                        int* task_ctr, const int* up_flags, const TensorMaps& tm, int max_kw, int num_sms,
                        cudaStream_t st, const int32_t* qidx, int ncrit, int crit_sms);

// Debugging builds (-DHQR_PROGRESS): progress buffer in host-mapped memory, dumped after
// HQR_PROGRESS_SECS seconds (then the process exits).  No-op otherwise.
void debug_progress_init();
// Debugging builds (-DHQR_TIMING): per-step timestamps; reset before a sweep, print after it.
void debug_timing(int nsteps, bool reset);

}  // namespace hqr
