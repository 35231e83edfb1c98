// step.hpp -- the fused wavefront-step kernel (step.cu): task queue types and launcher.
#pragma once
#include <cstdint>
#include <vector>

#include "kernels.hpp"

namespace hqr {

constexpr int kTaskLeft = 0, kTaskRight = 1, kTaskZ = 2, kTaskChase = 3;
constexpr int kMaxChaseBulges = 64;  // bulges per window the fused chase handles

struct Task {       // one claimable unit of work of a wavefront step
  int32_t type;     // kTaskLeft / kTaskRight / kTaskZ / kTaskChase
  int32_t win;      // window index within the step (kTaskChase: within the next step)
  int32_t tile0, ntiles;
  int64_t r_lo, r_hi;  // kTaskRight: H rows [r_lo, r_hi), tiles of right_rows(KP) from r_lo
};

struct StepCounters {  // per step, zeroed before the sweep
  int next;     // next task to claim
  int l_done;   // left tiles done x 4 (one release add per consumer warp)
  int rn_done;  // near-right tiles done x 4
  int pad;
};

struct ChunkSizes {   // tiles per task, per phase
  int left = 16, near = 16, bulk = 32;
  int tail = 1500, tail_chunk = 8;  // the queue's last `tail` tiles in chunks of `tail_chunk`
};

// Tasks of one step in queue order (L, Rn, C, Z, Rf).
void build_step_tasks(const StepArgs& a, const WindowDesc* wins, int nwin, const WindowDesc* next_wins,
                      int nnext, int64_t sp, const ChunkSizes& cs, std::vector<Task>* out, int* nL,
                      int* nRn);

// One persistent launch (one CTA per SM) running the step's task queue.  Needs the TMA path.
// nL / nRn: tasks of the L / Rn phases; nLt / nRnt: their tiles (completion is counted per tile).
cudaError_t launch_step(const StepArgs& a, const StepArgs& an, const Task* tasks, int ntasks, int nL,
                        int nRn, int nLt, int nRnt, StepCounters* ctr, const TensorMaps& tm, int max_kw, int num_sms,
                        cudaStream_t st);

// Debugging builds (-DHQR_PROGRESS): progress buffer in host-mapped memory, dumped after
// HQR_PROGRESS_SECS seconds (then the process exits).  No-op otherwise.
void debug_progress_init();
// Debugging builds (-DHQR_TIMING): per-step timestamps; reset before a sweep, print after it.
void debug_timing(int nsteps, bool reset);

}  // namespace hqr
