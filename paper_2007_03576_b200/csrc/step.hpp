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
  int l_done;   // completed left chunks
  int rn_done;  // completed near-right chunks
  int pad;
};

struct ChunkSizes {   // tiles per task, per phase
  int left = 12, near = 6, bulk = 24;
  int tail = 1200, tail_chunk = 6;  // the queue's last `tail` tiles in chunks of `tail_chunk`
};

// Tasks of one step in queue order (L, Rn, C, Z, Rf).
void build_step_tasks(const StepArgs& a, const WindowDesc* wins, int nwin, const WindowDesc* next_wins,
                      int nnext, int64_t sp, const ChunkSizes& cs, std::vector<Task>* out, int* nL,
                      int* nRn);

// One persistent launch (one CTA per SM) running the step's task queue.  Needs the TMA path.
cudaError_t launch_step(const StepArgs& a, const StepArgs& an, const Task* tasks, int ntasks, int nL,
                        int nRn, StepCounters* ctr, const TensorMaps& tm, int max_kw, int num_sms,
                        cudaStream_t st);

}  // namespace hqr
