// dist.hpp -- host logic of the sharded (multi-GPU) sweep: layout, ownership, lending.
// Product path; no CUDA types (unit-tested through hqr_dist_query on the CPU).
//
// Layout (BASELINE north_star "H is block-column and Z block-row sharded"; the paper's distributed
// blocks, one process per GPU as one process per node):
//   * rank r owns H columns [cb[r], cb[r+1]) (all n rows, column-major, ld = n) followed by `halo`
//     spare columns; the boundaries cb[r] = n * sqrt(r / p) (rounded to even) balance the work,
//     which grows linearly with the column index (left updates reach column j from every window
//     left of j, right updates of the window at j span j rows);
//   * rank r owns Z rows [rb[r], rb[r+1]) (uniform, even), all n columns, ld = rows.
// Ownership: window W = [w0, w1] belongs to the rank owning column w0: it chases W, broadcasts Q_W
// (ncclBroadcast, root = owner) and applies the right update H(0:w0, W) Q_W.  Every rank applies
// the left update Q_W^T H(W, j) to the columns j > w1 it holds and Z(its rows, W) Q_W.
// Straddling window (w1 >= cb[owner+1], "the window slab moves when a bulge chain crosses a shard
// boundary"): for that step rank owner+1 lends its leading columns [cb[owner+1], w1] (whole columns,
// n rows) to the owner's halo, takes them out of its own left-update range, and gets them back at
// the end of the step.  The owner then holds every column of W and performs every update of the
// step on them (the chase, the left updates of the windows above, the right update of W).
// Shards are at least kmax + 8 columns wide, so a window meets at most two ranks.
#pragma once
#include <cmath>
#include <cstdint>
#include <vector>

#include "plan.hpp"

namespace hqr {

struct DistLayout {
  int world = 1;
  std::vector<int64_t> cb;  // H column boundaries, world + 1 entries
  std::vector<int64_t> rb;  // Z row boundaries, world + 1 entries
  int halo = 0;             // spare local H columns after the owned range
};

// Returns 0, or -11 when n is too small for `world` shards of width >= kmax + 8.
inline int make_layout(int64_t n, int world, int kmax, DistLayout* L) {
  L->world = world;
  L->halo = kmax;
  L->cb.assign(world + 1, 0);
  L->rb.assign(world + 1, 0);
  for (int r = 1; r < world; ++r) {
    int64_t c = (int64_t)std::llround((double)n * std::sqrt((double)r / world));
    int64_t q = (int64_t)std::llround((double)n * r / world);
    L->cb[r] = c & ~(int64_t)1;
    L->rb[r] = q & ~(int64_t)1;
  }
  L->cb[world] = n;
  L->rb[world] = n;
  for (int r = 0; r < world; ++r) {
    if (L->cb[r + 1] - L->cb[r] < kmax + 8) return -11;
    if (L->rb[r + 1] - L->rb[r] < 2) return -11;
  }
  return 0;
}

inline int owner_of_col(const DistLayout& L, int64_t col) {
  int r = 0;
  while (r + 1 < L.world && col >= L.cb[r + 1]) ++r;
  return r;
}

// What rank r does in one wavefront step.
struct RankStep {
  std::vector<int32_t> owned;  // indices into plan.windows: chase + Q broadcast root + right update
  int64_t lend_out = 0;        // my leading columns lent to rank r-1 during this step
  int64_t lend_in = 0;         // rank r+1's leading columns held in my halo during this step
  int64_t lc0 = 0, lc1 = 0;    // global columns [lc0, lc1) this rank left-updates (and holds)
};

inline void rank_step(const Plan& P, const DistLayout& L, int r, int step, RankStep* out) {
  RankStep rs;
  for (int i = P.step_begin[step]; i < P.step_begin[step + 1]; ++i) {
    const WindowDesc& w = P.windows[i];
    const int o = owner_of_col(L, w.w0);
    if (o == r) rs.owned.push_back(i);
    if (o + 1 < L.world && w.w1 >= L.cb[o + 1]) {  // straddles the boundary cb[o+1]
      const int64_t cnt = (int64_t)w.w1 - L.cb[o + 1] + 1;
      if (o == r) rs.lend_in = cnt;
      if (o + 1 == r) rs.lend_out = cnt;
    }
  }
  rs.lc0 = L.cb[r] + rs.lend_out;
  rs.lc1 = L.cb[r + 1] + rs.lend_in;
  *out = std::move(rs);
}

}  // namespace hqr
