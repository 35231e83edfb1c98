// plan.hpp -- host planner for one multishift QR sweep on B200 (product path; no CUDA types).
//
// Turns (n, ilo, ihi, nshifts, window) into the wavefront schedule the kernels execute:
//   * bulge chains ("the set of bulges can be divided into several subsets and
//     each subset can be associated with a corresponding bulge chasing window chain");
//   * each chain's sequence of overlapping diagonal windows (window of at most
//     2*b_tile, at most (b_tile-1)/3 bulges per window; here the window side k plays 2*b_tile, so a
//     chain holds nbc_max = floor((k-2)/6) bulges and a window advances s = k - 3*nbc_max - 1 rows);
//   * the wavefront: global step g runs one window of every active chain (disjoint diagonal blocks,
//     one CTA each), then that step's off-diagonal updates.  Chains are packed as tightly as the
//     disjointness allows ("the diagonal windows are packed as close to each other as possible"):
//     chain c starts L = ceil(k/s) steps after chain c-1.
// Chain 0 carries the first shift pairs (bulges 0..), so it is the lowest chain on the diagonal.
// Chain-local step t puts bulge jj of the chain at p = ilo - 1 + t - 3*jj (spacing 3).
// Window i of a chain covers rows/cols [ilo + i*s, min(ilo + i*s + k - 1, ihi)] and runs chain-local
// steps [T_i, T_{i+1}) with T_0 = 0, T_{i+1} = i*s + k - 3, so every active bulge keeps
// w0 <= p and p + 4 <= w1 (the bulge and the row it creates stay inside); the window whose bottom is
// ihi runs until the chain's top bulge has left through the final 2x2 reflector at p = ihi - 2.
// If the whole active block fits one window (N <= k) a single window holds all bulges.
// Several decoupled active blocks ("concurrent processing of several unreduced
// blocks"; BASELINE configs[4]) are planned independently and merged step by step: their windows
// lie in disjoint diagonal blocks, so one wavefront step simply carries windows of every block.
// See DESIGN.md §6 for the derivation and tests/test_abi_plan.py for the checks.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

namespace hqr {

constexpr int kChainCap = 13;  // bulges per chain (= the fused step kernel's warps)

struct WindowDesc {     // one diagonal window = one CTA of the chase kernel in one wavefront step
  int32_t chain;        // chain index (global over blocks; 0 = lowest chain of the first block)
  int32_t w0, w1;       // global row/col range [w0, w1] (inclusive)
  int32_t t0, t1;       // chain-local steps [t0, t1] (inclusive) run inside this window
  int32_t b0, nbc;      // bulges of the chain: global bulge indices b0 .. b0+nbc-1
  int32_t slot;         // Q workspace slot
  int32_t last;         // 1 if this is the chain's final window
  int32_t ilo, ihi;     // the active block this window's chain sweeps
  int32_t scan_lo, scan_hi;  // aftermath scan: rows [scan_lo, scan_hi] whose
                        // subdiagonal (and diagonal) entries are final once this window's chase
                        // is done -- set on the windows of each block's last chain (the topmost:
                        // nothing chases above it), scan_hi < scan_lo elsewhere
};

struct Plan {
  int64_t n = 0, ilo = 0, ihi = 0;
  int nb = 0;            // bulges = nshifts/2
  int k = 0;             // effective window side
  int nbc_max = 0;       // bulges per chain (max)
  int s = 0;             // window stride (rows per window)
  int lag = 0;           // steps between chain starts
  int nchains = 0;
  int nsteps = 0;
  int max_kw = 0;        // largest window side actually used
  int max_nbc = 0;
  std::vector<WindowDesc> windows;     // all windows, grouped by step
  std::vector<int32_t> step_begin;     // windows of step g: [step_begin[g], step_begin[g+1])
};

// Plans one active block [ilo, ihi] with nb bulges starting at global bulge b_base and global chain
// c_base; appends each chain's window sequence and start step.  Returns 0 or -9.
struct ChainPlan {
  int g0;                              // global step of the chain's first window
  std::vector<WindowDesc> windows;
};

// nbc_force > 0: use that many bulges per chain for the stride (s = k - 3 nbc_force - 1) -- the
// chains of several sweeps of one block (make_plan_sweeps) must share one stride; g_base: wavefront
// step of the first chain's start in units of lag chains (chain c starts at (g_base + c) lag);
// scan: mark the aftermath rows on the last chain.
inline int plan_block(int64_t n, int64_t ilo, int64_t ihi, int nb, int b_base, int c_base, int window,
                      int kmax, std::vector<ChainPlan>* chains, int* k_out, int* nbc_out, int* s_out,
                      int* lag_out, int nbc_force = 0, int g_base = 0, bool scan = true) {
  // aftermath rows: ilo-1 (the decoupling entry) .. ihi, clipped to rows that have a subdiagonal
  const int32_t scan0 = (int32_t)std::max<int64_t>(ilo - 1, 0), scan1 = (int32_t)std::min<int64_t>(ihi, n - 2);
  const int64_t N = ihi - ilo + 1;
  int64_t k = std::min<int64_t>({(int64_t)window, N, (int64_t)kmax});
  if (k < N && k < 8) return -9;
  *k_out = (int)k;
  if (N <= k) {
    // one window holds the whole active block: a single chain with every bulge
    ChainPlan cp;
    cp.g0 = g_base;
    WindowDesc w{};
    w.chain = c_base; w.w0 = (int32_t)ilo; w.w1 = (int32_t)ihi;
    w.t0 = 0; w.t1 = (int32_t)(N + 3 * (int64_t)nb - 5);  // top bulge's last p = ihi-2
    w.b0 = b_base; w.nbc = nb; w.slot = c_base; w.last = 1;
    w.ilo = (int32_t)ilo; w.ihi = (int32_t)ihi;
    w.scan_lo = scan ? scan0 : 0; w.scan_hi = scan ? scan1 : -1;
    cp.windows.push_back(w);
    chains->push_back(cp);
    *nbc_out = nb; *s_out = (int)N; *lag_out = 1;
    return 0;
  }
  // at most (k-2)/6 bulges fit a window; at most kChainCap so that the fused kernel's
  // chase runs every bulge of a step on its own warp (step.cu).  Fewer bulges per chain cost no
  // flops: the window advances further (s = k - 3*nbc - 1), so the chains have fewer windows.
  const int nbc_cap = std::min((int)((k - 2) / 6), kChainCap);
  const int C = (nb + nbc_cap - 1) / nbc_cap;
  const int base = nb / C, rem = nb % C;                 // remainders on the earliest chains
  const int nbc_max = std::max(base + (rem > 0 ? 1 : 0), nbc_force);
  const int s = (int)(k - 3 * nbc_max - 1);
  const int lag = (int)((k + s - 1) / s);
  *nbc_out = nbc_max; *s_out = s; *lag_out = lag;
  int b = b_base;
  for (int c = 0; c < C; ++c) {
    const int nbc = base + (c < rem ? 1 : 0);
    ChainPlan cp;
    cp.g0 = (g_base + c) * lag;
    for (int i = 0;; ++i) {
      WindowDesc w{};
      w.chain = c_base + c; w.b0 = b; w.nbc = nbc; w.slot = c_base + c;
      w.ilo = (int32_t)ilo; w.ihi = (int32_t)ihi;
      w.scan_lo = 0; w.scan_hi = -1;
      const int64_t w0 = ilo + (int64_t)i * s;
      const int64_t w1 = std::min<int64_t>(w0 + k - 1, ihi);
      w.w0 = (int32_t)w0; w.w1 = (int32_t)w1;
      w.t0 = (i == 0) ? 0 : (int32_t)((int64_t)(i - 1) * s + k - 3);
      if (w1 == ihi) {
        w.t1 = (int32_t)(N + 3 * (int64_t)nbc - 5);
        w.last = 1;
      } else {
        w.t1 = (int32_t)((int64_t)i * s + k - 4);
        w.last = 0;
      }
      if (scan && c == C - 1) {  // the block's last (topmost) chain: rows above the next window are final
        w.scan_lo = (i == 0) ? scan0 : w.w0;
        w.scan_hi = w.last ? scan1 : (int32_t)(w0 + s - 1);
      }
      cp.windows.push_back(w);
      if (w.last) break;
    }
    chains->push_back(cp);
    b += nbc;
  }
  return 0;
}

inline void merge_wavefront(const std::vector<ChainPlan>& chains, Plan* out);

// Builds the plan of one sweep over `nblocks` decoupled active blocks (ascending, disjoint).
// Block i has nshifts[i] shifts; its bulges are numbered after those of blocks 0..i-1.
// k_eff = min(window, N_i, kmax) per block.  Returns 0 or -9.  Other inputs must be valid.
inline int make_plan_multi(int64_t n, int nblocks, const int64_t* ilo, const int64_t* ihi,
                           const int* nshifts, int window, int kmax, Plan* out) {
  Plan P;
  P.n = n; P.ilo = ilo[0]; P.ihi = ihi[nblocks - 1];
  std::vector<ChainPlan> chains;
  int b_base = 0;
  for (int i = 0; i < nblocks; ++i) {
    int k, nbc, s, lag;
    const int nb = nshifts[i] / 2;
    int rc = plan_block(n, ilo[i], ihi[i], nb, b_base, (int)chains.size(), window, kmax, &chains, &k,
                        &nbc, &s, &lag);
    if (rc) return rc;
    if (i == 0) { P.k = k; P.nbc_max = nbc; P.s = s; P.lag = lag; }
    P.k = std::max(P.k, k);
    P.nbc_max = std::max(P.nbc_max, nbc);
    b_base += nb;
  }
  P.nb = b_base;
  merge_wavefront(chains, &P);
  *out = std::move(P);
  return 0;
}

// Several sweeps of one active block with known shift sets, overlapped (
// PAPER.md P:831-833 "two bulge chasing steps can be overlapped", P:706-765 priorities): sweep i
// is nshifts[i]/2 Francis double steps, applied after sweep i-1, so its chains are simply further
// chains of the same wavefront, started lag steps after sweep i-1's last chain -- the tightest
// packing the window geometry allows.  All chains share one stride (the largest bulge
// count per chain over the sweeps), so no chain catches up with the one below it.  The result is
// the sweeps applied one after another (the oracle applies them so); the fused kernel's
// dependency counters order every update exactly as for one sweep.  The aftermath rows are
// scanned by the last sweep's last chain.
inline int make_plan_sweeps(int64_t n, int64_t ilo, int64_t ihi, int nsweeps, const int* nshifts,
                            int window, int kmax, Plan* out) {
  Plan P;
  P.n = n; P.ilo = ilo; P.ihi = ihi;
  const int64_t N = ihi - ilo + 1;
  const int64_t k = std::min<int64_t>({(int64_t)window, N, (int64_t)kmax});
  if (k < N && k < 8) return -9;
  // common bulges-per-chain bound of all sweeps (plan_block's split of each sweep)
  int nbc_force = 0;
  if (N > k) {
    const int cap = std::min((int)((k - 2) / 6), kChainCap);
    for (int i = 0; i < nsweeps; ++i) {
      const int nb = nshifts[i] / 2, C = (nb + cap - 1) / cap;
      nbc_force = std::max(nbc_force, nb / C + (nb % C > 0 ? 1 : 0));
    }
  }
  std::vector<ChainPlan> chains;
  int b_base = 0;
  for (int i = 0; i < nsweeps; ++i) {
    int kk, nbc, s, lag;
    const int c0 = (int)chains.size();
    int rc = plan_block(n, ilo, ihi, nshifts[i] / 2, b_base, c0, window, kmax, &chains, &kk, &nbc, &s,
                        &lag, nbc_force, c0, i == nsweeps - 1);
    if (rc) return rc;
    if (i == 0) { P.k = kk; P.nbc_max = nbc; P.s = s; P.lag = lag; }
    P.nbc_max = std::max(P.nbc_max, nbc);
    b_base += nshifts[i] / 2;
  }
  P.nb = b_base;
  merge_wavefront(chains, &P);
  *out = std::move(P);
  return 0;
}

// wavefront: step g runs window (g - g0) of every chain; windows of a step are disjoint diagonal
// blocks, listed top first (the paper's reverse interleaved insertion order)
inline void merge_wavefront(const std::vector<ChainPlan>& chains, Plan* out) {
  Plan& P = *out;
  P.nchains = (int)chains.size();
  int nsteps = 0;
  for (auto& ch : chains) nsteps = std::max(nsteps, ch.g0 + (int)ch.windows.size());
  P.nsteps = nsteps;
  P.step_begin.push_back(0);
  for (int g = 0; g < nsteps; ++g) {
    const size_t first = P.windows.size();
    for (auto& ch : chains) {
      const int i = g - ch.g0;
      if (i >= 0 && i < (int)ch.windows.size()) P.windows.push_back(ch.windows[i]);
    }
    std::sort(P.windows.begin() + first, P.windows.end(),
              [](const WindowDesc& x, const WindowDesc& y) { return x.w0 < y.w0; });
    for (size_t i = first; i < P.windows.size(); ++i) {
      P.max_kw = std::max(P.max_kw, P.windows[i].w1 - P.windows[i].w0 + 1);
      P.max_nbc = std::max(P.max_nbc, P.windows[i].nbc);
    }
    P.step_begin.push_back((int32_t)P.windows.size());
  }
}

// Single active block.
inline int make_plan(int64_t n, int64_t ilo, int64_t ihi, int nshifts, int window, int kmax,
                     Plan* out) {
  return make_plan_multi(n, 1, &ilo, &ihi, &nshifts, window, kmax, out);
}

}  // namespace hqr
