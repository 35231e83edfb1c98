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
// See DESIGN.md "Planner" for the derivation and tests/test_plan.py for the checks.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

namespace hqr {

struct WindowDesc {     // one diagonal window = one CTA of the chase kernel in one wavefront step
  int32_t chain;        // chain index (0 = lowest / first shifts)
  int32_t w0, w1;       // global row/col range [w0, w1] (inclusive)
  int32_t t0, t1;       // chain-local steps [t0, t1] (inclusive) run inside this window
  int32_t b0, nbc;      // bulges of the chain: global bulge indices b0 .. b0+nbc-1
  int32_t slot;         // Q workspace slot
  int32_t last;         // 1 if this is the chain's final window
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

// Builds the plan.  k_eff = min(window, N, kmax).  Returns 0 or a negative code (-9: window
// too small for a multi-window chain).  Inputs are assumed already validated otherwise.
inline int make_plan(int64_t n, int64_t ilo, int64_t ihi, int nshifts, int window, int kmax,
                     Plan* out) {
  Plan P;
  P.n = n; P.ilo = ilo; P.ihi = ihi;
  P.nb = nshifts / 2;
  const int64_t N = ihi - ilo + 1;
  int64_t k = std::min<int64_t>({(int64_t)window, N, (int64_t)kmax});
  if (k < N && k < 8) return -9;
  P.k = (int)k;

  struct ChainInfo { int b0, nbc, g0, nwin; };
  std::vector<ChainInfo> chains;
  std::vector<std::vector<WindowDesc>> chain_windows;

  if (N <= k) {
    // one window holds the whole active block: a single chain with every bulge
    P.nbc_max = P.nb; P.s = (int)N; P.lag = 1; P.nchains = 1;
    WindowDesc w{};
    w.chain = 0; w.w0 = (int32_t)ilo; w.w1 = (int32_t)ihi;
    w.t0 = 0; w.t1 = (int32_t)(N + 3 * (int64_t)P.nb - 5);  // top bulge's last p = ihi-2
    w.b0 = 0; w.nbc = P.nb; w.slot = 0; w.last = 1;
    chain_windows.push_back({w});
    chains.push_back({0, P.nb, 0, 1});
  } else {
    int nbc_cap = (int)((k - 2) / 6);
    int C = (P.nb + nbc_cap - 1) / nbc_cap;
    int base = P.nb / C, rem = P.nb % C;                 // remainders on the earliest chains
    int nbc_max = base + (rem > 0 ? 1 : 0);
    P.nbc_max = nbc_max;
    P.s = (int)(k - 3 * nbc_max - 1);
    P.lag = (int)((k + P.s - 1) / P.s);
    P.nchains = C;
    int b = 0;
    for (int c = 0; c < C; ++c) {
      int nbc = base + (c < rem ? 1 : 0);
      std::vector<WindowDesc> ws;
      for (int i = 0;; ++i) {
        WindowDesc w{};
        w.chain = c; w.b0 = b; w.nbc = nbc;
        int64_t w0 = ilo + (int64_t)i * P.s;
        int64_t w1 = std::min<int64_t>(w0 + k - 1, ihi);
        w.w0 = (int32_t)w0; w.w1 = (int32_t)w1;
        w.t0 = (i == 0) ? 0 : (int32_t)((int64_t)(i - 1) * P.s + k - 3);
        if (w1 == ihi) {
          w.t1 = (int32_t)(N + 3 * (int64_t)nbc - 5);
          w.last = 1;
        } else {
          w.t1 = (int32_t)((int64_t)i * P.s + k - 4);
          w.last = 0;
        }
        w.slot = c;
        ws.push_back(w);
        if (w.last) break;
      }
      chains.push_back({b, nbc, c * P.lag, (int)ws.size()});
      chain_windows.push_back(ws);
      b += nbc;
    }
  }
  // wavefront: step g runs window (g - g0_c) of every chain with 0 <= g - g0_c < nwin_c.
  // Within a step, windows are listed top chain first (highest c) -- the paper's reverse
  // interleaved insertion order -- which is also ascending row order.
  int nsteps = 0;
  for (auto& ch : chains) nsteps = std::max(nsteps, ch.g0 + ch.nwin);
  P.nsteps = nsteps;
  P.step_begin.push_back(0);
  for (int g = 0; g < nsteps; ++g) {
    for (int c = (int)chains.size() - 1; c >= 0; --c) {
      int i = g - chains[c].g0;
      if (i >= 0 && i < chains[c].nwin) {
        WindowDesc w = chain_windows[c][i];
        P.windows.push_back(w);
        P.max_kw = std::max(P.max_kw, w.w1 - w.w0 + 1);
        P.max_nbc = std::max(P.max_nbc, w.nbc);
      }
    }
    P.step_begin.push_back((int32_t)P.windows.size());
  }
  *out = std::move(P);
  return 0;
}

}  // namespace hqr
