// bfgs_plan.h -- host-side sizing of the warp-per-start BFGS kernel (shared
// by bfgs.cu and the user-objective plug-in launcher plugin.cu).
#pragma once
#include <algorithm>

#include "bfgs_common.cuh"

namespace zeus {

// ---- sizing --------------------------------------------------------------
constexpr size_t kSmemLimit = 227 * 1024;
constexpr size_t kWsHeader = 256;

struct BfgsPlan {
  int wpb;       // warps per block
  int dr;        // register-resident H rows (0: smem / global)
  bool smem_h;   // (dr == 0) H in shared memory
  int ldh, tstride, bmax, nalpha;
  size_t warp_doubles;
  size_t smem;
};

inline int even(int v) { return (v + 1) & ~1; }

inline BfgsPlan bfgs_plan(int d, int nacc, int nterms, int iter_ls, int kt = 2) {
  BfgsPlan P{};
  P.dr = d <= 12 ? 12 : d <= 16 ? 16 : d <= 32 ? 32 : 0;
  P.tstride = std::max(1, nterms) | 1;
  // sizes depend on d only (never on iter_ls), so the workspace query and the
  // launch always agree on where H lives
  (void)iter_ls;
  P.bmax = std::max(1, std::min(32, kTermCap / std::max(1, nterms)));
  P.nalpha = kAlphaTable;
  P.ldh = d;  // lanes read consecutive columns: conflict-free for any ld
  // term buffer rows: NACC * kWarpTrialRows rows of tstride, + 32 alpha scratch
  const size_t vec = (size_t)4 * std::max(d, P.dr) + 5 * (size_t)d +
                     (size_t)(nacc + kt) * P.bmax * P.tstride + 32;  // + KT tangent rows
  size_t per_warp = even((int)vec);
  if (P.dr == 0) {
    const size_t with_h = per_warp + hsize(d, P.ldh);
    const int wpb = (int)std::min<size_t>(kBfgsWarps,
                                          (kSmemLimit - P.nalpha * 8) / (with_h * 8));
    if (wpb >= 1) {
      P.smem_h = true;
      P.wpb = wpb;
      per_warp = with_h;
    } else {
      P.smem_h = false;
      P.wpb = kBfgsWarps;
    }
  } else {
    P.smem_h = false;
    P.wpb = kBfgsWarps;
  }
  P.warp_doubles = per_warp;
  P.smem = (P.nalpha + per_warp * P.wpb) * sizeof(double);
  return P;
}

}  // namespace zeus
