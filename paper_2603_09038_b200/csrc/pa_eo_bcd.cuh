// pa_eo_bcd.cuh — BP1 even-odd body with stages B, C and D fused in
// registers (EO cfgs 50-53; pa_pipe.cuh runs stage_bcd between stage A and
// stage E when the body has FUSED_BCD).
//
// After the staged scatter the BP1 kernel is bound by the
// L1 LSU data pipe, almost all of it shared-memory wavefronts at ncu's ideal:
// every contraction stage round-trips its output through shared memory.  Here
// one thread owns an (element, a) slab and keeps it in registers through
//   B  y:   T2[b][k]  = sum_j B[b][j] T1[a][j][k]          (d lines of d -> q)
//   C  z:   g[c]      = sum_k B[c][k] T2[b][k], g *= D(a,b,c),
//           W[b][k']  = sum_c B[c][k'] g[c]                 (q lines, in place)
//   D  y^T: R[a][j'][k'] = sum_b B[b][j'] W[b][k']          (d lines of q -> d)
// reading its T1 plane (d^2 values) from shared memory and writing R over the
// same plane (only this thread touches it): the T2 and W round trips and two
// CTA barriers per batch go away.  Same sums as the line bodies (even-odd
// folded, tensor.py:220-241 up to FP64 rounding).
//
// Layouts (EoBcdLay): T1 = R at e*SE + a + QP (j + d k), QP = q|1 — stage A's
// lines (e, j, k) write a fixed a with odd stride QP, the fused threads
// (e, a) read a fixed (j, k) at e*SE + a with SE = q (mod 16): both
// conflict-free.  Region 0 only holds the staged scatter's output (X layout).
#pragma once

#include "pa_dfma_eo.cuh"

namespace fk {

template <int D, int Q, int E>
struct EoBcdLay {
  static constexpr bool W_OVER_T2 = true;  // R lives in region 1 (sr = s1), sw = region 0
  static constexpr bool NO_C = true;       // the line stages B-D never run
  static constexpr int MG = 0, MA = 0, MB = 0, MC = 0, MD = 0, ME = 0;
  static constexpr int LS = D | 1, QP = Q | 1;
  static constexpr int XS = D * D * LS;
  // smallest SE >= plane extent with SE = Q (mod 16)
  static constexpr int EXT = (Q - 1) + QP * (D * D - 1) + 1;
  static constexpr int SE = EXT + (((Q - EXT) % 16) + 16) % 16;
  using X = BufLay<XS, 0, 1, LS, D * LS>;
  using T1 = BufLay<SE, 0, 1, QP, QP * D>;
  using R = T1;
  using T2 = BufLay<XS, 0, 0, 0, 0>;  // unused (region 0 = staged scatter output)
  using W = T2;
};

template <int D, int Q, int E_, int T_>
struct EoBcdBody : DfmaEoBody<D, Q, 1, E_, T_, EoBcdLay<D, Q, E_>, false, true> {
  using Base = DfmaEoBody<D, Q, 1, E_, T_, EoBcdLay<D, Q, E_>, false, true>;
  using Tab = typename Base::Tab;
  using G = GlobalLayout<D, Q, 1>;
  using LY = EoBcdLay<D, Q, E_>;
  static constexpr int E = E_, T = T_;
  static constexpr bool FUSED_BCD = true;
  static constexpr bool QF_OK = false;
  static_assert(Base::YS_FITS, "staged scatter output must fit in region 0");

  __device__ __forceinline__ static void stage_bcd(const Tab& tb, double* s1, const double* db, int ne) {
    const double* tab = tb.t[0];
    constexpr int N = E * Q;
    for (int t = threadIdx.x; t < N; t += T) {
      const int e = t / Q, a = t - e * Q;
      if (e >= ne) continue;
      double* pl = s1 + e * LY::SE + a;  // T1(a, j, k) / R(a, j, k) at pl[QP (j + d k)]
      double t2[D][Q];                   // [k][b]: T2, then W in place
#pragma unroll
      for (int k = 0; k < D; ++k) {
        double xr[D];
#pragma unroll
        for (int j = 0; j < D; ++j) xr[j] = pl[LY::QP * (j + D * k)];
        contract_eo<D, Q, +1>(tab + Tab::TB, xr, t2[k]);
      }
      const double* pd = db + e * G::PS + a;
#pragma unroll
      for (int b = 0; b < Q; ++b) {
        double tin[D], g[Q], w[D];
#pragma unroll
        for (int k = 0; k < D; ++k) tin[k] = t2[k][b];
        contract_eo<D, Q, +1>(tab + Tab::TB, tin, g);
#pragma unroll
        for (int c = 0; c < Q; ++c) g[c] *= pd[Q * (b + Q * c)];
        contract_eo<Q, D, +1>(tab + Tab::TBT, g, w);
#pragma unroll
        for (int k = 0; k < D; ++k) t2[k][b] = w[k];
      }
#pragma unroll
      for (int k = 0; k < D; ++k) {
        double r[D];
        contract_eo<Q, D, +1>(tab + Tab::TBT, t2[k], r);
#pragma unroll
        for (int j = 0; j < D; ++j) pl[LY::QP * (j + D * k)] = r[j];
      }
    }
  }
};

}  // namespace fk
