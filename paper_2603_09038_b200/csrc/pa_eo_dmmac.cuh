// pa_eo_dmmac.cuh — hybrid body (variant dmma, cfgs 12-13): the even-odd FMA
// stages A, B, D, E of pa_dfma_eo.cuh with stage C (z-contraction, D,
// transposed z — the largest stage, three components) on the FP64 tensor
// cores.
//
// Stage C rows are the (element, a, b) lines of the batch (q^2 per element:
// whole 8-row tiles at q = 8), K = k (d <= 8 -> one or two k-steps), N = c
// (q <= 8): DMMA.8x8x4 with the basis fragments in registers; D is applied
// on the accumulators; the accumulators are re-laid out as A fragments of
// the transposed z contraction by two shuffles per k-step (rows kept, K = c)
// and W is stored from the C fragments.  T2 / W keep the searched EO layouts
// of the geometry (not in place: W must not overwrite T2 lines other warps
// still read).  p <= 6 with q = p + 2 (d, q <= 8).
#pragma once

#include "pa_dfma_eo.cuh"
#include "pa_dmma.cuh"
#include "pa_dmma_warp.cuh"

namespace fk {

template <int D, int Q, int NC, int E_, int T_, class LP, bool PP = true, bool SR = true>
struct EoDmmaCBody : DfmaEoBody<D, Q, NC, E_, T_, LP, PP, SR> {
  using Base = DfmaEoBody<D, Q, NC, E_, T_, LP, PP, SR>;
  using G = GlobalLayout<D, Q, NC>;
  using LT2 = typename LP::T2;
  using LW = typename LP::W;
  static_assert(!LP::W_OVER_T2, "DMMA stage C writes W beside T2");
  static_assert(D <= 8 && Q <= 8, "one 8-wide tile per line");
  static constexpr bool QF_OK = false;  // no quadratic-form twin
  static constexpr int T = T_, NW = T_ / 32, KD = (D + 3) / 4, KQ = (Q + 3) / 4;
  static constexpr int Q3 = Q * Q * Q;
  // the folded tables of the FMA stages plus the raw ones for the fragments
  struct Tab : Base::Tab {
    double rB[Q * D], rG[Q * D];
  };
  static void fill(Tab& tb, const double* B, const double* Gr) {
    Base::fill(tb, B, Gr);
    for (int n = 0; n < Q * D; ++n) {
      tb.rB[n] = B[n];
      tb.rG[n] = Gr[n];
    }
  }

  template <bool MF = false>
  __device__ __forceinline__ static void stage_c(const Tab& tb, int, const double* s0, const double* db,
                                                 double* sw, int ne, double*) {
    static_assert(!MF, "matrix-free runs the FMA body");
    const int L = threadIdx.x & 31, warp = threadIdx.x >> 5, r4 = L >> 2, c4 = L & 3;
    const int rows = ne * Q * Q;
    if (warp * 8 >= rows) return;
    double fB[KD], fG[KD], tB[KQ], tG[KQ];
#pragma unroll
    for (int ks = 0; ks < KD; ++ks) {  // forward: Bop(k, c) = T[c][k]
      const int k = 4 * ks + c4, n = r4;
      const bool ok = k < D && n < Q;
      fB[ks] = ok ? tb.rB[n * D + k] : 0.0;
      fG[ks] = ok ? tb.rG[n * D + k] : 0.0;
    }
#pragma unroll
    for (int ks = 0; ks < KQ; ++ks) {  // transposed: Bop(c, k') = T[c][k']
      const int c = 4 * ks + c4, n = r4;
      const bool ok = c < Q && n < D;
      tB[ks] = ok ? tb.rB[c * D + n] : 0.0;
      tG[ks] = ok ? tb.rG[c * D + n] : 0.0;
    }
    for (int m0 = warp * 8; m0 < rows; m0 += NW * 8) {
      const int m = m0 + r4;
      const int mm = m < rows ? m : rows - 1;
      const int e = mm / (Q * Q), ab = mm - e * (Q * Q), a = ab % Q, b = ab / Q;
      double g[NC][2];
#pragma unroll
      for (int s = 0; s < NC; ++s) g[s][0] = g[s][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KD; ++ks) {
        const int kk = 4 * ks + c4;
#pragma unroll
        for (int s = 0; s < NC; ++s) {
          const double av = kk < D ? s0[LT2::at(e, s, a, b, kk)] : 0.0;
          dmma884(g[s][0], g[s][1], av, (NC == 3 && s == 2) ? fG[ks] : fB[ks]);
        }
      }
      // D at qp = a + Q (b + Q c), c = 2 c4 + h (rows beyond the batch are dropped)
      const double* pe = db + e * G::PS + a + Q * b;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 2 * c4 + h;
        if (c < Q) {
          const double* pc = pe + c * Q * Q;
          if constexpr (NC == 3) {
            const double g0 = g[0][h], g1 = g[1][h], g2 = g[2][h];
            const double d00 = pc[0], d01 = pc[Q3], d02 = pc[2 * Q3];
            const double d11 = pc[3 * Q3], d12 = pc[4 * Q3], d22 = pc[5 * Q3];
            g[0][h] = fma(d02, g2, fma(d01, g1, d00 * g0));
            g[1][h] = fma(d12, g2, fma(d11, g1, d01 * g0));
            g[2][h] = fma(d22, g2, fma(d12, g1, d02 * g0));
          } else {
            g[0][h] *= pc[0];
          }
        }
      }
      double w[NC][2];
#pragma unroll
      for (int s = 0; s < NC; ++s) w[s][0] = w[s][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KQ; ++ks)
#pragma unroll
        for (int s = 0; s < NC; ++s) {
          const double av = frag_same(g[s][0], g[s][1], ks);
          dmma884(w[s][0], w[s][1], av, (NC == 3 && s == 2) ? tG[ks] : tB[ks]);
        }
      if (m < rows) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kp = 2 * c4 + h;
          if (kp < D) {
#pragma unroll
            for (int s = 0; s < NC; ++s) sw[LW::at(e, s, a, b, kp)] = w[s][h];
          }
        }
      }
    }
  }
};

}  // namespace fk
