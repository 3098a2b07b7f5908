// pa_dfma.cuh — contraction stages of the fused PA apply, register-blocked
// FP64-FMA ("line") variant.  Plugs into pa_pipe.cuh.
//
//   stage A  contract x: thread per line (j,k): B x, G x       (tensor.py:177-210)
//   stage B  contract y: thread per line (k,a): 3 component chains
//   stage C  contract z, apply D (6-comp symmetric, BP3; w|J| BP1),
//            transposed z — all in registers for line (a,b)
//   stage D  transposed y: thread per line (a,k)
//   stage E  transposed x: thread per line (j,k) + atomic scatter-add
//            (Restriction.scatter_add, feklab/mesh.py:133-137)
//
// MFEM-style stage sharing: BP3 costs 2(4qd^3+6q^2d^2+6q^3d)+15q^3 flops per
// element instead of the reference's three independent chains
// (apply_gradient_3d, tensor.py:244-260).  Each thread keeps NL lines in
// registers; one 8-byte shared load of a line value feeds q (2q, 3q) FMAs and
// one basis-table load feeds NL lines.
//
// Basis tables (measured): sm_100a ptxas feeds double
// constants to DFMA through uniform registers (LDCU + UR operand).  With the
// 2qd table entries loop-invariant it hoists them out of the persistent loop,
// overflows the 63-entry uniform register file and spills through vector
// registers (R2UR / MOV.SPILL: ~1000 of 2000 warp instructions per element);
// reading rows from shared memory instead costs LDS wavefronts the kernel
// does not have.  The kernel parameter therefore carries TWO copies of the
// tables and batch `it` reads copy it&1: the loads stay loop-variant, so each
// row is fetched (LDCU.128, 2 entries) right where it is used and shared by
// the NL lines of the thread.
#pragma once

#include "pa_common.cuh"

namespace fk {

template <int D, int Q>
struct __align__(16) RowTables {
  static constexpr int DP = D + (D & 1), QP = Q + (Q & 1);  // 16-byte row pitch
  static constexpr int TB = 0, TG = Q * DP, TBT = 2 * Q * DP, TGT = 2 * Q * DP + D * QP;
  static constexpr int SZ = 2 * Q * DP + 2 * D * QP;
  double t[2][SZ];  // two copies of: B[a][i], G[a][i] rows; Bt[i][a], Gt[i][a] rows
};

// Run f(t0) over the stage's lines t0 = threadIdx.x + k*STEP < n.  When every
// line fits in one pass (LMAX <= STEP, the configured geometries) there is no
// loop at all, so nothing invites ptxas to hoist basis-table loads into
// vector registers (and shuttle them back with R2UR for every DFMA).
template <int STEP, int LMAX, typename F>
__device__ __forceinline__ void lines_loop(int n, F f) {
  if constexpr (LMAX <= STEP) {
    if ((int)threadIdx.x < n) f((int)threadIdx.x);
  } else {
    for (int t0 = threadIdx.x; t0 < n; t0 += STEP) f(t0);
  }
}

template <int N>
__device__ __forceinline__ void ld_row(const double* __restrict__ p, double (&r)[N]) {
#pragma unroll
  for (int i = 0; i + 1 < N; i += 2) {
    const double2 v = *reinterpret_cast<const double2*>(p + i);
    r[i] = v.x;
    r[i + 1] = v.y;
  }
  if constexpr (N & 1) r[N - 1] = p[N - 1];
}

template <int D, int Q, int NC, int E_, int T_, int NL_>
struct DfmaBody {
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  using Tab = RowTables<D, Q>;
  static constexpr int LS = L::LS, LQ = L::LQ, P0 = L::P0, P1 = L::P1, Q3 = L::Q3;
  static constexpr bool IP = false;  // W written to the T1/W region (not in place)
  static constexpr int XS = D * D * LS;
  static constexpr int DP = Tab::DP, QP = Tab::QP;
  static constexpr int E = E_, T = T_, EXTRA = 0;
  static constexpr int NL = NL_;                                        // lines per thread
  static constexpr int NLC = (NC == 3 && 6 * D * NL_ > 60) ? 1 : NL_;  // stage C (register-heavy)

  static void fill(Tab& tb, const double* B, const double* Gr) {
    for (int c = 0; c < 2; ++c)
      for (int a = 0; a < Q; ++a)
        for (int i = 0; i < D; ++i) {
          tb.t[c][Tab::TB + a * DP + i] = B[a * D + i];
          tb.t[c][Tab::TG + a * DP + i] = Gr[a * D + i];
          tb.t[c][Tab::TBT + i * QP + a] = B[a * D + i];
          tb.t[c][Tab::TGT + i * QP + a] = Gr[a * D + i];
        }
  }

  __device__ static void init(const Tab&, double*) {}

  // X [v=(j,k)][i] -> T1 [s][a][k][j]
  __device__ __forceinline__ static void stage_a(const Tab& tb, int it, const double* xb,
                                                 double* s1, int ne, double*) {
    const double* tab = tb.t[it & 1];
    const int n = ne * D * D;
    lines_loop<NL * T, E * D * D>(n, [&](int t0) {
      double xr[NL][D];
      double* o[NL];
      bool ok[NL];
#pragma unroll
      for (int h = 0; h < NL; ++h) {
        const int t = t0 + h * T;
        ok[h] = t < n;
        const int tt = ok[h] ? t : t0;
        const int e = tt / (D * D), v = tt - e * (D * D);
        const double* in = xb + e * XS + v * LS;
#pragma unroll
        for (int i = 0; i < D; ++i) xr[h][i] = in[i];
        o[h] = s1 + e * P1 + (v / D) * LS + (v % D);
      }
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        double br[D];
        ld_row(tab + Tab::TB + a * DP, br);
#pragma unroll
        for (int h = 0; h < NL; ++h) {
          double bx = br[0] * xr[h][0];
#pragma unroll
          for (int i = 1; i < D; ++i) bx = fma(br[i], xr[h][i], bx);
          if (ok[h]) o[h][a * D * LS] = bx;
        }
        if constexpr (NC == 3) {
          double gr[D];
          ld_row(tab + Tab::TG + a * DP, gr);
#pragma unroll
          for (int h = 0; h < NL; ++h) {
            double gx = gr[0] * xr[h][0];
#pragma unroll
            for (int i = 1; i < D; ++i) gx = fma(gr[i], xr[h][i], gx);
            if (ok[h]) o[h][Q * D * LS + a * D * LS] = gx;
          }
        }
      }
    });
  }

  // T1 [s][a][k][j] (line u = k + D a) -> T2 [s][b][a][k]
  __device__ __forceinline__ static void stage_b(const Tab& tb, int it, const double* s1, double* s0,
                                                 int ne, double*) {
    const double* tab = tb.t[it & 1];
    const int n = ne * D * Q;
    lines_loop<NL * T, E * D * Q>(n, [&](int t0) {
      double bx[NL][D], gx[NL][D];
      double* o[NL];
      bool ok[NL];
#pragma unroll
      for (int h = 0; h < NL; ++h) {
        const int t = t0 + h * T;
        ok[h] = t < n;
        const int tt = ok[h] ? t : t0;
        const int e = tt / (D * Q), u = tt - e * (D * Q);
        const double* in = s1 + e * P1 + u * LS;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          bx[h][j] = in[j];
          if constexpr (NC == 3) gx[h][j] = in[Q * D * LS + j];
        }
        o[h] = s0 + e * P0 + (u / D) * LS + (u % D);
      }
#pragma unroll
      for (int b = 0; b < Q; ++b) {
        double br[D];
        ld_row(tab + Tab::TB + b * DP, br);
        if constexpr (NC == 3) {
          double gr[D];
          ld_row(tab + Tab::TG + b * DP, gr);
#pragma unroll
          for (int h = 0; h < NL; ++h) {
            double c0 = br[0] * gx[h][0];
            double c1 = gr[0] * bx[h][0];
            double c2 = br[0] * bx[h][0];
#pragma unroll
            for (int j = 1; j < D; ++j) {
              c0 = fma(br[j], gx[h][j], c0);
              c1 = fma(gr[j], bx[h][j], c1);
              c2 = fma(br[j], bx[h][j], c2);
            }
            if (ok[h]) {
              o[h][b * Q * LS] = c0;
              o[h][Q * Q * LS + b * Q * LS] = c1;
              o[h][2 * Q * Q * LS + b * Q * LS] = c2;
            }
          }
        } else {
#pragma unroll
          for (int h = 0; h < NL; ++h) {
            double c = br[0] * bx[h][0];
#pragma unroll
            for (int j = 1; j < D; ++j) c = fma(br[j], bx[h][j], c);
            if (ok[h]) o[h][b * Q * LS] = c;
          }
        }
      }
    });
  }

  // T2 [s][b][a][k] (line r = a + Q b) + D -> W [s][k][a][b]
  __device__ __forceinline__ static void stage_c(const Tab& tb, int it, const double* s0,
                                                 const double* db, double* s1, int ne, double*) {
    const double* tab = tb.t[it & 1];
    const int n = ne * Q * Q;
    constexpr int NS = NC;
    lines_loop<NLC * T, E * Q * Q>(n, [&](int t0) {
      double tin[NLC][NS][D], w[NLC][NS][D];
      const double* pe[NLC];
      double* o[NLC];
      bool ok[NLC];
#pragma unroll
      for (int h = 0; h < NLC; ++h) {
        const int t = t0 + h * T;
        ok[h] = t < n;
        const int tt = ok[h] ? t : t0;
        const int e = tt / (Q * Q), r = tt - e * (Q * Q);
        const double* in = s0 + e * P0 + r * LS;
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int k = 0; k < D; ++k) {
            tin[h][s][k] = in[s * Q * Q * LS + k];
            w[h][s][k] = 0.0;
          }
        pe[h] = db + e * G::PS + r;
        o[h] = s1 + e * P1 + (r % Q) * LQ + (r / Q);
      }
#pragma unroll
      for (int c = 0; c < Q; ++c) {
        double br[D], gr[D];
        ld_row(tab + Tab::TB + c * DP, br);
        if constexpr (NC == 3) ld_row(tab + Tab::TG + c * DP, gr);
#pragma unroll
        for (int h = 0; h < NLC; ++h) {
          const double* pc = pe[h] + c * Q * Q;
          if constexpr (NC == 3) {
            double g0 = br[0] * tin[h][0][0];
            double g1 = br[0] * tin[h][1][0];
            double g2 = gr[0] * tin[h][2][0];
#pragma unroll
            for (int k = 1; k < D; ++k) {
              g0 = fma(br[k], tin[h][0][k], g0);
              g1 = fma(br[k], tin[h][1][k], g1);
              g2 = fma(gr[k], tin[h][2][k], g2);
            }
            const double d00 = pc[0 * Q3], d01 = pc[1 * Q3], d02 = pc[2 * Q3];
            const double d11 = pc[3 * Q3], d12 = pc[4 * Q3], d22 = pc[5 * Q3];
            const double o0 = fma(d02, g2, fma(d01, g1, d00 * g0));
            const double o1 = fma(d12, g2, fma(d11, g1, d01 * g0));
            const double o2 = fma(d22, g2, fma(d12, g1, d02 * g0));
#pragma unroll
            for (int k = 0; k < D; ++k) {
              w[h][0][k] = fma(br[k], o0, w[h][0][k]);
              w[h][1][k] = fma(br[k], o1, w[h][1][k]);
              w[h][2][k] = fma(gr[k], o2, w[h][2][k]);
            }
          } else {
            double g = br[0] * tin[h][0][0];
#pragma unroll
            for (int k = 1; k < D; ++k) g = fma(br[k], tin[h][0][k], g);
            const double oo = pc[0] * g;
#pragma unroll
            for (int k = 0; k < D; ++k) w[h][0][k] = fma(br[k], oo, w[h][0][k]);
          }
        }
      }
#pragma unroll
      for (int h = 0; h < NLC; ++h) {
        if (!ok[h]) continue;
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int k = 0; k < D; ++k) o[h][s * D * Q * LQ + k * Q * LQ] = w[h][s][k];
      }
    });
  }

  // W [s][k][a][b] (line u = a + Q k) -> R [s][k][j][a]
  __device__ __forceinline__ static void stage_d(const Tab& tb, int it, const double* s1, double* s0,
                                                 int ne, double*) {
    const double* tab = tb.t[it & 1];
    const int n = ne * Q * D;
    lines_loop<NL * T, E * Q * D>(n, [&](int t0) {
      double w[NL][NC][Q];
      double* o[NL];
      bool ok[NL];
#pragma unroll
      for (int h = 0; h < NL; ++h) {
        const int t = t0 + h * T;
        ok[h] = t < n;
        const int tt = ok[h] ? t : t0;
        const int e = tt / (Q * D), u = tt - e * (Q * D);
        const double* in = s1 + e * P1 + u * LQ;
#pragma unroll
        for (int s = 0; s < NC; ++s)
#pragma unroll
          for (int b = 0; b < Q; ++b) w[h][s][b] = in[s * D * Q * LQ + b];
        o[h] = s0 + e * P0 + (u / Q) * D * LQ + (u % Q);
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double bt[Q];
        ld_row(tab + Tab::TBT + j * QP, bt);
        if constexpr (NC == 3) {
          double gt[Q];
          ld_row(tab + Tab::TGT + j * QP, gt);
#pragma unroll
          for (int h = 0; h < NL; ++h) {
            double rg = bt[0] * w[h][0][0];
            double rb = gt[0] * w[h][1][0];
#pragma unroll
            for (int b = 1; b < Q; ++b) {
              rg = fma(bt[b], w[h][0][b], rg);
              rb = fma(gt[b], w[h][1][b], rb);
            }
#pragma unroll
            for (int b = 0; b < Q; ++b) rb = fma(bt[b], w[h][2][b], rb);
            if (ok[h]) {
              o[h][j * LQ] = rg;
              o[h][D * D * LQ + j * LQ] = rb;
            }
          }
        } else {
#pragma unroll
          for (int h = 0; h < NL; ++h) {
            double rr = bt[0] * w[h][0][0];
#pragma unroll
            for (int b = 1; b < Q; ++b) rr = fma(bt[b], w[h][0][b], rr);
            if (ok[h]) o[h][j * LQ] = rr;
          }
        }
      }
    });
  }

  // R [s][k][j][a] (line v = j + D k) -> y (atomic scatter-add)
  __device__ __forceinline__ static void stage_e(const Tab& tb, int it, const double* s0,
                                                 const int* gslot, double* y, int ne, double*) {
    const double* tab = tb.t[it & 1];
    constexpr int NR = (NC == 3) ? 2 : 1;
    const int n = ne * D * D;
    lines_loop<NL * T, E * D * D>(n, [&](int t0) {
      double rv[NL][NR][Q];
      const int* g[NL];
      bool ok[NL];
#pragma unroll
      for (int h = 0; h < NL; ++h) {
        const int t = t0 + h * T;
        ok[h] = t < n;
        const int tt = ok[h] ? t : t0;
        const int e = tt / (D * D), v = tt - e * (D * D);
        const double* in = s0 + e * P0 + v * LQ;
#pragma unroll
        for (int s = 0; s < NR; ++s)
#pragma unroll
          for (int a = 0; a < Q; ++a) rv[h][s][a] = in[s * D * D * LQ + a];
        g[h] = gslot + e * G::GS + v * D;
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double bt[Q];
        ld_row(tab + Tab::TBT + i * QP, bt);
        if constexpr (NC == 3) {
          double gt[Q];
          ld_row(tab + Tab::TGT + i * QP, gt);
#pragma unroll
          for (int h = 0; h < NL; ++h) {
            double acc = gt[0] * rv[h][0][0];
#pragma unroll
            for (int a = 1; a < Q; ++a) acc = fma(gt[a], rv[h][0][a], acc);
#pragma unroll
            for (int a = 0; a < Q; ++a) acc = fma(bt[a], rv[h][1][a], acc);
            if (ok[h]) atomicAdd(y + g[h][i], acc);
          }
        } else {
#pragma unroll
          for (int h = 0; h < NL; ++h) {
            double acc = bt[0] * rv[h][0][0];
#pragma unroll
            for (int a = 1; a < Q; ++a) acc = fma(bt[a], rv[h][0][a], acc);
            if (ok[h]) atomicAdd(y + g[h][i], acc);
          }
        }
      }
    });
  }
};

}  // namespace fk
