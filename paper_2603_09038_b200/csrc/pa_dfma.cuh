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
// (apply_gradient_3d, tensor.py:244-260).  Each thread keeps its line in
// registers; one 8-byte shared load of the line feeds q (or 2q, 3q) FMAs.
//
// Basis tables: sm_100a ptxas turns every double kernel-parameter operand
// into LDCU + uniform-register traffic and, when it hoists the 2qd table
// entries out of the persistent loop, spills the uniform register file
// (measured: ~1000 of 2000 warp instructions per element were R2UR / IMAD /
// LDCU moves).  The tables therefore live in shared memory as 16-byte-aligned
// rows (B[a][*], G[a][*] and the transposes) and each row is read with
// LDS.128 broadcasts right where it is used (__syncthreads between stages
// keeps the compiler from hoisting them): 0.5 load per table entry, no
// register pressure from the tables.
#pragma once

#include "pa_common.cuh"

namespace fk {

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

template <int D, int Q, int NC, int E_, int T_>
struct DfmaBody {
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  static constexpr int LS = L::LS, LQ = L::LQ, P0 = L::P0, P1 = L::P1, Q3 = L::Q3;
  static constexpr int XS = D * D * LS;
  static constexpr int DP = D + (D & 1), QP = Q + (Q & 1);  // 16-byte row pitch
  // smem table offsets (doubles): B[a][i], G[a][i] rows of D; Bt[i][a], Gt[i][a] rows of Q
  static constexpr int TB = 0, TG = TB + Q * DP, TBT = TG + Q * DP, TGT = TBT + D * QP;
  static constexpr int E = E_, T = T_, EXTRA = TGT + D * QP;

  __device__ static void init(const Tables<D, Q>& tb, double* t) {
    for (int n = threadIdx.x; n < Q * D; n += T) {
      const int a = n / D, i = n % D;
      t[TB + a * DP + i] = tb.B[n];
      t[TG + a * DP + i] = tb.G[n];
      t[TBT + i * QP + a] = tb.B[n];
      t[TGT + i * QP + a] = tb.G[n];
    }
  }

  // X [v=(j,k)][i] -> T1 [s][a][k][j]
  __device__ __forceinline__ static void stage_a(const Tables<D, Q>&, const double* xb, double* s1,
                                                 int ne, const double* tab) {
    for (int t = threadIdx.x; t < ne * D * D; t += T) {
      const int e = t / (D * D), v = t - e * (D * D);
      const double* in = xb + e * XS + v * LS;
      double xr[D];
#pragma unroll
      for (int i = 0; i < D; ++i) xr[i] = in[i];
      double* o = s1 + e * P1 + (v / D) * LS + (v % D);
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        double br[D];
        ld_row(tab + TB + a * DP, br);
        double bx = br[0] * xr[0];
#pragma unroll
        for (int i = 1; i < D; ++i) bx = fma(br[i], xr[i], bx);
        o[a * D * LS] = bx;
        if constexpr (NC == 3) {
          double gr[D];
          ld_row(tab + TG + a * DP, gr);
          double gx = gr[0] * xr[0];
#pragma unroll
          for (int i = 1; i < D; ++i) gx = fma(gr[i], xr[i], gx);
          o[Q * D * LS + a * D * LS] = gx;
        }
      }
    }
  }

  // T1 [s][a][k][j] (line u = k + D a) -> T2 [s][b][a][k]
  __device__ __forceinline__ static void stage_b(const Tables<D, Q>&, const double* s1, double* s0,
                                                 int ne, const double* tab) {
    for (int t = threadIdx.x; t < ne * D * Q; t += T) {
      const int e = t / (D * Q), u = t - e * (D * Q);
      const double* in = s1 + e * P1 + u * LS;
      double bx[D];
#pragma unroll
      for (int j = 0; j < D; ++j) bx[j] = in[j];
      const int k = u % D, a = u / D;
      double* o = s0 + e * P0 + a * LS + k;
      if constexpr (NC == 3) {
        double gx[D];
#pragma unroll
        for (int j = 0; j < D; ++j) gx[j] = in[Q * D * LS + j];
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          double br[D], gr[D];
          ld_row(tab + TB + b * DP, br);
          ld_row(tab + TG + b * DP, gr);
          double c0 = br[0] * gx[0];
          double c1 = gr[0] * bx[0];
          double c2 = br[0] * bx[0];
#pragma unroll
          for (int j = 1; j < D; ++j) {
            c0 = fma(br[j], gx[j], c0);
            c1 = fma(gr[j], bx[j], c1);
            c2 = fma(br[j], bx[j], c2);
          }
          o[b * Q * LS] = c0;
          o[Q * Q * LS + b * Q * LS] = c1;
          o[2 * Q * Q * LS + b * Q * LS] = c2;
        }
      } else {
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          double br[D];
          ld_row(tab + TB + b * DP, br);
          double c = br[0] * bx[0];
#pragma unroll
          for (int j = 1; j < D; ++j) c = fma(br[j], bx[j], c);
          o[b * Q * LS] = c;
        }
      }
    }
  }

  // T2 [s][b][a][k] (line r = a + Q b) + D -> W [s][k][a][b]
  __device__ __forceinline__ static void stage_c(const Tables<D, Q>&, const double* s0,
                                                 const double* db, double* s1, int ne,
                                                 const double* tab) {
    for (int t = threadIdx.x; t < ne * Q * Q; t += T) {
      const int e = t / (Q * Q), r = t - e * (Q * Q);
      const double* in = s0 + e * P0 + r * LS;
      const double* pe = db + e * G::PS + r;
      const int a = r % Q, b = r / Q;
      double* o = s1 + e * P1 + a * LQ + b;
      if constexpr (NC == 3) {
        double t0[D], t1[D], t2[D], w0[D], w1[D], w2[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          t0[k] = in[k];
          t1[k] = in[Q * Q * LS + k];
          t2[k] = in[2 * Q * Q * LS + k];
          w0[k] = 0.0;
          w1[k] = 0.0;
          w2[k] = 0.0;
        }
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double br[D], gr[D];
          ld_row(tab + TB + c * DP, br);
          ld_row(tab + TG + c * DP, gr);
          double g0 = br[0] * t0[0];
          double g1 = br[0] * t1[0];
          double g2 = gr[0] * t2[0];
#pragma unroll
          for (int k = 1; k < D; ++k) {
            g0 = fma(br[k], t0[k], g0);
            g1 = fma(br[k], t1[k], g1);
            g2 = fma(gr[k], t2[k], g2);
          }
          const double* pc = pe + c * Q * Q;
          const double d00 = pc[0 * Q3], d01 = pc[1 * Q3], d02 = pc[2 * Q3];
          const double d11 = pc[3 * Q3], d12 = pc[4 * Q3], d22 = pc[5 * Q3];
          const double o0 = fma(d02, g2, fma(d01, g1, d00 * g0));
          const double o1 = fma(d12, g2, fma(d11, g1, d01 * g0));
          const double o2 = fma(d22, g2, fma(d12, g1, d02 * g0));
#pragma unroll
          for (int k = 0; k < D; ++k) {
            w0[k] = fma(br[k], o0, w0[k]);
            w1[k] = fma(br[k], o1, w1[k]);
            w2[k] = fma(gr[k], o2, w2[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
          o[k * Q * LQ] = w0[k];
          o[D * Q * LQ + k * Q * LQ] = w1[k];
          o[2 * D * Q * LQ + k * Q * LQ] = w2[k];
        }
      } else {
        double tt[D], w[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          tt[k] = in[k];
          w[k] = 0.0;
        }
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          double br[D];
          ld_row(tab + TB + c * DP, br);
          double g = br[0] * tt[0];
#pragma unroll
          for (int k = 1; k < D; ++k) g = fma(br[k], tt[k], g);
          const double oo = pe[c * Q * Q] * g;
#pragma unroll
          for (int k = 0; k < D; ++k) w[k] = fma(br[k], oo, w[k]);
        }
#pragma unroll
        for (int k = 0; k < D; ++k) o[k * Q * LQ] = w[k];
      }
    }
  }

  // W [s][k][a][b] (line u = a + Q k) -> R [s][k][j][a]
  __device__ __forceinline__ static void stage_d(const Tables<D, Q>&, const double* s1, double* s0,
                                                 int ne, const double* tab) {
    for (int t = threadIdx.x; t < ne * Q * D; t += T) {
      const int e = t / (Q * D), u = t - e * (Q * D);
      const double* in = s1 + e * P1 + u * LQ;
      const int a = u % Q, k = u / Q;
      double* o = s0 + e * P0 + k * D * LQ + a;
      if constexpr (NC == 3) {
        double w0[Q], w1[Q], w2[Q];
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          w0[b] = in[b];
          w1[b] = in[D * Q * LQ + b];
          w2[b] = in[2 * D * Q * LQ + b];
        }
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double bt[Q], gt[Q];
          ld_row(tab + TBT + j * QP, bt);
          ld_row(tab + TGT + j * QP, gt);
          double rg = bt[0] * w0[0];
          double rb = gt[0] * w1[0];
#pragma unroll
          for (int b = 1; b < Q; ++b) {
            rg = fma(bt[b], w0[b], rg);
            rb = fma(gt[b], w1[b], rb);
          }
#pragma unroll
          for (int b = 0; b < Q; ++b) rb = fma(bt[b], w2[b], rb);
          o[j * LQ] = rg;
          o[D * D * LQ + j * LQ] = rb;
        }
      } else {
        double w[Q];
#pragma unroll
        for (int b = 0; b < Q; ++b) w[b] = in[b];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double bt[Q];
          ld_row(tab + TBT + j * QP, bt);
          double rr = bt[0] * w[0];
#pragma unroll
          for (int b = 1; b < Q; ++b) rr = fma(bt[b], w[b], rr);
          o[j * LQ] = rr;
        }
      }
    }
  }

  // R [s][k][j][a] (line v = j + D k) -> y (atomic scatter-add)
  __device__ __forceinline__ static void stage_e(const Tables<D, Q>&, const double* s0,
                                                 const int* gslot, double* y, int ne,
                                                 const double* tab) {
    for (int t = threadIdx.x; t < ne * D * D; t += T) {
      const int e = t / (D * D), v = t - e * (D * D);
      const double* in = s0 + e * P0 + v * LQ;
      const int* g = gslot + e * G::GS + v * D;
      if constexpr (NC == 3) {
        double rg[Q], rb[Q];
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          rg[a] = in[a];
          rb[a] = in[D * D * LQ + a];
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double bt[Q], gt[Q];
          ld_row(tab + TBT + i * QP, bt);
          ld_row(tab + TGT + i * QP, gt);
          double acc = gt[0] * rg[0];
#pragma unroll
          for (int a = 1; a < Q; ++a) acc = fma(gt[a], rg[a], acc);
#pragma unroll
          for (int a = 0; a < Q; ++a) acc = fma(bt[a], rb[a], acc);
          atomicAdd(y + g[i], acc);
        }
      } else {
        double rr[Q];
#pragma unroll
        for (int a = 0; a < Q; ++a) rr[a] = in[a];
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double bt[Q];
          ld_row(tab + TBT + i * QP, bt);
          double acc = bt[0] * rr[0];
#pragma unroll
          for (int a = 1; a < Q; ++a) acc = fma(bt[a], rr[a], acc);
          atomicAdd(y + g[i], acc);
        }
      }
    }
  }
};

}  // namespace fk
