// pa_dfma.cuh — fused BP1/BP3 PA apply, register-blocked FP64-FMA ("line") variant.
//
// One persistent CTA processes batches of E elements.  Per batch:
//
//   gather   x[gid] -> X (smem), gids kept in smem for the scatter
//            (Restriction.gather, feklab/mesh.py:130-131)
//   stage A  contract x: thread per line (j,k): B x, G x           (tensor.py:177-210)
//   stage B  contract y: thread per line (k,a): 3 component chains
//   stage C  contract z, apply D (6-comp symmetric, BP3; w|J| BP1),
//            transposed z — all in registers for line (a,b)
//   stage D  transposed y: thread per line (a,k)
//   stage E  transposed x: thread per line (j,k), atomic scatter-add to y
//            (Restriction.scatter_add, feklab/mesh.py:133-137)
//
// MFEM-style stage sharing: BP3 costs 2(4qd^3+6q^2d^2+6q^3d)+15q^3 flops per
// element instead of the reference's three independent chains
// (apply_gradient_3d, tensor.py:244-260).  Each thread keeps its line in
// registers and every FMA takes its basis entry from the constant bank
// (kernel parameter), so one 8-byte shared load feeds q (or 2q, 3q) FMAs.
#pragma once

#include "pa_common.cuh"

namespace fk {

template <int D, int Q, int NC, int E, int T>
__global__ void __launch_bounds__(T) pa_dfma_kernel(const __grid_constant__ Tables<D, Q> tb,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y,
                                                    const int* __restrict__ gids,
                                                    const double* __restrict__ pa,
                                                    const unsigned char* __restrict__ mask,
                                                    int nel) {
  using L = LineLayout<D, Q, NC>;
  constexpr int D3 = L::D3, Q3 = L::Q3, NPA = L::NPA;
  constexpr int LS = L::LS, LQ = L::LQ, P0 = L::P0, P1 = L::P1;
  extern __shared__ __align__(16) double smem[];
  double* s0 = smem;
  double* s1 = smem + E * P0;
  int* sg = reinterpret_cast<int*>(s1 + E * P1);

  const int nbatch = (nel + E - 1) / E;
  const size_t pa_total = (size_t)nel * NPA * Q3;
  if (threadIdx.x == 0 && blockIdx.x < nbatch)
    prefetch_range_l2(pa, (size_t)blockIdx.x * E * NPA * Q3, (size_t)E * NPA * Q3, pa_total);

  for (int batch = blockIdx.x; batch < nbatch; batch += gridDim.x) {
    const int e0 = batch * E;
    if (threadIdx.x == 0) {
      const int nb = batch + gridDim.x;
      if (nb < nbatch) prefetch_range_l2(pa, (size_t)nb * E * NPA * Q3, (size_t)E * NPA * Q3, pa_total);
    }
    // ---- gather -------------------------------------------------------
    for (int t = threadIdx.x; t < E * D3; t += T) {
      const int e = t / D3, l = t - e * D3;
      int gid = -1;
      double v = 0.0;
      if (e0 + e < nel) {
        gid = __ldg(gids + (size_t)e0 * D3 + t);
        v = __ldg(x + gid);
        if (mask != nullptr && __ldg(mask + gid)) v = 0.0;
      }
      sg[t] = gid;
      s0[e * P0 + (l / D) * LS + (l % D)] = v;
    }
    __syncthreads();

    // ---- stage A: contract x (i -> a); line v = j + D*k ----------------
    for (int t = threadIdx.x; t < E * D * D; t += T) {
      const int e = t / (D * D), v = t - e * (D * D);
      const double* in = s0 + e * P0 + v * LS;
      double xr[D];
#pragma unroll
      for (int i = 0; i < D; ++i) xr[i] = in[i];
      double* o = s1 + e * P1 + (v / D) * LS + (v % D);
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        double bx = tb.B[a * D] * xr[0];
#pragma unroll
        for (int i = 1; i < D; ++i) bx = fma(tb.B[a * D + i], xr[i], bx);
        o[a * D * LS] = bx;
        if constexpr (NC == 3) {
          double gx = tb.G[a * D] * xr[0];
#pragma unroll
          for (int i = 1; i < D; ++i) gx = fma(tb.G[a * D + i], xr[i], gx);
          o[Q * D * LS + a * D * LS] = gx;
        }
      }
    }
    __syncthreads();

    // ---- stage B: contract y (j -> b); line u = k + D*a ----------------
    for (int t = threadIdx.x; t < E * D * Q; t += T) {
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
          double c0 = tb.B[b * D] * gx[0];
          double c1 = tb.G[b * D] * bx[0];
          double c2 = tb.B[b * D] * bx[0];
#pragma unroll
          for (int j = 1; j < D; ++j) {
            c0 = fma(tb.B[b * D + j], gx[j], c0);
            c1 = fma(tb.G[b * D + j], bx[j], c1);
            c2 = fma(tb.B[b * D + j], bx[j], c2);
          }
          o[b * Q * LS] = c0;
          o[Q * Q * LS + b * Q * LS] = c1;
          o[2 * Q * Q * LS + b * Q * LS] = c2;
        }
      } else {
#pragma unroll
        for (int b = 0; b < Q; ++b) {
          double c = tb.B[b * D] * bx[0];
#pragma unroll
          for (int j = 1; j < D; ++j) c = fma(tb.B[b * D + j], bx[j], c);
          o[b * Q * LS] = c;
        }
      }
    }
    __syncthreads();

    // ---- stage C: contract z, D, transposed z; line r = a + Q*b ---------
    for (int t = threadIdx.x; t < E * Q * Q; t += T) {
      const int e = t / (Q * Q), r = t - e * (Q * Q);
      const bool valid = (e0 + e) < nel;
      const double* in = s0 + e * P0 + r * LS;
      const double* pe = pa + ((size_t)(e0 + e) * NPA * Q3 + r);
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
          double g0 = tb.B[c * D] * t0[0];
          double g1 = tb.B[c * D] * t1[0];
          double g2 = tb.G[c * D] * t2[0];
#pragma unroll
          for (int k = 1; k < D; ++k) {
            g0 = fma(tb.B[c * D + k], t0[k], g0);
            g1 = fma(tb.B[c * D + k], t1[k], g1);
            g2 = fma(tb.G[c * D + k], t2[k], g2);
          }
          double d00 = 0, d01 = 0, d02 = 0, d11 = 0, d12 = 0, d22 = 0;
          if (valid) {
            const double* pc = pe + c * Q * Q;
            d00 = ld_stream(pc + 0 * Q3);
            d01 = ld_stream(pc + 1 * Q3);
            d02 = ld_stream(pc + 2 * Q3);
            d11 = ld_stream(pc + 3 * Q3);
            d12 = ld_stream(pc + 4 * Q3);
            d22 = ld_stream(pc + 5 * Q3);
          }
          const double o0 = fma(d02, g2, fma(d01, g1, d00 * g0));
          const double o1 = fma(d12, g2, fma(d11, g1, d01 * g0));
          const double o2 = fma(d22, g2, fma(d12, g1, d02 * g0));
#pragma unroll
          for (int k = 0; k < D; ++k) {
            w0[k] = fma(tb.B[c * D + k], o0, w0[k]);
            w1[k] = fma(tb.B[c * D + k], o1, w1[k]);
            w2[k] = fma(tb.G[c * D + k], o2, w2[k]);
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
          double g = tb.B[c * D] * tt[0];
#pragma unroll
          for (int k = 1; k < D; ++k) g = fma(tb.B[c * D + k], tt[k], g);
          const double dd = valid ? ld_stream(pe + c * Q * Q) : 0.0;
          const double oo = dd * g;
#pragma unroll
          for (int k = 0; k < D; ++k) w[k] = fma(tb.B[c * D + k], oo, w[k]);
        }
#pragma unroll
        for (int k = 0; k < D; ++k) o[k * Q * LQ] = w[k];
      }
    }
    __syncthreads();

    // ---- stage D: transposed y (b -> j); line u = a + Q*k ---------------
    for (int t = threadIdx.x; t < E * Q * D; t += T) {
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
          double rg = tb.B[j] * w0[0];
          double rb = tb.G[j] * w1[0];
#pragma unroll
          for (int b = 1; b < Q; ++b) {
            rg = fma(tb.B[b * D + j], w0[b], rg);
            rb = fma(tb.G[b * D + j], w1[b], rb);
          }
#pragma unroll
          for (int b = 0; b < Q; ++b) rb = fma(tb.B[b * D + j], w2[b], rb);
          o[j * LQ] = rg;
          o[D * D * LQ + j * LQ] = rb;
        }
      } else {
        double w[Q];
#pragma unroll
        for (int b = 0; b < Q; ++b) w[b] = in[b];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double rr = tb.B[j] * w[0];
#pragma unroll
          for (int b = 1; b < Q; ++b) rr = fma(tb.B[b * D + j], w[b], rr);
          o[j * LQ] = rr;
        }
      }
    }
    __syncthreads();

    // ---- stage E: transposed x (a -> i) + scatter; line v = j + D*k ------
    for (int t = threadIdx.x; t < E * D * D; t += T) {
      const int e = t / (D * D), v = t - e * (D * D);
      const double* in = s0 + e * P0 + v * LQ;
      const int* g = sg + e * D3 + v * D;
      if constexpr (NC == 3) {
        double rg[Q], rb[Q];
#pragma unroll
        for (int a = 0; a < Q; ++a) {
          rg[a] = in[a];
          rb[a] = in[D * D * LQ + a];
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double acc = tb.G[i] * rg[0];
#pragma unroll
          for (int a = 1; a < Q; ++a) acc = fma(tb.G[a * D + i], rg[a], acc);
#pragma unroll
          for (int a = 0; a < Q; ++a) acc = fma(tb.B[a * D + i], rb[a], acc);
          const int gid = g[i];
          if (gid >= 0) atomicAdd(y + gid, acc);
        }
      } else {
        double rr[Q];
#pragma unroll
        for (int a = 0; a < Q; ++a) rr[a] = in[a];
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double acc = tb.B[i] * rr[0];
#pragma unroll
          for (int a = 1; a < Q; ++a) acc = fma(tb.B[a * D + i], rr[a], acc);
          const int gid = g[i];
          if (gid >= 0) atomicAdd(y + gid, acc);
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace fk
