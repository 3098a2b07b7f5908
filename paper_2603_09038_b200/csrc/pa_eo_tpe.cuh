// pa_eo_tpe.cuh — BP1 at p <= 2: one thread per element, every contraction
// in registers (EO cfgs 58-59).
//
// At p = 1-2 the line kernels are bound by the L1 LSU pipe (ncu, BP1 p = 2:
// L1 88%, 43 shared-memory wavefronts per element, 7.2 barrier stalls per
// issue) — an element is only d^3 = 8-27 nodes and q^3 = 27-64 points, so
// per-element shared-memory round trips and CTA barriers dominate.  Here a
// lane owns a whole element:
//   x     gathered straight into registers (closed-form ids; lanes hold
//         consecutive elements, so a warp-wide load covers a few rows)
//   A, B  per z-plane k: T1(j, a) = B x, then T2(k, b, a) = B T1
//   C     per (b, a): z, D, z^T in registers, in place over T2
//   D, E  per z-plane k': R(j, a) = B^T W, y(i) = B^T R -> RED.F64 (lanes
//         on consecutive elements: node-ordered, ~2 sectors per row)
// D is the only shared-memory traffic: one bulk copy per element (lane l
// issues element l's) into the warp's slot array, pitch SP = 2 (mod 16)
// doubles; the next group's copies go out as soon as stage C has read D.
// Same even-odd sums as the line bodies (tensor.py:220-241).
#pragma once

#include <cstdint>

#include "pa_async.cuh"
#include "pa_common.cuh"
#include "pa_dfma_eo.cuh"
#include "pa_pipe.cuh"

namespace fk {

template <int D, int Q, int W>
struct TpeLayout {
  using G = GlobalLayout<D, Q, 1>;
  static constexpr int Q3 = Q * Q * Q;
  static constexpr int CPY = (Q3 + 1) & ~1;  // doubles copied per element (16-byte multiple)
  static_assert(CPY <= G::PS, "copy window inside the element's PA data");
  static constexpr int SP = CPY + (((2 - CPY) % 16) + 16) % 16;  // even, = 2 (mod 16)
  static constexpr int WS = 32 * SP;                               // doubles per warp
  static constexpr size_t SMEM = 16ull * W + 8ull * W * WS;
};

template <int D, int Q, int W, int MINB = 1>
__global__ void __launch_bounds__(32 * W, MINB) tpe_kernel(const __grid_constant__ FoldTables<D, Q> tb,
                                                     const double* __restrict__ x, double* __restrict__ y,
                                                     const double* __restrict__ pa,
                                                     const uint32_t* __restrict__ ebits, int nel,
                                                     const StructIds sid) {
  using LY = TpeLayout<D, Q, W>;
  using G = GlobalLayout<D, Q, 1>;
  using Tab = FoldTables<D, Q>;
  static_assert(D * D * D <= 64, "Dirichlet bits in one or two words");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int L = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw) + 2 * warp;
  double* dbuf = reinterpret_cast<double*>(smem_raw + 16 * W) + warp * LY::WS;
  const double* tab = tb.t[0];
  const int ngroups = (nel + 31) / 32;
  const int gw = blockIdx.x * W + warp, nw = gridDim.x * W;
  if (gw >= ngroups) return;
  if (L == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int t = L; t < LY::WS; t += 32) dbuf[t] = 0.0;  // idle lanes of a ragged group read zeros
  fence_proxy_async();
  __syncwarp();
  // group g's PA data: lane l copies element 32 g + l into its slot
  auto issue = [&](int g) {
    const int ne = min(32, nel - g * 32);
    if (L == 0) mbar_expect_tx(bar, 8u * LY::CPY * (uint32_t)ne);
    __syncwarp();
    if (L < ne) bulk_g2s(dbuf + L * LY::SP, pa + (size_t)(g * 32 + L) * G::PS, 8u * LY::CPY, bar);
  };
  uint32_t phase = 0;
  issue(gw);
  for (int g = gw; g < ngroups; g += nw) {
    const int e = g * 32 + L;
    const bool act = e < nel;
    const int ee = act ? e : nel - 1;  // idle lanes compute a valid element, scatter nothing
    const int eg = (int)(sid.e0 + ee);
    const int eyz = fast_div(eg, sid.mnx, sid.snx), ez = fast_div(eyz, sid.mny, sid.sny);
    const int ex = eg - eyz * sid.nx, ey = eyz - ez * sid.ny;
    const int base = ex * sid.p + sid.npx * (ey * sid.p + sid.npy * (ez * sid.p));
    const uint32_t bits = ebits ? ebits[(size_t)ee * G::MS] : 0u;
    const uint32_t bits1 = (ebits && D * D * D > 32) ? ebits[(size_t)ee * G::MS + 1] : 0u;
    // ---- gather + stages A, B per z-plane k
    double t2[D][Q][Q];  // [k][b][a]: T2, then W in place
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double t1[D][Q];  // [j][a]
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double xr[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
          const int l = i + D * (j + D * k);
          const double v = x[base + i + sid.npx * (j + sid.npy * k)];
          const uint32_t w = l < 32 ? bits : bits1;
          xr[i] = ((w >> (l & 31)) & 1u) ? 0.0 : v;
        }
        contract_eo<D, Q, +1>(tab + Tab::TB, xr, t1[j]);
      }
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        double in[D], o[Q];
#pragma unroll
        for (int j = 0; j < D; ++j) in[j] = t1[j][a];
        contract_eo<D, Q, +1>(tab + Tab::TB, in, o);
#pragma unroll
        for (int b = 0; b < Q; ++b) t2[k][b][a] = o[b];
      }
    }
    // ---- stage C: z, D, z^T per (b, a)
    mbar_wait(bar, phase);
    phase ^= 1u;
    const double* dl = dbuf + L * LY::SP;
#pragma unroll
    for (int b = 0; b < Q; ++b)
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        double in[D], gq[Q], w[D];
#pragma unroll
        for (int k = 0; k < D; ++k) in[k] = t2[k][b][a];
        contract_eo<D, Q, +1>(tab + Tab::TB, in, gq);
#pragma unroll
        for (int c = 0; c < Q; ++c) gq[c] *= dl[a + Q * (b + Q * c)];
        contract_eo<Q, D, +1>(tab + Tab::TBT, gq, w);
#pragma unroll
        for (int k = 0; k < D; ++k) t2[k][b][a] = w[k];
      }
    __syncwarp();  // every lane has read its D slot
    if (g + nw < ngroups) {
      fence_proxy_async();
      issue(g + nw);
    }
    // ---- stages D, E per z-plane k', scatter-add
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double r[D][Q];  // [j][a]
#pragma unroll
      for (int a = 0; a < Q; ++a) {
        double in[Q], o[D];
#pragma unroll
        for (int b = 0; b < Q; ++b) in[b] = t2[k][b][a];
        contract_eo<Q, D, +1>(tab + Tab::TBT, in, o);
#pragma unroll
        for (int j = 0; j < D; ++j) r[j][a] = o[j];
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double o[D];
        contract_eo<Q, D, +1>(tab + Tab::TBT, r[j], o);
        if (act) {
#pragma unroll
          for (int i = 0; i < D; ++i) atomicAdd(y + base + i + sid.npx * (j + sid.npy * k), o[i]);
        }
      }
    }
  }
}

}  // namespace fk
