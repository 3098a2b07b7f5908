// pa_diag.cuh — assembled diagonal of the PA operator (Jacobi preconditioner).
// Setup-time only; templated per order like the fused kernels.
#pragma once

#include <cstdint>

#include "pa_common.cuh"

namespace fk {

// Assembled diagonal of A = sum_e G_e^T A_e G_e (Jacobi preconditioner).
// diag_e(i,j,k) = sum_{abc} sum_{s,t} D_st(abc) dphi_s dphi_t with
// dphi_0 = G_ai B_bj B_ck, dphi_1 = B_ai G_bj B_ck, dphi_2 = B_ai B_bj G_ck;
// BP1: sum_{abc} D(abc) (B_ai B_bj B_ck)^2.  One thread per (element, node).
template <int D, int Q, int NC>
__global__ void diagonal_kernel(const __grid_constant__ Tables<D, Q> tb,
                                double* __restrict__ diag, const int* __restrict__ gids,
                                const double* __restrict__ pa, int64_t nel) {
  constexpr int D3 = D * D * D, Q3 = Q * Q * Q;
  using G = GlobalLayout<D, Q, NC>;
  const int64_t total = nel * D3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / D3;
    const int l = (int)(t - e * D3);
    const int i = l % D, j = (l / D) % D, k = l / (D * D);
    const double* pe = pa + e * G::PS;
    double acc = 0.0;
    for (int c = 0; c < Q; ++c) {
      const double bc = tb.B[c * D + k], gc = tb.G[c * D + k];
      for (int b = 0; b < Q; ++b) {
        const double bb = tb.B[b * D + j], gb = tb.G[b * D + j];
        for (int a = 0; a < Q; ++a) {
          const double ba = tb.B[a * D + i], ga = tb.G[a * D + i];
          const int qp = a + Q * (b + Q * c);
          if constexpr (NC == 3) {
            const double p0 = ga * bb * bc, p1 = ba * gb * bc, p2 = ba * bb * gc;
            acc += pe[0 * Q3 + qp] * p0 * p0 + pe[3 * Q3 + qp] * p1 * p1 +
                   pe[5 * Q3 + qp] * p2 * p2 +
                   2.0 * (pe[1 * Q3 + qp] * p0 * p1 + pe[2 * Q3 + qp] * p0 * p2 +
                          pe[4 * Q3 + qp] * p1 * p2);
          } else {
            const double p0 = ba * bb * bc;
            acc += pe[qp] * p0 * p0;
          }
        }
      }
    }
    atomicAdd(diag + gids[e * G::GS + l], acc);
  }
}

}  // namespace fk
