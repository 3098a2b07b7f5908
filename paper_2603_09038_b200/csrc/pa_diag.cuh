// pa_diag.cuh — assembled diagonal of the PA operator (Jacobi preconditioner).
// Setup-time only; templated per order like the fused kernels.
#pragma once

#include <cstdint>

#include "pa_common.cuh"

namespace fk {

// Assembled diagonal of A = sum_e G_e^T A_e G_e (Jacobi preconditioner).
// diag_e(i,j,k) = sum_{s<=t} w_st sum_{abc} D_st(abc) X_st[a][i] Y_st[b][j] Z_st[c][k]
// with w = 1 (s = t) or 2, and per-dimension factors X_st = X_s X_t (X_0 = G,
// X_1 = X_2 = B; Y_1 = G; Z_2 = G; everything else B), since
// dphi_0 = G_ai B_bj B_ck, dphi_1 = B_ai G_bj B_ck, dphi_2 = B_ai B_bj G_ck.
// BP1: D (B_ai B_bj B_ck)^2.  Sum-factorised per (s,t) pair: three
// contractions q^3 -> d q^2 -> d^2 q -> d^3, one CTA per element.
template <int D, int Q, int NC>
__global__ void __launch_bounds__(128) diagonal_kernel(const __grid_constant__ Tables<D, Q> tb,
                                                       double* __restrict__ diag,
                                                       const int* __restrict__ gids,
                                                       const double* __restrict__ pa, int64_t nel) {
  constexpr int D3 = D * D * D, Q3 = Q * Q * Q;
  constexpr int NP = (NC == 3) ? 6 : 1;
  using G = GlobalLayout<D, Q, NC>;
  __shared__ double sB[Q * D], sG[Q * D];
  __shared__ double s0[Q3], s1[D * Q * Q], s2[D * D * Q], acc[D3];
  for (int t = threadIdx.x; t < Q * D; t += blockDim.x) {
    sB[t] = tb.B[t];
    sG[t] = tb.G[t];
  }
  // pairs (s,t) in PA component order 00 01 02 11 12 22
  constexpr int PS_[6] = {0, 0, 0, 1, 1, 2}, PT_[6] = {0, 1, 2, 1, 2, 2};
  for (int64_t e = blockIdx.x; e < nel; e += gridDim.x) {
    for (int l = threadIdx.x; l < D3; l += blockDim.x) acc[l] = 0.0;
    for (int pr = 0; pr < NP; ++pr) {
      const int ps = PS_[pr], pt = PT_[pr];
      const double w = (ps == pt) ? 1.0 : 2.0;
      const double* X0 = (NC == 3 && ps == 0) ? sG : sB;  // x factor of s
      const double* X1 = (NC == 3 && pt == 0) ? sG : sB;
      const double* Y0 = (NC == 3 && ps == 1) ? sG : sB;
      const double* Y1 = (NC == 3 && pt == 1) ? sG : sB;
      const double* Z0 = (NC == 3 && ps == 2) ? sG : sB;
      const double* Z1 = (NC == 3 && pt == 2) ? sG : sB;
      __syncthreads();
      const double* pe = pa + e * G::PS + pr * Q3;
      for (int t = threadIdx.x; t < Q3; t += blockDim.x) s0[t] = pe[t];
      __syncthreads();
      // s1[i + D(b + Q c)] = sum_a X[a][i] s0[a + Q(b + Q c)]
      for (int t = threadIdx.x; t < D * Q * Q; t += blockDim.x) {
        const int i = t % D, bc = t / D;
        double v = 0.0;
        for (int a = 0; a < Q; ++a) v = fma(X0[a * D + i] * X1[a * D + i], s0[a + Q * bc], v);
        s1[t] = v;
      }
      __syncthreads();
      // s2[i + D(j + D c)] = sum_b Y[b][j] s1[i + D(b + Q c)]
      for (int t = threadIdx.x; t < D * D * Q; t += blockDim.x) {
        const int i = t % D, j = (t / D) % D, c = t / (D * D);
        double v = 0.0;
        for (int b = 0; b < Q; ++b) v = fma(Y0[b * D + j] * Y1[b * D + j], s1[i + D * (b + Q * c)], v);
        s2[t] = v;
      }
      __syncthreads();
      // acc[i + D(j + D k)] += w sum_c Z[c][k] s2[i + D(j + D c)]
      for (int t = threadIdx.x; t < D3; t += blockDim.x) {
        const int ij = t % (D * D), k = t / (D * D);
        double v = 0.0;
        for (int c = 0; c < Q; ++c) v = fma(Z0[c * D + k] * Z1[c * D + k], s2[ij + D * D * c], v);
        acc[t] += w * v;
      }
    }
    __syncthreads();
    for (int l = threadIdx.x; l < D3; l += blockDim.x) atomicAdd(diag + gids[e * G::GS + l], acc[l]);
  }
}

}  // namespace fk
