// pa_common.cuh — shared definitions for the fused PA operator kernels.
//
// Element tensors follow the reference's cyclic convention
// (feklab/tensor.py:1-8, 177-210): each contraction stage reads lines along
// the contracted (fastest) index and appends the new index as the slowest,
// so after three stages an element block is back in canonical x-fastest order.
// Lines are padded to an odd number of doubles so that 32 lanes reading 32
// different lines of 8-byte words hit distinct shared-memory banks.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fk {

constexpr int odd_up(int n) { return n | 1; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr int cmax3(int a, int b, int c) { return cmax(a, cmax(b, c)); }

// 1D tables passed BY VALUE as a kernel parameter: they live in the constant
// bank, and with fully unrolled loops every DFMA takes its basis entry as a
// c[0x0][imm] operand — no registers or shared-memory loads spent on B, G.
template <int D, int Q>
struct Tables {
  double B[Q * D];  // B[a*D + i] = L_i(x_a)      (Basis1D.values, row-major q x d)
  double G[Q * D];  // G[a*D + i] = L_i'(x_a)     (Basis1D.gradients)
};

// Shared-memory layout of one element for the DFMA line kernel.
// NC = number of reference-gradient components (3 for BP3, 1 for BP1).
//
//   X  [v=(j,k)][i]        D*D lines of LS   (gathered input, canonical)
//   T1 [s][a][k][j]        after x-contraction (s: B x, G x)
//   T2 [s][b][a][k]        after y-contraction (s: comp0, comp1, comp2)
//   W  [s][k][a][b]        after z-contraction + D + transposed z
//   R  [s][k][j][a]        after transposed y (s: G-path, B-path)
//
// Region P0 holds X, then T2, then R; region P1 holds T1, then W.
template <int D, int Q, int NC>
struct LineLayout {
  static constexpr int LS = odd_up(D);
  static constexpr int LQ = odd_up(Q);
  static constexpr int NA = (NC == 3) ? 2 : 1;
  static constexpr int NB = NC;
  static constexpr int NW = NC;
  static constexpr int NR = (NC == 3) ? 2 : 1;
  static constexpr int X_SZ = D * D * LS;
  static constexpr int T1_SZ = NA * Q * D * LS;
  static constexpr int T2_SZ = NB * Q * Q * LS;
  static constexpr int W_SZ = NW * D * Q * LQ;
  static constexpr int R_SZ = NR * D * D * LQ;
  static constexpr int P0 = odd_up(cmax3(X_SZ, T2_SZ, R_SZ));
  static constexpr int P1 = odd_up(cmax(T1_SZ, W_SZ));
  static constexpr int D3 = D * D * D;
  static constexpr int Q3 = Q * Q * Q;
  static constexpr int NPA = (NC == 3) ? 6 : 1;  // stored PA components per point

  static constexpr size_t smem_bytes(int E) {
    return sizeof(double) * (size_t)E * (P0 + P1) + sizeof(int) * (size_t)E * D3;
  }
};

// PA element stride: even and = q^2 (+1) mod 16 (see fk_internal.h pa_stride)
constexpr int pa_pad(int n, int q) { return (((n - q * q) % 16 + 16) % 16 > 1) ? pa_pad(n + 2, q) : n; }

// Global (HBM) layout strides per element, padded so every per-batch range
// is a 16-byte multiple (cp.async.bulk granularity).  Host code mirrors
// these in fk_api.cu (pa_stride / gid_stride / bits_stride).
template <int D, int Q, int NC>
struct GlobalLayout {
  static constexpr int NPA = (NC == 3) ? 6 : 1;
  static constexpr int PS = pa_pad(((NPA * Q * Q * Q + 1) / 2) * 2, Q);  // doubles of PA data per element
  static constexpr int GS = ((D * D * D + 3) / 4) * 4;        // int32 gather ids per element
  static constexpr int MW = (D * D * D + 31) / 32;            // Dirichlet bit words per element
  static constexpr int MS = ((MW + 3) / 4) * 4;               // padded
};

// L2 bulk prefetch (sm_90+): one instruction moves a contiguous range of the
// next batch's PA data toward L2 so the later per-thread loads hit L2.
__device__ __forceinline__ void prefetch_l2(const void* ptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

__device__ __forceinline__ void prefetch_range_l2(const double* base, size_t first, size_t count,
                                                  size_t total) {
  // first/count in doubles; round to 16-byte granules inside [0, total_padded)
  if (count == 0 || first >= total) return;
  size_t last = first + count;
  if (last > total) last = total;
  uintptr_t a = reinterpret_cast<uintptr_t>(base + first) & ~uintptr_t(15);
  uintptr_t b = (reinterpret_cast<uintptr_t>(base + last) + 15) & ~uintptr_t(15);
  prefetch_l2(reinterpret_cast<const void*>(a), static_cast<uint32_t>(b - a));
}

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

}  // namespace fk
