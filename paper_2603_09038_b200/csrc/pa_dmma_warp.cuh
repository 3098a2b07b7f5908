// pa_dmma_warp.cuh — warp-per-element DMMA PA apply with the contraction
// stages chained in registers (variant dmma, cfgs 9-11; d, q <= 8).
//
// Every contraction is a set of 8x8x(4k) DMMA tiles (mma.sync.m8n8k4.f64,
// SASS DMMA.8x8x4; lane L: A(L/4, L%4), B(L%4, L/4), C(L/4, 2(L%4)+{0,1}),
// feklab/mma.py:70-143).  One warp owns one element at a time and never
// meets a CTA barrier:
//
//   x (i,j,k)      gathered straight into A fragments, one 8x8 tile per k
//                  (rows j, K = i; closed-form ids, Dirichlet bits)
//   A  x-contr.    C_k(j, a) = X_k B^T / G^T                    per k tile
//   B  y-contr.    A = C_k^T (rows a, K = j: 8x8 fragment transpose by
//                  shuffles), C'_k(a, b) for the three BP3 components
//   -> T2[a][comp][k][b]  shared memory (conflict-free: XOR swizzle of b
//                  by k, per-a stride = 8 mod 16, 16-byte stores)
//   C  z + D + z^T per a tile: rows b, K = k; D applied on the accumulators
//                  (PA data read through L2); C -> A re-layout (rows b,
//                  K = c) by shuffles; z^T
//   D  y^T         A = w^T (rows k', K = b: transpose), R_a, R_b
//   -> R[a][r][k'][j'] shared memory, written in place over consumed T2 tiles
//   E  x^T per k' tile: rows j', K = a; scatter-add from the C fragments
//
// Basis fragments (forward: Bop(i, a) = T[a][i]; transposed: Bop(a, i) =
// T[a][i]) live in registers for the whole kernel.  MFEM stage sharing as
// the other bodies: BP3 needs 2 + 3 GEMMs before z, 3 + 3 at z, 3 at y^T, 2
// at x^T per tile.
#pragma once

#include <cstdint>

#include "pa_common.cuh"
#include "pa_dmma.cuh"
#include "pa_pipe.cuh"

// independent 8x8 tiles interleaved per loop trip (ILP across the DMMA ->
// shuffle -> DMMA chains; the kernel is latency-bound at one warp per element)
#ifndef FK_WDMMA_UNROLL
#define FK_WDMMA_UNROLL 2
#endif

namespace fk {

constexpr int kWdmmaUnroll = FK_WDMMA_UNROLL;

template <int D, int Q, int NC>
struct WarpDmmaLayout {
  static_assert(D <= 8 && Q <= 8, "warp DMMA tiles hold d, q <= 8");
  static constexpr int KD = (D + 3) / 4, KQ = (Q + 3) / 4;
  static constexpr int NR = NC == 3 ? 2 : 1;
  static constexpr int X = NC * 64 + 8;   // T2 per-a stride (doubles), = 8 mod 16
  static constexpr int Y = NR * 64 + 4;   // R per-a stride, = 4 mod 16 (<= X: R fits in place)
  static constexpr int WS = 8 * X;        // doubles per warp
  static constexpr int FR = 32 * 2 * (KD + KQ);  // basis fragments (doubles)
  static_assert(Y <= X, "R must fit in place over T2");
};

// T2 word of (component block base, k row, b): XOR-swizzled b keeps both the
// fragment reads (b = L/4, k = 4s + L%4) and the 16-byte pair stores free of
// bank conflicts
__device__ __forceinline__ int t2w(int k, int b) { return k * 8 + (b ^ (((k >> 1) & 1) << 2)); }

// A fragment of the TRANSPOSE of an 8x8 C tile, k-step ks:
// lane L needs C[4ks + L%4][L/4] = lane 4(4ks + L%4) + (L/4)/2, element (L/4)%2
__device__ __forceinline__ double frag_transpose(double c0, double c1, int ks) {
  const int L = threadIdx.x & 31;
  const int src = 4 * (4 * ks + (L & 3)) + ((L >> 2) >> 1);
  const double v0 = __shfl_sync(0xffffffffu, c0, src);
  const double v1 = __shfl_sync(0xffffffffu, c1, src);
  return ((L >> 2) & 1) ? v1 : v0;
}
// A fragment of the SAME C tile (rows kept, K = its columns), k-step ks:
// lane L needs C[L/4][4ks + L%4] = lane 4(L/4) + 2ks + (L%4)/2, element L%2
__device__ __forceinline__ double frag_same(double c0, double c1, int ks) {
  const int L = threadIdx.x & 31;
  const int src = (L & ~3) + 2 * ks + ((L & 3) >> 1);
  const double v0 = __shfl_sync(0xffffffffu, c0, src);
  const double v1 = __shfl_sync(0xffffffffu, c1, src);
  return (L & 1) ? v1 : v0;
}

template <int D, int Q, int NC, int W>
__global__ void __launch_bounds__(32 * W) dmma_warp_kernel(const __grid_constant__ Tables<D, Q> tb,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ y,
                                                           const double* __restrict__ pa,
                                                           const uint32_t* __restrict__ ebits,
                                                           int nel, const StructIds sid) {
  using LY = WarpDmmaLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  constexpr int KD = LY::KD, KQ = LY::KQ, X = LY::X, Y = LY::Y;
  constexpr int Q3 = Q * Q * Q;
  extern __shared__ __align__(16) double wsm[];
  const int L = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r4 = L >> 2, c4 = L & 3;
  double* ws = wsm + warp * LY::WS;
  // work region zeroed once: padded rows/columns must stay finite
  for (int t = L; t < LY::WS; t += 32) ws[t] = 0.0;
  // basis fragments in registers: fB/fG forward (K over a d-index, N over q),
  // tB/tG transposed (K over a q-index, N over d)
  double fB[KD], fG[KD], tBf[KQ], tGf[KQ];
#pragma unroll
  for (int ks = 0; ks < KD; ++ks) {
    const int k = 4 * ks + c4, n = r4;
    const bool ok = k < D && n < Q;
    fB[ks] = ok ? tb.B[n * D + k] : 0.0;
    fG[ks] = ok ? tb.G[n * D + k] : 0.0;
  }
#pragma unroll
  for (int ks = 0; ks < KQ; ++ks) {
    const int k = 4 * ks + c4, n = r4;
    const bool ok = k < Q && n < D;
    tBf[ks] = ok ? tb.B[k * D + n] : 0.0;
    tGf[ks] = ok ? tb.G[k * D + n] : 0.0;
  }
  __syncwarp();

  const int gwarp = blockIdx.x * W + warp, nwarp = gridDim.x * W;
  // PA data toward L2 one element ahead (cp.async.bulk.prefetch.L2): the
  // per-lane fragment loads of stage C then hit L2, not DRAM
  if (L == 0 && gwarp < nel)
    prefetch_l2(pa + (size_t)gwarp * G::PS, (uint32_t)(8 * G::PS));
  for (int e = gwarp; e < nel; e += nwarp) {
    if (L == 0 && e + nwarp < nel)
      prefetch_l2(pa + (size_t)(e + nwarp) * G::PS, (uint32_t)(8 * G::PS));
    // closed-form element base id (h1_restriction, mesh.py:157-164)
    const int eg = (int)(sid.e0 + e);
    const int eyz = fast_div(eg, sid.mnx, sid.snx), ez = fast_div(eyz, sid.mny, sid.sny);
    const int ex = eg - eyz * sid.nx, ey = eyz - ez * sid.ny;
    const int base = ex * sid.p + sid.npx * (ey * sid.p + sid.npy * (ez * sid.p));
    const uint32_t* bits = ebits ? ebits + (size_t)e * G::MS : nullptr;
    const double* pe = pa + (size_t)e * G::PS;
    // x tile k in A-fragment form (rows j, K = i), Dirichlet inputs zeroed
    auto load_x = [&](int k, double (&af)[KD]) {
#pragma unroll
      for (int ks = 0; ks < KD; ++ks) {
        const int i = 4 * ks + c4, j = r4;
        double v = 0.0;
        if (i < D && j < D) {
          const int l = i + D * (j + D * k);
          v = x[base + i + sid.npx * (j + sid.npy * k)];
          if (bits && ((bits[l >> 5] >> (l & 31)) & 1u)) v = 0.0;
        }
        af[ks] = v;
      }
    };
    // D at this lane's two fragment points of a tile (qp = a + Q (b + Q c))
    constexpr int NPC = NC == 3 ? 6 : 1;
    auto load_d = [&](int a, double (&dv)[2][NPC]) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int b = r4, c = 2 * c4 + h;
        const bool ok = b < Q && c < Q;
        const double* pc = pe + a + Q * ((ok ? b : 0) + Q * (ok ? c : 0));
#pragma unroll
        for (int m = 0; m < NPC; ++m) dv[h][m] = ok ? pc[m * Q3] : 0.0;
      }
    };
    // ---- x gather + stages A, B (per k tile, the next tile's gather in flight), T2 stores
    double xn[KD];
    load_x(0, xn);
#pragma unroll kWdmmaUnroll
    for (int k = 0; k < D; ++k) {
      double af[KD];
#pragma unroll
      for (int ks = 0; ks < KD; ++ks) af[ks] = xn[ks];
      if (k + 1 < D) load_x(k + 1, xn);
      double cb0 = 0.0, cb1 = 0.0, cg0 = 0.0, cg1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KD; ++ks) {
        dmma884(cb0, cb1, af[ks], fB[ks]);
        if constexpr (NC == 3) dmma884(cg0, cg1, af[ks], fG[ks]);
      }
      // stage B: rows a, K = j
      double p0[NC][2];
#pragma unroll
      for (int s = 0; s < NC; ++s) p0[s][0] = p0[s][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KD; ++ks) {
        const double ab = frag_transpose(cb0, cb1, ks);
        if constexpr (NC == 3) {
          const double ag = frag_transpose(cg0, cg1, ks);
          dmma884(p0[0][0], p0[0][1], ag, fB[ks]);  // comp 0: G_x B_y
          dmma884(p0[1][0], p0[1][1], ab, fG[ks]);  // comp 1: B_x G_y
          dmma884(p0[2][0], p0[2][1], ab, fB[ks]);  // comp 2: B_x B_y
        } else {
          dmma884(p0[0][0], p0[0][1], ab, fB[ks]);
        }
      }
      // T2[a][s][k][b]: lane holds (a = L/4, b = 2 c4, 2 c4 + 1)
#pragma unroll
      for (int s = 0; s < NC; ++s) {
        double2* dst = reinterpret_cast<double2*>(ws + r4 * X + s * 64 + t2w(k, 2 * c4));
        *dst = make_double2(p0[s][0], p0[s][1]);
      }
    }
    __syncwarp();
    // ---- stages C (z, D, z^T) and D (y^T) per a tile, R stores in place;
    // the next tile's PA data in flight
    double dn[2][NPC];
    load_d(0, dn);
#pragma unroll kWdmmaUnroll
    for (int a = 0; a < Q; ++a) {
      double dc[2][NPC];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int m = 0; m < NPC; ++m) dc[h][m] = dn[h][m];
      if (a + 1 < Q) load_d(a + 1, dn);
      const double* t2 = ws + a * X;
      double g[NC][2];
#pragma unroll
      for (int s = 0; s < NC; ++s) g[s][0] = g[s][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KD; ++ks) {
        const int kk = 4 * ks + c4;
#pragma unroll
        for (int s = 0; s < NC; ++s) {
          const double av = t2[s * 64 + t2w(kk, r4)];
          dmma884(g[s][0], g[s][1], av, (NC == 3 && s == 2) ? fG[ks] : fB[ks]);
        }
      }
      // D at qp = a + Q (b + Q c): lane b = L/4, c = 2 c4 + h
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if constexpr (NC == 3) {
          const double g0 = g[0][h], g1 = g[1][h], g2 = g[2][h];
          const double d00 = dc[h][0], d01 = dc[h][1], d02 = dc[h][2];
          const double d11 = dc[h][3], d12 = dc[h][4], d22 = dc[h][5];
          g[0][h] = fma(d02, g2, fma(d01, g1, d00 * g0));
          g[1][h] = fma(d12, g2, fma(d11, g1, d01 * g0));
          g[2][h] = fma(d22, g2, fma(d12, g1, d02 * g0));
        } else {
          g[0][h] *= dc[h][0];
        }
      }
      // z^T: rows b, K = c
      double w[NC][2];
#pragma unroll
      for (int s = 0; s < NC; ++s) w[s][0] = w[s][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KQ; ++ks)
#pragma unroll
        for (int s = 0; s < NC; ++s) {
          const double av = frag_same(g[s][0], g[s][1], ks);
          dmma884(w[s][0], w[s][1], av, (NC == 3 && s == 2) ? tGf[ks] : tBf[ks]);
        }
      // y^T: rows k', K = b (transpose of w): R_a = B_y^T w0, R_b = G_y^T w1 + B_y^T w2
      double ra0 = 0.0, ra1 = 0.0, rb0 = 0.0, rb1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KQ; ++ks) {
        const double a0 = frag_transpose(w[0][0], w[0][1], ks);
        dmma884(ra0, ra1, a0, tBf[ks]);
        if constexpr (NC == 3) {
          const double a1 = frag_transpose(w[1][0], w[1][1], ks);
          const double a2 = frag_transpose(w[2][0], w[2][1], ks);
          dmma884(rb0, rb1, a1, tGf[ks]);
          dmma884(rb0, rb1, a2, tBf[ks]);
        }
      }
      __syncwarp();  // every lane has read T2 tile a before R overwrites it
      // R[a][r][k'][j']: lane holds (k' = L/4, j' = 2 c4, 2 c4 + 1)
      double* rt = ws + a * Y + r4 * 8 + 2 * c4;
      *reinterpret_cast<double2*>(rt) = make_double2(ra0, ra1);
      if constexpr (NC == 3) *reinterpret_cast<double2*>(rt + 64) = make_double2(rb0, rb1);
    }
    __syncwarp();
    // ---- stage E (x^T) per k' tile, scatter-add
#pragma unroll kWdmmaUnroll
    for (int kp = 0; kp < D; ++kp) {
      double y0 = 0.0, y1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KQ; ++ks) {
        const int aa = 4 * ks + c4;  // K = a
        const double* rr = ws + aa * Y + kp * 8 + r4;
        if constexpr (NC == 3) {
          dmma884(y0, y1, rr[0], tGf[ks]);   // G_x^T R_a
          dmma884(y0, y1, rr[64], tBf[ks]);  // B_x^T R_b
        } else {
          dmma884(y0, y1, rr[0], tBf[ks]);
        }
      }
      const int jp = r4;
      if (jp < D) {
        const int i0 = 2 * c4;
        const int g0 = base + sid.npx * (jp + sid.npy * kp);
        if (i0 < D) atomicAdd(y + g0 + i0, y0);
        if (i0 + 1 < D) atomicAdd(y + g0 + i0 + 1, y1);
      }
    }
    __syncwarp();  // stage E reads of R done before the next element's T2 stores
  }
}

template <int D, int Q, int NC, int W>
struct WarpDmmaKernel {
  using LY = WarpDmmaLayout<D, Q, NC>;
  static constexpr int E = W, T = 32 * W;
  static constexpr size_t SMEM = sizeof(double) * (size_t)W * LY::WS;
  static void launch(const OpView& v, const double* x, double* y, int blocks, cudaStream_t s);
};

}  // namespace fk
