// pa_dmma.cuh — contraction stages of the fused PA apply on the FP64 tensor
// cores: warp-level mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4, the
// only FP64 tensor instruction sm_100a has; tcgen05 has no f64 kind).
// Plugs into pa_pipe.cuh.
//
// Each stage is a batched small GEMM  C[m][n] = sum_k A[m][k] * Bop[k][n]:
//   m = (element, line) rows of all E elements of the CTA (batching along M
//       removes the M-padding waste of per-element tiles),
//   k = the contracted 1D index (K-concatenated where two legs are summed),
//   n = the new 1D index (N-concatenated where one input feeds both B and G).
// Fragment semantics follow the reference's emulation (feklab/mma.py:70-143):
// lane L holds A(L/4, L%4), B(L%4, L/4), C(L/4, 2(L%4)+{0,1}); padded entries
// of the B operand are zero (mma.py:283-296).  B fragments (basis tables,
// pre-swizzled per lane into shared memory once per CTA) are held in
// registers for the whole stage.
//
// Branch-free operand loads: the K padding of A reads the neighbouring line
// (finite data: all work regions are zeroed once per CTA and afterwards only
// hold computed values) and is annihilated by the zero rows of Bop; rows past
// the batch are clamped to the last valid row; only stores are predicated.
//
// Stage C keeps its accumulators in registers: the three gradient components
// land in identical C-fragment positions, D is applied in registers, and the
// C fragments are re-laid out as A fragments of the transposed z-contraction
// with two warp shuffles per k-step — no shared-memory round trip.
#pragma once

#include "pa_common.cuh"

namespace fk {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }

// Batched stage over 8-row tiles of rows [0, rows), distributed over warps.
// arow(m) -> const double* of row m's A operand (k-th entry at arow(m)[k]);
// store(m, n, c0, c1) writes C[m][n], C[m][n+1] (caller predicates on n).
template <int NW, int KS, int NT, typename ARow, typename Store>
__device__ __forceinline__ void dmma_stage(int rows, const double* __restrict__ frag, ARow arow,
                                           Store store) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, c = lane & 3;
  if (warp * 8 >= rows) return;
  double bf[NT][KS];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bf[nt][ks] = frag[(nt * KS + ks) * 32 + lane];
  for (int m0 = warp * 8; m0 < rows; m0 += NW * 8) {
    const int m = m0 + r;
    const int mm = m < rows ? m : rows - 1;
    const double* ap = arow(mm) + c;
    double acc[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const double a = ap[4 * ks];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma884(acc[nt][0], acc[nt][1], a, bf[nt][ks]);
    }
    if (m < rows) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) store(mm, nt * 8 + 2 * c, acc[nt][0], acc[nt][1]);
    }
  }
}

// Same with a K-concatenated A operand: entries [0, K1) from p1(m), [K1, ...) from p2(m).
template <int NW, int KS, int NT, int K1, typename ARow1, typename ARow2, typename Store>
__device__ __forceinline__ void dmma_stage2(int rows, const double* __restrict__ frag, ARow1 arow1,
                                            ARow2 arow2, Store store) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, c = lane & 3;
  if (warp * 8 >= rows) return;
  double bf[NT][KS];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bf[nt][ks] = frag[(nt * KS + ks) * 32 + lane];
  for (int m0 = warp * 8; m0 < rows; m0 += NW * 8) {
    const int m = m0 + r;
    const int mm = m < rows ? m : rows - 1;
    const double* p1 = arow1(mm);
    const double* p2 = arow2(mm) - K1;
    double acc[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = 4 * ks + c;
      const double a = (k < K1 ? p1 : p2)[k];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma884(acc[nt][0], acc[nt][1], a, bf[nt][ks]);
    }
    if (m < rows) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) store(mm, nt * 8 + 2 * c, acc[nt][0], acc[nt][1]);
    }
  }
}

template <int D, int Q, int NC, int E_, int T_>
struct DmmaBody {
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  using Tab = Tables<D, Q>;
  static constexpr int E = E_, T = T_, NW = T_ / 32;
  static constexpr int LS = L::LS, LQ = L::LQ, P0 = L::P0, P1 = L::P1, Q3 = L::Q3, D3 = L::D3;
  static constexpr bool IP = false;
  static constexpr int XS = D * D * LS;
  static constexpr int KD = cdiv(D, 4), KQ = cdiv(Q, 4), K2Q = cdiv(2 * Q, 4);
  static constexpr int NQ = cdiv(Q, 8), N2Q = cdiv(2 * Q, 8), ND = cdiv(D, 8);
  static constexpr int NA = (NC == 3) ? N2Q : NQ;
  // per-lane fragment tables in smem (doubles; 32 per (ntile, kstep))
  static constexpr int F_A = 0;                    // [B;G] (BP1: B), K = D
  static constexpr int F_B1 = F_A + NA * KD * 32;  // [G;B] (BP1: B), K = D
  static constexpr int F_CB = F_B1 + NA * KD * 32; // B, K = D
  static constexpr int F_CG = F_CB + NQ * KD * 32; // G, K = D
  static constexpr int F_TB = F_CG + NQ * KD * 32; // B^T, K = Q
  static constexpr int F_TG = F_TB + ND * KQ * 32; // G^T, K = Q
  static constexpr int F_GB = F_TG + ND * KQ * 32; // [G^T;B^T], K = 2Q
  static constexpr int SLACK = 32;                 // K-padding reads past the last line
  static constexpr int EXTRA = F_GB + ND * K2Q * 32 + SLACK;

  static void fill(Tab& tb, const double* B, const double* Gr) {
    for (int n = 0; n < Q * D; ++n) {
      tb.B[n] = B[n];
      tb.G[n] = Gr[n];
    }
  }

  template <typename Bop>
  __device__ static void fill_frag(double* fr, int off, int ntiles, int ksteps, Bop bop) {
    for (int t = threadIdx.x; t < ntiles * ksteps * 32; t += T) {
      const int l = t & 31, ks = (t >> 5) % ksteps, nt = (t >> 5) / ksteps;
      fr[off + t] = bop(4 * ks + (l & 3), 8 * nt + (l >> 2));
    }
  }

  // frag(nt, ks, L) = Bop[4ks + L%4][8nt + L/4]  (work regions were zeroed by the pipe)
  __device__ static void init(const Tab& tb, double* fr) {
    if constexpr (NC == 3) {
      fill_frag(fr, F_A, NA, KD, [&](int k, int n) {
        return k >= D ? 0.0 : n < Q ? tb.B[n * D + k] : n < 2 * Q ? tb.G[(n - Q) * D + k] : 0.0;
      });
      fill_frag(fr, F_B1, NA, KD, [&](int k, int n) {
        return k >= D ? 0.0 : n < Q ? tb.G[n * D + k] : n < 2 * Q ? tb.B[(n - Q) * D + k] : 0.0;
      });
    } else {
      fill_frag(fr, F_A, NA, KD, [&](int k, int n) { return (k < D && n < Q) ? tb.B[n * D + k] : 0.0; });
      fill_frag(fr, F_B1, NA, KD, [&](int k, int n) { return (k < D && n < Q) ? tb.B[n * D + k] : 0.0; });
    }
    fill_frag(fr, F_CB, NQ, KD, [&](int k, int n) { return (k < D && n < Q) ? tb.B[n * D + k] : 0.0; });
    fill_frag(fr, F_CG, NQ, KD, [&](int k, int n) { return (k < D && n < Q) ? tb.G[n * D + k] : 0.0; });
    fill_frag(fr, F_TB, ND, KQ, [&](int k, int n) { return (k < Q && n < D) ? tb.B[k * D + n] : 0.0; });
    fill_frag(fr, F_TG, ND, KQ, [&](int k, int n) { return (k < Q && n < D) ? tb.G[k * D + n] : 0.0; });
    fill_frag(fr, F_GB, ND, K2Q, [&](int k, int n) {
      return n >= D ? 0.0 : k < Q ? tb.G[k * D + n] : k < 2 * Q ? tb.B[(k - Q) * D + n] : 0.0;
    });
  }

  // rows (e, v = j + D k), K = i, N = [B;G] a  ->  T1 [s][a][k][j]
  __device__ __forceinline__ static void stage_a(const Tab&, int, const double* xb, double* s1, int ne,
                                                 double* fr) {
    auto arow = [&](int m) { return xb + (m / (D * D)) * XS + (m % (D * D)) * LS; };
    auto store = [&](int m, int n, double c0, double c1) {
      const int e = m / (D * D), v = m - e * (D * D);
      double* o = s1 + e * P1 + (v / D) * LS + (v % D);
      // n < Q: B x (s=0, a = n); Q <= n < 2Q: G x (s=1, a = n - Q); a*D*LS + s*Q*D*LS = n*D*LS
      constexpr int NOUT = (NC == 3) ? 2 * Q : Q;
      if (n < NOUT) o[n * D * LS] = c0;
      if (n + 1 < NOUT) o[(n + 1) * D * LS] = c1;
    };
    dmma_stage<NW, KD, NA>(ne * D * D, fr + F_A, arow, store);
  }

  // rows (e, u = k + D a), K = j  ->  T2 [s][b][a][k]
  __device__ __forceinline__ static void stage_b(const Tab&, int, const double* s1, double* s0, int ne,
                                                 double* fr) {
    // T2 offset of (s, b) for row u: s*Q*Q*LS + b*Q*LS + (u/D)*LS + u%D
    auto obase = [&](int m) {
      const int e = m / (D * Q), u = m - e * (D * Q);
      return s0 + e * P0 + (u / D) * LS + (u % D);
    };
    auto abx = [&](int m) { return s1 + (m / (D * Q)) * P1 + (m % (D * Q)) * LS; };
    if constexpr (NC == 3) {
      // B x -> [G;B]: comp1 = G_y B_x (s=1, n < Q), comp2 = B_y B_x (s=2, n >= Q):
      // offset (s-1+1)*Q*Q*LS + b*Q*LS = Q*Q*LS + n*Q*LS for both halves
      auto st12 = [&](int m, int n, double c0, double c1) {
        double* o = obase(m) + Q * Q * LS;
        if (n < 2 * Q) o[n * Q * LS] = c0;
        if (n + 1 < 2 * Q) o[(n + 1) * Q * LS] = c1;
      };
      dmma_stage<NW, KD, N2Q>(ne * D * Q, fr + F_B1, abx, st12);
      auto agx = [&](int m) { return s1 + (m / (D * Q)) * P1 + Q * D * LS + (m % (D * Q)) * LS; };
      auto st0 = [&](int m, int n, double c0, double c1) {
        double* o = obase(m);
        if (n < Q) o[n * Q * LS] = c0;
        if (n + 1 < Q) o[(n + 1) * Q * LS] = c1;
      };
      dmma_stage<NW, KD, NQ>(ne * D * Q, fr + F_CB, agx, st0);
    } else {
      auto st0 = [&](int m, int n, double c0, double c1) {
        double* o = obase(m);
        if (n < Q) o[n * Q * LS] = c0;
        if (n + 1 < Q) o[(n + 1) * Q * LS] = c1;
      };
      dmma_stage<NW, KD, NQ>(ne * D * Q, fr + F_B1, abx, st0);
    }
  }

  // rows (e, r = a + Q b): z-contraction, D (from smem), transposed z -> W [s][k][a][b]
  __device__ __forceinline__ static void stage_c(const Tab&, int, const double* s0, const double* db,
                                                 double* s1, int ne, double* fr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, rr = lane >> 2, cc = lane & 3;
    const int rows = ne * Q * Q;
    if (warp * 8 >= rows) return;
    double fcb[NQ][KD], fcg[NQ][KD], ftb[ND][KQ], ftg[ND][KQ];
#pragma unroll
    for (int nt = 0; nt < NQ; ++nt)
#pragma unroll
      for (int ks = 0; ks < KD; ++ks) {
        fcb[nt][ks] = fr[F_CB + (nt * KD + ks) * 32 + lane];
        fcg[nt][ks] = NC == 3 ? fr[F_CG + (nt * KD + ks) * 32 + lane] : 0.0;
      }
#pragma unroll
    for (int nt = 0; nt < ND; ++nt)
#pragma unroll
      for (int ks = 0; ks < KQ; ++ks) {
        ftb[nt][ks] = fr[F_TB + (nt * KQ + ks) * 32 + lane];
        ftg[nt][ks] = NC == 3 ? fr[F_TG + (nt * KQ + ks) * 32 + lane] : 0.0;
      }
    const int src = (lane & ~3) + ((lane & 3) >> 1);
    for (int m0 = warp * 8; m0 < rows; m0 += NW * 8) {
      const int m = m0 + rr;
      const int mm = m < rows ? m : rows - 1;
      const int e = mm / (Q * Q), r = mm - e * (Q * Q);
      const double* ap = s0 + e * P0 + r * LS + cc;
      double g[NC][NQ][2];
#pragma unroll
      for (int s = 0; s < NC; ++s)
#pragma unroll
        for (int nt = 0; nt < NQ; ++nt) g[s][nt][0] = g[s][nt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KD; ++ks) {
#pragma unroll
        for (int s = 0; s < NC; ++s) {
          const double a = ap[s * Q * Q * LS + 4 * ks];
#pragma unroll
          for (int nt = 0; nt < NQ; ++nt)
            dmma884(g[s][nt][0], g[s][nt][1], a, (NC == 3 && s == 2) ? fcg[nt][ks] : fcb[nt][ks]);
        }
      }
      // pointwise D on the fragments: entry (m, c = 8nt + 2cc + h), qp = r + Q^2 c
      // (columns c >= Q hold 0 and stay 0; their D address is clamped in range)
      const double* pe = db + e * G::PS + r;
#pragma unroll
      for (int nt = 0; nt < NQ; ++nt) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = nt * 8 + 2 * cc + h;
          const double* pc = pe + (c < Q ? c : Q - 1) * Q * Q;
          if constexpr (NC == 3) {
            const double d00 = pc[0], d01 = pc[Q3], d02 = pc[2 * Q3];
            const double d11 = pc[3 * Q3], d12 = pc[4 * Q3], d22 = pc[5 * Q3];
            const double g0 = g[0][nt][h], g1 = g[1][nt][h], g2 = g[2][nt][h];
            g[0][nt][h] = fma(d02, g2, fma(d01, g1, d00 * g0));
            g[1][nt][h] = fma(d12, g2, fma(d11, g1, d01 * g0));
            g[2][nt][h] = fma(d22, g2, fma(d12, g1, d02 * g0));
          } else {
            g[0][nt][h] *= pc[0];
          }
        }
      }
      // transposed z: W_s[m][k'] = sum_c Mat_s[c][k'] o_s[m][c]; A fragments from
      // C fragments: A(row, 4ks + L%4) lives in lane 4(L/4) + 2(ks%2) + (L%4)/2,
      // register (L%2), of C tile ks/2.
      double w[NC][ND][2];
#pragma unroll
      for (int s = 0; s < NC; ++s)
#pragma unroll
        for (int nt = 0; nt < ND; ++nt) w[s][nt][0] = w[s][nt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KQ; ++ks) {
        const int tile = ks >> 1, sl = src + 2 * (ks & 1);
#pragma unroll
        for (int s = 0; s < NC; ++s) {
          const double v0 = __shfl_sync(0xffffffffu, g[s][tile][0], sl);
          const double v1 = __shfl_sync(0xffffffffu, g[s][tile][1], sl);
          const double a = (lane & 1) ? v1 : v0;
#pragma unroll
          for (int nt = 0; nt < ND; ++nt)
            dmma884(w[s][nt][0], w[s][nt][1], a, (NC == 3 && s == 2) ? ftg[nt][ks] : ftb[nt][ks]);
        }
      }
      if (m < rows) {
        double* o = s1 + e * P1 + (r % Q) * LQ + (r / Q);
#pragma unroll
        for (int nt = 0; nt < ND; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int kk = nt * 8 + 2 * cc + h;
            if (kk < D) {
#pragma unroll
              for (int s = 0; s < NC; ++s) o[s * D * Q * LQ + kk * Q * LQ] = w[s][nt][h];
            }
          }
      }
    }
  }

  // rows (e, u = a + Q k), K = b (transposed y) -> R [s][k][j][a]
  __device__ __forceinline__ static void stage_d(const Tab&, int, const double* s1, double* s0, int ne,
                                                 double* fr) {
    auto obase = [&](int m) {
      const int e = m / (Q * D), u = m - e * (Q * D);
      return s0 + e * P0 + (u / Q) * D * LQ + (u % Q);
    };
    auto a0 = [&](int m) { return s1 + (m / (Q * D)) * P1 + (m % (Q * D)) * LQ; };
    auto st0 = [&](int m, int n, double c0, double c1) {
      double* o = obase(m);
      if (n < D) o[n * LQ] = c0;
      if (n + 1 < D) o[(n + 1) * LQ] = c1;
    };
    dmma_stage<NW, KQ, ND>(ne * Q * D, fr + F_TB, a0, st0);  // rG = B^T w0 (BP1: r = B^T w)
    if constexpr (NC == 3) {
      auto a1 = [&](int m) { return s1 + (m / (Q * D)) * P1 + D * Q * LQ + (m % (Q * D)) * LQ; };
      auto a2 = [&](int m) { return s1 + (m / (Q * D)) * P1 + 2 * D * Q * LQ + (m % (Q * D)) * LQ; };
      auto st1 = [&](int m, int n, double c0, double c1) {
        double* o = obase(m) + D * D * LQ;
        if (n < D) o[n * LQ] = c0;
        if (n + 1 < D) o[(n + 1) * LQ] = c1;
      };
      dmma_stage2<NW, K2Q, ND, Q>(ne * Q * D, fr + F_GB, a1, a2, st1);  // rB = G^T w1 + B^T w2
    }
  }

  // rows (e, v = j + D k), K = a (transposed x) -> atomic scatter-add
  __device__ __forceinline__ static void stage_e(const Tab&, int, const double* s0, const int* gslot,
                                                 double* y, int ne, double* fr) {
    auto store = [&](int m, int n, double c0, double c1) {
      const int e = m / (D * D), v = m - e * (D * D);
      const int* g = gslot + e * G::GS + v * D;
      if (n < D) atomicAdd(y + g[n], c0);
      if (n + 1 < D) atomicAdd(y + g[n + 1], c1);
    };
    auto a0 = [&](int m) { return s0 + (m / (D * D)) * P0 + (m % (D * D)) * LQ; };
    if constexpr (NC == 3) {
      auto a1 = [&](int m) { return s0 + (m / (D * D)) * P0 + D * D * LQ + (m % (D * D)) * LQ; };
      dmma_stage2<NW, K2Q, ND, Q>(ne * D * D, fr + F_GB, a0, a1, store);
    } else {
      dmma_stage<NW, KQ, ND>(ne * D * D, fr + F_TB, a0, store);
    }
  }
};

}  // namespace fk
