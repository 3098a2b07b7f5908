// pa_dmma_map.cuh — the paper's DMMA PA dataflow (§IV-B..D) for the
// stage shapes the reference ships conflict-free tile maps for: BP3 / BP1 at
// p = 3, q = 5 (m16n5k4, m20n5k4, m25n5k4 forward; m25n4k5, m20n4k5, m16n4k5
// transposed; feklab/mappings/*.map, decoded from pa_dmma_maps.cuh, which
// tools/gen_dmma_maps.py generates through paper_2603_09038_b200.mapping).
//
// As in the paper, every contraction is one small per-element GEMM on
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) with the operands in shared memory:
//   * cyclic index order (§IV-D): each stage contracts the fastest index of
//     its input and appends the new index slowest, so every A operand is
//     K-fastest and every C result is stored m-fastest ("packed"):
//       X(i,j,k) -x-> T1(j,k,a) -y-> T2(k,a,b) -z-> [D] G3(a,b,c)
//       -x^T-> W(b,c,i) -y^T-> R(c,i,j) -z^T-> y_e(i,j,k) -> scatter-add
//   * warp w of an element computes the rows f_m[w][0..7], the columns
//     f_n[...] and reduces over f_k[...] of its map (§IV-C, lane L holds
//     A(L/4, L%4), B(L%4, L/4), C(L/4, 2(L%4)+{0,1}), mma.py:70-143); PAD
//     rows are computed on a valid row and dropped, PAD k slots meet zero
//     B-fragment rows, PAD columns are dropped;
//   * B operands (basis tables) are per-lane fragments built once per CTA.
// Four warps per element (the widest map), E elements per CTA.  BP3 keeps
// MFEM's stage sharing: 2 + 3 forward GEMMs before the z stage, 3 + 3 at z,
// (2 + 1) accumulated GEMMs at y^T and 2 accumulated at z^T.
#pragma once

#include "pa_common.cuh"
#include "pa_dmma.cuh"
#include "pa_dmma_maps.cuh"

namespace fk {

template <class MP>
__device__ __forceinline__ int map_m(int w, int r) {
  return (int)((MP::fm(w) >> (5 * r)) & 31u) - 1;
}
template <class MP>
__device__ __forceinline__ int map_n(int slot) {
  return (int)((MP::FN >> (4 * slot)) & 15u) - 1;
}
template <class MP>
__device__ __forceinline__ int map_k(int slot) {
  return (int)((MP::FK >> (4 * slot)) & 15u) - 1;
}

// acc += A * Bop over map MP for warp slot w; A(m, k) = a[k + K m] (K-fastest)
template <class MP>
__device__ __forceinline__ void map_mma(int w, const double* __restrict__ a,
                                        const double* __restrict__ frag, double (&acc)[MP::NT][2]) {
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  const int m = map_m<MP>(w, r);
  const double* arow = a + MP::K * (m < 0 ? 0 : m);
#pragma unroll
  for (int kt = 0; kt < MP::KT; ++kt) {
    const int k = map_k<MP>(4 * kt + c);
    const double av = arow[k < 0 ? 0 : k];
#pragma unroll
    for (int nt = 0; nt < MP::NT; ++nt)
      dmma884(acc[nt][0], acc[nt][1], av, frag[(nt * MP::KT + kt) * 32 + lane]);
  }
}

// f(m, n, value) for every valid C entry this lane holds
template <class MP, typename F>
__device__ __forceinline__ void map_store(int w, const double (&acc)[MP::NT][2], F f) {
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  const int m = map_m<MP>(w, r);
  if (m < 0) return;
#pragma unroll
  for (int nt = 0; nt < MP::NT; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = map_n<MP>(8 * nt + 2 * c + h);
      if (n >= 0) f(m, n, acc[nt][h]);
    }
}

template <class MP>
__device__ __forceinline__ void zero_acc(double (&acc)[MP::NT][2]) {
#pragma unroll
  for (int nt = 0; nt < MP::NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
}

template <int NC, int E_>
struct DmmaMapBody {
  static constexpr int D = 4, Q = 5;
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  using Tab = Tables<D, Q>;
  using MA = Map<16, 5, 4>;   // x:   (j,k) x i -> a
  using MB = Map<20, 5, 4>;   // y:   (k,a) x j -> b
  using MC = Map<25, 5, 4>;   // z:   (a,b) x k -> c
  using MCT = Map<25, 4, 5>;  // x^T: (b,c) x a -> i
  using MDT = Map<20, 4, 5>;  // y^T: (c,i) x b -> j
  using MET = Map<16, 4, 5>;  // z^T: (i,j) x c -> k
  static constexpr int E = E_, T = 128 * E_, NWE = 4;
  static constexpr bool IP = true;  // W in region 0 (over T2), R in region 1
  static constexpr bool XLAY = true;
  static constexpr int NS = NC == 3 ? 2 : 1;  // T1 / R components
  // per-element regions (doubles, 16-aligned): X canonical (i,j,k); region 0:
  // T2 (NC x 100) then W (NC x 100); region 1: T1 (NS x 80), G3 (NC x 125),
  // then R (NS x 80)
  static constexpr int XS = 64;
  static constexpr int P0 = (NC * 100 + 15) / 16 * 16;
  static constexpr int P1 = (NC * 125 + 15) / 16 * 16;
  // fragment tables (EXTRA): [B fwd | G fwd] per map (MA, MB, MC: 32 doubles;
  // MCT, MDT, MET: 64 doubles), B first then G
  static constexpr int F_A = 0, F_B = 64, F_C = 128, F_CT = 192, F_DT = 320, F_ET = 448;
  static constexpr int EXTRA = 576;

  __device__ __forceinline__ static int xoff(int e, int l) { return e * XS + l; }
  __device__ __forceinline__ static void gather_map(int t, int& e, int& l) {
    e = t / (D * D * D);
    l = t - e * (D * D * D);
  }

  static void fill(Tab& tb, const double* B, const double* Gr) {
    for (int n = 0; n < Q * D; ++n) {
      tb.B[n] = B[n];
      tb.G[n] = Gr[n];
    }
  }

  // frag[(nt KT + kt) 32 + L] = Bop(f_k[4kt + L%4], f_n[8nt + L/4]); forward:
  // Bop(i, a) = T[a][i]; transposed: Bop(a, i) = T[a][i]; PAD -> 0
  template <class MP, bool TR>
  __device__ static void fill_map(double* fr, const double* tab) {
    for (int t = threadIdx.x; t < MP::NT * MP::KT * 32; t += T) {
      const int l = t & 31, kt = (t >> 5) % MP::KT, nt = (t >> 5) / MP::KT;
      const int k = map_k<MP>(4 * kt + (l & 3)), n = map_n<MP>(8 * nt + (l >> 2));
      fr[t] = (k < 0 || n < 0) ? 0.0 : TR ? tab[k * D + n] : tab[n * D + k];
    }
  }
  __device__ static void init(const Tab& tb, double* fr) {
    fill_map<MA, false>(fr + F_A, tb.B);
    fill_map<MA, false>(fr + F_A + 32, tb.G);
    fill_map<MB, false>(fr + F_B, tb.B);
    fill_map<MB, false>(fr + F_B + 32, tb.G);
    fill_map<MC, false>(fr + F_C, tb.B);
    fill_map<MC, false>(fr + F_C + 32, tb.G);
    fill_map<MCT, true>(fr + F_CT, tb.B);
    fill_map<MCT, true>(fr + F_CT + 64, tb.G);
    fill_map<MDT, true>(fr + F_DT, tb.B);
    fill_map<MDT, true>(fr + F_DT + 64, tb.G);
    fill_map<MET, true>(fr + F_ET, tb.B);
    fill_map<MET, true>(fr + F_ET + 64, tb.G);
  }

  // warp -> (element, slot 0..3)
  __device__ __forceinline__ static int elem() { return (int)(threadIdx.x >> 5) / NWE; }
  __device__ __forceinline__ static int slot() { return (int)(threadIdx.x >> 5) % NWE; }

  // x: T1[s](m + 16 a), m = j + 4k, s = 0 (B x), 1 (G x)
  __device__ __forceinline__ static void stage_a(const Tab&, int, const double* xb, double* s1, int ne,
                                                 double* fr) {
    const int e = elem(), w4 = slot();
    if (e >= ne || (NC == 1 && w4 >= MA::W)) return;
    const int s = w4 / MA::W, w = w4 % MA::W;
    double acc[MA::NT][2];
    zero_acc<MA>(acc);
    map_mma<MA>(w, xb + e * XS, fr + F_A + 32 * s, acc);
    double* o = s1 + e * P1 + s * 80;
    map_store<MA>(w, acc, [&](int m, int n, double v) { o[m + 16 * n] = v; });
  }

  // y: T2[c](m' + 20 b), m' = k + 4a; BP3 comps 0 = (G x) B_y, 1 = (B x) G_y, 2 = (B x) B_y
  __device__ __forceinline__ static void stage_b(const Tab&, int, const double* s1, double* s0, int ne,
                                                 double* fr) {
    const int e = elem(), w4 = slot();
    if (e >= ne) return;
    constexpr int NTASK = NC * MB::W;
    for (int t = w4; t < NTASK; t += NWE) {
      const int c = t / MB::W, w = t % MB::W;
      const int src = (NC == 3 && c == 0) ? 1 : 0;
      const int g = (NC == 3 && c == 1) ? 1 : 0;
      double acc[MB::NT][2];
      zero_acc<MB>(acc);
      map_mma<MB>(w, s1 + e * P1 + src * 80, fr + F_B + 32 * g, acc);
      double* o = s0 + e * P0 + c * 100;
      map_store<MB>(w, acc, [&](int m, int n, double v) { o[m + 20 * n] = v; });
    }
  }

  // z + D -> G3[s](m'' + 25 c) (region 1), barrier, x^T -> W[s](m + 25 i) (region 0)
  __device__ __forceinline__ static void stage_c(const Tab&, int, const double* s0, const double* db,
                                                 double* sw, int ne, double* fr) {
    const int e = elem(), w = slot();
    // G3 goes to region 1 (T1 is dead): the pipe lays region 1 out right after
    // region 0's E * P0 doubles (PipeSmem OFF_S1) and passes sw = region 0 (IP)
    double* r1 = sw + E * P0 + e * P1;
    if (e < ne) {
      double acc[NC][MC::NT][2];
#pragma unroll
      for (int s = 0; s < NC; ++s) {
        zero_acc<MC>(acc[s]);
        map_mma<MC>(w, s0 + e * P0 + s * 100, fr + F_C + ((NC == 3 && s == 2) ? 32 : 0), acc[s]);
      }
      // pointwise D at qp = m'' + 25 c (PA layout [comp][qp], operator.py:147-193)
      const double* pe = db + e * G::PS;
      const int lane = threadIdx.x & 31, r = lane >> 2, cc = lane & 3;
      const int m = map_m<MC>(w, r);
      if (m >= 0) {
#pragma unroll
        for (int nt = 0; nt < MC::NT; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int n = map_n<MC>(8 * nt + 2 * cc + h);
            if (n < 0) continue;
            const double* pc = pe + m + 25 * n;
            if constexpr (NC == 3) {
              const double g0 = acc[0][nt][h], g1 = acc[1][nt][h], g2 = acc[2][nt][h];
              const double d00 = pc[0], d01 = pc[125], d02 = pc[250];
              const double d11 = pc[375], d12 = pc[500], d22 = pc[625];
              acc[0][nt][h] = fma(d02, g2, fma(d01, g1, d00 * g0));
              acc[1][nt][h] = fma(d12, g2, fma(d11, g1, d01 * g0));
              acc[2][nt][h] = fma(d22, g2, fma(d12, g1, d02 * g0));
            } else {
              acc[0][nt][h] *= pc[0];
            }
          }
      }
#pragma unroll
      for (int s = 0; s < NC; ++s) {
        double* o = r1 + s * 125;
        map_store<MC>(w, acc[s], [&](int mm, int n, double v) { o[mm + 25 * n] = v; });
      }
    }
    __syncthreads();  // G3 complete; T2 (region 0) dead
    if (e < ne) {
#pragma unroll
      for (int s = 0; s < NC; ++s) {
        double acc[MCT::NT][2];
        zero_acc<MCT>(acc);
        // comp 0 carries G_x: its x^T uses G^T, comps 1, 2 use B^T
        map_mma<MCT>(w, r1 + s * 125, fr + F_CT + ((NC == 3 && s == 0) ? 64 : 0), acc);
        double* o = sw + e * P0 + s * 100;
        map_store<MCT>(w, acc, [&](int m, int n, double v) { o[m + 25 * n] = v; });
      }
    }
  }

  // y^T: R_a = B_y^T W0 + G_y^T W1, R_b = B_y^T W2 (BP1: R = B_y^T W0) -> R[r](m + 20 j)
  __device__ __forceinline__ static void stage_d(const Tab&, int, const double* sw, double* sr, int ne,
                                                 double* fr) {
    const int e = elem(), w4 = slot();
    if (e >= ne) return;
    constexpr int NTASK = NS * MDT::W;
    const double* we = sw + e * P0;
    for (int t = w4; t < NTASK; t += NWE) {
      const int rr = t / MDT::W, w = t % MDT::W;
      double acc[MDT::NT][2];
      zero_acc<MDT>(acc);
      if (NC == 3 && rr == 0) {
        map_mma<MDT>(w, we, fr + F_DT, acc);
        map_mma<MDT>(w, we + 100, fr + F_DT + 64, acc);
      } else {
        map_mma<MDT>(w, we + (NC == 3 ? 200 : 0), fr + F_DT, acc);
      }
      double* o = sr + e * P1 + rr * 80;
      map_store<MDT>(w, acc, [&](int m, int n, double v) { o[m + 20 * n] = v; });
    }
  }

  // z^T: y_e = B_z^T R_a + G_z^T R_b (BP1: B_z^T R) at node m + 16 k -> scatter-add
  __device__ __forceinline__ static void stage_e(const Tab&, int, const double* sr, const int* gslot,
                                                 double* y, int ne, double* fr) {
    const int e = elem(), w = slot();
    if (e >= ne || w >= MET::W) return;
    const double* re = sr + e * P1;
    double acc[MET::NT][2];
    zero_acc<MET>(acc);
    map_mma<MET>(w, re, fr + F_ET, acc);
    if constexpr (NC == 3) map_mma<MET>(w, re + 80, fr + F_ET + 64, acc);
    const int* g = gslot + e * G::GS;
    map_store<MET>(w, acc, [&](int m, int n, double v) { atomicAdd(y + g[m + 16 * n], v); });
  }
};

}  // namespace fk
