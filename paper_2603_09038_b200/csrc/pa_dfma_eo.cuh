// pa_dfma_eo.cuh — contraction stages of the fused PA apply, FP64-FMA lines
// with even-odd (symmetry) folding.  Plugs into pa_pipe.cuh.
//
// GLL nodes and Gauss points are symmetric about the element centre, so the
// 1D tables satisfy  B[q-1-a][d-1-i] = B[a][i]  and  G[q-1-a][d-1-i] = -G[a][i].
// A contraction out[a] = sum_i N[a][i] in[i] with N[no-1-a][ni-1-i] = S N[a][i]
// folds into  e_i = in_i + in_{ni-1-i},  o_i = in_i - in_{ni-1-i}:
//     E_a = sum_i Ne[a][i] e_i (+ Nm[a] in_mid),   O_a = sum_i No[a][i] o_i,
//     out[a] = E_a + O_a,   out[no-1-a] = S (E_a - O_a),
// with Ne = (N[a][i] + N[a][ni-1-i])/2, No = (N[a][i] - N[a][ni-1-i])/2 —
// half the multiply-adds and half the table entries of the direct sum
// (Kronbichler & Kormann's even-odd decomposition).  Same operator as the
// reference's ascending sums (tensor.py:177-210) up to FP64 rounding; the
// host symmetrises the given tables (averaging the mirrored entries, whose
// difference is ~1e-16 for the reference's tables) and only selects this
// body when that symmetry holds (fk_api.cu: tables_symmetric).
//
// Dataflow, layouts and the ping-pong parameter tables are those of
// pa_dfma.cuh (see its header for the ptxas uniform-register finding).
#pragma once

#include "pa_common.cuh"
#include "pa_dfma.cuh"

namespace fk {

// Folded table of an (NO x NI) matrix: rows a < HO, each
// [Ne(a, 0..HI-1) | No(a, 0..HI-1) | Nm(a) if NI odd], row pitch RP (16-byte).
template <int NO, int NI>
struct Fold {
  static constexpr int HI = NI / 2, HO = (NO + 1) / 2, RL = 2 * HI + (NI & 1), RP = RL + (RL & 1);
  static constexpr int SIZE = HO * RP;
};

template <int D, int Q>
struct __align__(16) FoldTables {
  using FQD = Fold<Q, D>;  // B, G   (q x d)
  using FDQ = Fold<D, Q>;  // B^T, G^T (d x q)
  static constexpr int TB = 0, TG = FQD::SIZE, TBT = 2 * FQD::SIZE, TGT = 2 * FQD::SIZE + FDQ::SIZE;
  static constexpr int SZ = 2 * FQD::SIZE + 2 * FDQ::SIZE;
  double t[2][SZ];  // two copies (ping-pong by batch parity, see pa_dfma.cuh)
};

// host: fold N (NO x NI, row-major) with symmetry sign S into dst (Fold layout)
template <int NO, int NI>
inline void fold_table(double* dst, const double* N, int S) {
  using F = Fold<NO, NI>;
  for (int a = 0; a < F::HO; ++a) {
    double* row = dst + a * F::RP;
    for (int k = 0; k < F::RP; ++k) row[k] = 0.0;
    auto sym = [&](int aa, int i) {  // symmetrised entry N[aa][i]
      return 0.5 * (N[aa * NI + i] + S * N[(NO - 1 - aa) * NI + (NI - 1 - i)]);
    };
    const bool mid_row = (a == NO - 1 - a);
    for (int i = 0; i < F::HI; ++i) {
      const double n1 = sym(a, i), n2 = sym(a, NI - 1 - i);
      double ne = 0.5 * (n1 + n2), no = 0.5 * (n1 - n2);
      if (mid_row) {
        if (S > 0) no = 0.0;
        else ne = 0.0;
      }
      row[i] = ne;
      row[F::HI + i] = no;
    }
    if (NI & 1) row[2 * F::HI] = (mid_row && S < 0) ? 0.0 : sym(a, F::HI);
  }
}

// out = N in, N given folded at t (Fold<NO,NI> layout), symmetry sign S
template <int NI, int NO, int S>
__device__ __forceinline__ void contract_eo(const double* __restrict__ t, const double (&in)[NI],
                                            double (&out)[NO]) {
  using F = Fold<NO, NI>;
  constexpr int HI = F::HI;
  double xe[HI > 0 ? HI : 1], xo[HI > 0 ? HI : 1];
#pragma unroll
  for (int i = 0; i < HI; ++i) {
    xe[i] = in[i] + in[NI - 1 - i];
    xo[i] = in[i] - in[NI - 1 - i];
  }
#pragma unroll
  for (int a = 0; a < F::HO; ++a) {
    double row[F::RL];
    ld_row(t + a * F::RP, row);
    double E, O;
    if constexpr (NI & 1) {
      E = row[2 * HI] * in[HI];
#pragma unroll
      for (int i = 0; i < HI; ++i) E = fma(row[i], xe[i], E);
    } else {
      E = row[0] * xe[0];
#pragma unroll
      for (int i = 1; i < HI; ++i) E = fma(row[i], xe[i], E);
    }
    if constexpr (HI > 0) {
      O = row[HI] * xo[0];
#pragma unroll
      for (int i = 1; i < HI; ++i) O = fma(row[HI + i], xo[i], O);
    } else {
      O = 0.0;
    }
    if (a == NO - 1 - a) {
      out[a] = E + O;
    } else {
      out[a] = E + O;
      out[NO - 1 - a] = (S > 0) ? (E - O) : (O - E);
    }
  }
}

// IP (in place): stage C reads its T2 line into registers, the CTA syncs,
// and W overwrites T2 in region 0; R then lives in region 1.  The two work
// regions shrink from max(T2,R)+max(T1,W) to max(T2,W)+max(T1,R) doubles
// per element, which buys one more resident CTA per SM at p=4.
template <int D, int Q, int NC, int E_, int T_, bool IP_ = false>
struct DfmaEoBody {
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  using Tab = FoldTables<D, Q>;
  static constexpr bool IP = IP_;
  static constexpr int LS = L::LS, LQ = L::LQ, Q3 = L::Q3;
  static constexpr int P0 = IP ? odd_up(cmax3(L::X_SZ, L::T2_SZ, L::W_SZ)) : L::P0;
  static constexpr int P1 = IP ? odd_up(cmax(L::T1_SZ, L::R_SZ)) : L::P1;
  static constexpr int WST = IP ? P0 : P1;  // element stride of the region holding W
  static constexpr int RST = IP ? P1 : P0;  // ... and R
  static constexpr int XS = D * D * LS;
  static constexpr int E = E_, T = T_, EXTRA = 0;
  static_assert(!IP || E * Q * Q <= T, "in-place stage C needs one pass over its lines");

  static void fill(Tab& tb, const double* B, const double* Gr) {
    double Bt[Q * D], Gt[Q * D];
    for (int a = 0; a < Q; ++a)
      for (int i = 0; i < D; ++i) {
        Bt[i * Q + a] = B[a * D + i];
        Gt[i * Q + a] = Gr[a * D + i];
      }
    for (int c = 0; c < 2; ++c) {
      fold_table<Q, D>(tb.t[c] + Tab::TB, B, +1);
      fold_table<Q, D>(tb.t[c] + Tab::TG, Gr, -1);
      fold_table<D, Q>(tb.t[c] + Tab::TBT, Bt, +1);
      fold_table<D, Q>(tb.t[c] + Tab::TGT, Gt, -1);
    }
  }

  __device__ static void init(const Tab&, double*) {}

  // X [v=(j,k)][i] -> T1 [s][a][k][j]
  __device__ __forceinline__ static void stage_a(const Tab& tb, int it, const double* xb, double* s1,
                                                 int ne, double*) {
    const double* tab = tb.t[it & 1];
    lines_loop<T, E * D * D>(ne * D * D, [&](int t) {
      const int e = t / (D * D), v = t - e * (D * D);
      const double* in = xb + e * XS + v * LS;
      double xr[D], bx[Q];
#pragma unroll
      for (int i = 0; i < D; ++i) xr[i] = in[i];
      double* o = s1 + e * P1 + (v / D) * LS + (v % D);
      contract_eo<D, Q, +1>(tab + Tab::TB, xr, bx);
#pragma unroll
      for (int a = 0; a < Q; ++a) o[a * D * LS] = bx[a];
      if constexpr (NC == 3) {
        double gx[Q];
        contract_eo<D, Q, -1>(tab + Tab::TG, xr, gx);
#pragma unroll
        for (int a = 0; a < Q; ++a) o[Q * D * LS + a * D * LS] = gx[a];
      }
    });
  }

  // T1 [s][a][k][j] (line u = k + D a) -> T2 [s][b][a][k]
  __device__ __forceinline__ static void stage_b(const Tab& tb, int it, const double* s1, double* s0,
                                                 int ne, double*) {
    const double* tab = tb.t[it & 1];
    lines_loop<T, E * D * Q>(ne * D * Q, [&](int t) {
      const int e = t / (D * Q), u = t - e * (D * Q);
      const double* in = s1 + e * P1 + u * LS;
      double bx[D];
#pragma unroll
      for (int j = 0; j < D; ++j) bx[j] = in[j];
      double* o = s0 + e * P0 + (u / D) * LS + (u % D);
      double c[Q];
      if constexpr (NC == 3) {
        double gx[D];
#pragma unroll
        for (int j = 0; j < D; ++j) gx[j] = in[Q * D * LS + j];
        contract_eo<D, Q, +1>(tab + Tab::TB, gx, c);  // comp0 = B_y G_x
#pragma unroll
        for (int b = 0; b < Q; ++b) o[b * Q * LS] = c[b];
        contract_eo<D, Q, -1>(tab + Tab::TG, bx, c);  // comp1 = G_y B_x
#pragma unroll
        for (int b = 0; b < Q; ++b) o[Q * Q * LS + b * Q * LS] = c[b];
        contract_eo<D, Q, +1>(tab + Tab::TB, bx, c);  // comp2 = B_y B_x
#pragma unroll
        for (int b = 0; b < Q; ++b) o[2 * Q * Q * LS + b * Q * LS] = c[b];
      } else {
        contract_eo<D, Q, +1>(tab + Tab::TB, bx, c);
#pragma unroll
        for (int b = 0; b < Q; ++b) o[b * Q * LS] = c[b];
      }
    });
  }

  // T2 [s][b][a][k] (line r = a + Q b) + D -> W [s][k][a][b] (region sw, stride WST)
  __device__ __forceinline__ static void stage_c(const Tab& tb, int it, const double* s0,
                                                 const double* db, double* sw, int ne, double*) {
    const double* tab = tb.t[it & 1];
    const int n = ne * Q * Q;
    constexpr int NIT = (E * Q * Q + T - 1) / T;
#pragma unroll
    for (int pass = 0; pass < NIT; ++pass) {
      const int t0 = threadIdx.x + pass * T;
      const bool act = t0 < n;
      const int t = act ? t0 : 0;
      const int e = t / (Q * Q), r = t - e * (Q * Q);
      const double* in = s0 + e * P0 + r * LS;
      double tin[NC][D];
#pragma unroll
      for (int s = 0; s < NC; ++s)
#pragma unroll
        for (int k = 0; k < D; ++k) tin[s][k] = in[s * Q * Q * LS + k];
      if constexpr (IP) __syncthreads();  // every T2 line is in registers: W may overwrite it
      if (!act) continue;
      const double* pe = db + e * G::PS + r;
      double* o = sw + e * WST + (r % Q) * LQ + (r / Q);
      if constexpr (NC == 3) {
        double g0[Q], g1[Q], g2[Q];
        contract_eo<D, Q, +1>(tab + Tab::TB, tin[0], g0);
        contract_eo<D, Q, +1>(tab + Tab::TB, tin[1], g1);
        contract_eo<D, Q, -1>(tab + Tab::TG, tin[NC - 1], g2);
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const double* pc = pe + c * Q * Q;
          const double d00 = pc[0 * Q3], d01 = pc[1 * Q3], d02 = pc[2 * Q3];
          const double d11 = pc[3 * Q3], d12 = pc[4 * Q3], d22 = pc[5 * Q3];
          const double a0 = g0[c], a1 = g1[c], a2 = g2[c];
          g0[c] = fma(d02, a2, fma(d01, a1, d00 * a0));
          g1[c] = fma(d12, a2, fma(d11, a1, d01 * a0));
          g2[c] = fma(d22, a2, fma(d12, a1, d02 * a0));
        }
        double w[D];
        contract_eo<Q, D, +1>(tab + Tab::TBT, g0, w);
#pragma unroll
        for (int k = 0; k < D; ++k) o[k * Q * LQ] = w[k];
        contract_eo<Q, D, +1>(tab + Tab::TBT, g1, w);
#pragma unroll
        for (int k = 0; k < D; ++k) o[D * Q * LQ + k * Q * LQ] = w[k];
        contract_eo<Q, D, -1>(tab + Tab::TGT, g2, w);
#pragma unroll
        for (int k = 0; k < D; ++k) o[2 * D * Q * LQ + k * Q * LQ] = w[k];
      } else {
        double g[Q], w[D];
        contract_eo<D, Q, +1>(tab + Tab::TB, tin[0], g);
#pragma unroll
        for (int c = 0; c < Q; ++c) g[c] *= pe[c * Q * Q];
        contract_eo<Q, D, +1>(tab + Tab::TBT, g, w);
#pragma unroll
        for (int k = 0; k < D; ++k) o[k * Q * LQ] = w[k];
      }
    }
  }

  // W [s][k][a][b] (line u = a + Q k) -> R [s][k][j][a]   (W stride WST, R stride RST)
  __device__ __forceinline__ static void stage_d(const Tab& tb, int it, const double* sw, double* sr,
                                                 int ne, double*) {
    const double* tab = tb.t[it & 1];
    lines_loop<T, E * Q * D>(ne * Q * D, [&](int t) {
      const int e = t / (Q * D), u = t - e * (Q * D);
      const double* in = sw + e * WST + u * LQ;
      double* o = sr + e * RST + (u / Q) * D * LQ + (u % Q);
      double wv[Q], r0[D];
#pragma unroll
      for (int b = 0; b < Q; ++b) wv[b] = in[b];
      contract_eo<Q, D, +1>(tab + Tab::TBT, wv, r0);  // rG = B^T w0 (BP1: r = B^T w)
#pragma unroll
      for (int j = 0; j < D; ++j) o[j * LQ] = r0[j];
      if constexpr (NC == 3) {
        double r1[D];
#pragma unroll
        for (int b = 0; b < Q; ++b) wv[b] = in[D * Q * LQ + b];
        contract_eo<Q, D, -1>(tab + Tab::TGT, wv, r0);  // G^T w1
#pragma unroll
        for (int b = 0; b < Q; ++b) wv[b] = in[2 * D * Q * LQ + b];
        contract_eo<Q, D, +1>(tab + Tab::TBT, wv, r1);  // B^T w2
#pragma unroll
        for (int j = 0; j < D; ++j) o[D * D * LQ + j * LQ] = r0[j] + r1[j];
      }
    });
  }

  // R [s][k][j][a] (line v = j + D k) -> y (atomic scatter-add)
  __device__ __forceinline__ static void stage_e(const Tab& tb, int it, const double* sr,
                                                 const int* gslot, double* y, int ne, double*) {
    const double* tab = tb.t[it & 1];
    lines_loop<T, E * D * D>(ne * D * D, [&](int t) {
      const int e = t / (D * D), v = t - e * (D * D);
      const double* in = sr + e * RST + v * LQ;
      const int* g = gslot + e * G::GS + v * D;
      double rv[Q], out[D];
#pragma unroll
      for (int a = 0; a < Q; ++a) rv[a] = in[a];
      if constexpr (NC == 3) {
        double o2[D];
        contract_eo<Q, D, -1>(tab + Tab::TGT, rv, out);  // G^T rG
#pragma unroll
        for (int a = 0; a < Q; ++a) rv[a] = in[D * D * LQ + a];
        contract_eo<Q, D, +1>(tab + Tab::TBT, rv, o2);  // B^T rB
#pragma unroll
        for (int i = 0; i < D; ++i) atomicAdd(y + g[i], out[i] + o2[i]);
      } else {
        contract_eo<Q, D, +1>(tab + Tab::TBT, rv, out);
#pragma unroll
        for (int i = 0; i < D; ++i) atomicAdd(y + g[i], out[i]);
      }
    });
  }
};

}  // namespace fk
