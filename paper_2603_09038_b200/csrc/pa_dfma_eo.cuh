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
  // matrix-free (MF) factors: 1D quadrature weights, |J| and jinv_s^2
  // (operator.py:137-144, 280-286: the reference's MF recomputes the diagonal
  // w|J|J^-1 of the axis-aligned box per element instead of reading dmat)
  double mfw[Q + (Q & 1)];
  double mfc[4];  // detJ, jinv_0^2, jinv_1^2, jinv_2^2
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

// one folded row applied to a folded input: E (even part, + middle entry) and O
template <int NI, int RL, int HI>
__device__ __forceinline__ void eo_row(const double (&row)[RL], const double* xe, const double* xo,
                                       double mid, double& E, double& O) {
  if constexpr (NI & 1) {
    E = row[2 * HI] * mid;
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
}

template <int NI>
__device__ __forceinline__ void eo_fold(const double (&in)[NI], double* xe, double* xo) {
#pragma unroll
  for (int i = 0; i < NI / 2; ++i) {
    xe[i] = in[i] + in[NI - 1 - i];
    xo[i] = in[i] - in[NI - 1 - i];
  }
}

template <int NO, int S>
__device__ __forceinline__ void eo_out(int a, double E, double O, double (&out)[NO]) {
  out[a] = E + O;
  if (a != NO - 1 - a) out[NO - 1 - a] = (S > 0) ? (E - O) : (O - E);
}

// out = N in, N given folded at t (Fold<NO,NI> layout), symmetry sign S
template <int NI, int NO, int S>
__device__ __forceinline__ void contract_eo(const double* __restrict__ t, const double (&in)[NI],
                                            double (&out)[NO]) {
  using F = Fold<NO, NI>;
  constexpr int HI = F::HI;
  double xe[HI > 0 ? HI : 1], xo[HI > 0 ? HI : 1];
  eo_fold<NI>(in, xe, xo);
#pragma unroll
  for (int a = 0; a < F::HO; ++a) {
    double row[F::RL];
    ld_row(t + a * F::RP, row);
    double E, O;
    eo_row<NI, F::RL, HI>(row, xe, xo, in[HI], E, O);
    eo_out<NO, S>(a, E, O, out);
  }
}

// the same table applied to two inputs: every folded row is loaded once
// (LDCU.128 table loads were ~18% of the BP3 kernel's instructions)
template <int NI, int NO, int S>
__device__ __forceinline__ void contract_eo2(const double* __restrict__ t, const double (&in0)[NI],
                                             const double (&in1)[NI], double (&out0)[NO],
                                             double (&out1)[NO]) {
  using F = Fold<NO, NI>;
  constexpr int HI = F::HI;
  double xe0[HI > 0 ? HI : 1], xo0[HI > 0 ? HI : 1], xe1[HI > 0 ? HI : 1], xo1[HI > 0 ? HI : 1];
  eo_fold<NI>(in0, xe0, xo0);
  eo_fold<NI>(in1, xe1, xo1);
#pragma unroll
  for (int a = 0; a < F::HO; ++a) {
    double row[F::RL];
    ld_row(t + a * F::RP, row);
    double E, O;
    eo_row<NI, F::RL, HI>(row, xe0, xo0, in0[HI], E, O);
    eo_out<NO, S>(a, E, O, out0);
    eo_row<NI, F::RL, HI>(row, xe1, xo1, in1[HI], E, O);
    eo_out<NO, S>(a, E, O, out1);
  }
}

// two inputs through one table: shared row loads (SR) or two separate passes
template <bool SR, int NI, int NO, int S>
__device__ __forceinline__ void contract_pair(const double* __restrict__ t, const double (&in0)[NI],
                                              const double (&in1)[NI], double (&out0)[NO],
                                              double (&out1)[NO]) {
  if constexpr (SR) {
    contract_eo2<NI, NO, S>(t, in0, in1, out0, out1);
  } else {
    contract_eo<NI, NO, S>(t, in0, out0);
    contract_eo<NI, NO, S>(t, in1, out1);
  }
}

// ---------------------------------------------------------------------------
// Shared-memory layouts.  Every intermediate buffer has a padded linear layout
//     word(e, s, i1, i2, i3) = e*SE + s*SS + i1*S1 + i2*S2 + i3*S3
// in the canonical index order
//     X  (i, j, k)   gathered dofs            T1 (a, j, k)   after x
//     T2 (a, b, k)   after y                  W  (a, b, k)   after z, D, z^T
//     R  (a, j, k)   after y^T
// and every stage maps its threads to lines through a LineMap (element-major
// or element-minor, either line index fastest).  The layouts and maps of the
// tuned geometries come from tools/smem_strides.py, which minimises
// shared-memory wavefronts (bank conflicts and partially filled half-warps)
// for the stage access patterns below.
template <int SE, int SS, int S1, int S2, int S3>
struct BufLay {
  static constexpr int se = SE;
  __device__ __forceinline__ static int at(int e, int s, int i1, int i2, int i3) {
    return e * SE + s * SS + i1 * S1 + i2 * S2 + i3 * S3;
  }
};

// thread t -> (element e, line indices p1 < N1, p2 < N2)
//   M = 0: element-major, p1 fastest     M = 1: element-major, p2 fastest
//   M = 2: element-minor, p1 fastest     M = 3: element-minor, p2 fastest
template <int M, int E, int N1, int N2>
__device__ __forceinline__ void line_map(int t, int& e, int& p1, int& p2) {
  constexpr int L = N1 * N2;
  int l;
  if constexpr (M < 2) {
    e = t / L;
    l = t - e * L;
  } else {
    l = t / E;
    e = t - l * E;
  }
  if constexpr (M == 0 || M == 2) {
    p2 = l / N1;
    p1 = l - p2 * N1;
  } else {
    p1 = l / N2;
    p2 = l - p1 * N2;
  }
}

// The line layout of the first even-odd kernels (odd line pitches LS = D|1,
// LQ = Q|1; W over T1 or, in place, over T2), expressed as BufLays.
template <int D, int Q, int NC, bool IP>
struct EoLayDefault {
  using L = LineLayout<D, Q, NC>;
  static constexpr int LS = L::LS, LQ = L::LQ;
  static constexpr int P0 = IP ? odd_up(cmax3(L::X_SZ, L::T2_SZ, L::W_SZ)) : L::P0;
  static constexpr int P1 = IP ? odd_up(cmax(L::T1_SZ, L::R_SZ)) : L::P1;
  static constexpr int WST = IP ? P0 : P1, RST = IP ? P1 : P0;
  static constexpr bool W_OVER_T2 = IP;
  static constexpr int MG = 0, MA = 0, MB = 1, MC = 0, MD = 0, ME = 0;
  using X = BufLay<D * D * LS, 0, 1, LS, D * LS>;
  using T1 = BufLay<P1, Q * D * LS, D * LS, 1, LS>;
  using T2 = BufLay<P0, Q * Q * LS, LS, Q * LS, 1>;
  using W = BufLay<WST, D * Q * LQ, LQ, 1, Q * LQ>;
  using R = BufLay<RST, D * D * LQ, 1, LQ, D * LQ>;
};

// layout policies of bodies that replace stages B-D (pa_eo_bcd.cuh: NO_C)
template <class LP, class = void>
struct LayNoC {
  static constexpr bool value = false;
};
template <class LP>
struct LayNoC<LP, decltype((void)LP::NO_C)> {
  static constexpr bool value = LP::NO_C;
};

// Even-odd FP64-FMA body over layout policy LP (EoLayDefault or a searched
// layout).  W_OVER_T2 (in place): stage C reads its T2 line into registers,
// the CTA syncs, and W overwrites T2 in region 0; R then lives in region 1 —
// max(T2,W)+max(T1,R) instead of max(T2,R)+max(T1,W) doubles per element.
//
// PP (ping-pong tables, pa_dfma.cuh header): batch `it` reads table copy it&1,
// so the loads stay loop-variant and ptxas cannot hoist the whole table into
// (spilled) registers.  At p >= 6 with three components the dynamic index
// instead makes ptxas fall back from uniform LDCU to per-thread LDC and holds
// 126-165 registers (vs 75-88 static); PP = false uses the static copy 0.
template <int D, int Q, int NC, int E_, int T_, class LP, bool PP = true, bool SR = true>
struct DfmaEoBody {
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  using Tab = FoldTables<D, Q>;
  using LX = typename LP::X;
  using LT1 = typename LP::T1;
  using LT2 = typename LP::T2;
  using LW = typename LP::W;
  using LR = typename LP::R;
  static constexpr bool IP = LP::W_OVER_T2;
  static constexpr int Q3 = L::Q3;
  static constexpr int E = E_, T = T_, EXTRA = 0;
  // region 0: T2 then R (or W); region 1: T1 then W (or R); per-element
  // strides as the pipeline expects (it allocates E * P0 and E * P1 doubles)
  static constexpr int R0 = cmax(E * LT2::se, E * (IP ? LW::se : LR::se));
  static constexpr int R1 = cmax(E * LT1::se, E * (IP ? LR::se : LW::se));
  static constexpr int P0 = (R0 + E - 1) / E, P1 = (R1 + E - 1) / E;
  // X buffer (pa_pipe.cuh gathers into it through xoff / gather_map)
  static constexpr bool XLAY = true;
  static constexpr int XS = LX::se;
  __device__ __forceinline__ static int xoff(int e, int l) {
    const int k = l / (D * D), j = (l / D) % D, i = l % D;
    return LX::at(e, 0, i, j, k);
  }
  __device__ __forceinline__ static void gather_map(int t, int& e, int& l) {
    if constexpr (LP::MG < 2) {
      e = t / (D * D * D);
      l = t - e * (D * D * D);
    } else {
      l = t / E;
      e = t - l * E;
    }
  }
  static_assert(!IP || E * Q * Q <= T || LayNoC<LP>::value, "in-place stage C needs one pass over its lines");

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

  static void fill_mf(Tab& tb, const double* w, double detj, const double* jinv) {
    for (int a = 0; a < Q; ++a) tb.mfw[a] = w[a];
    tb.mfc[0] = detj;
    for (int s = 0; s < 3; ++s) tb.mfc[1 + s] = jinv[s] * jinv[s];
  }

  __device__ static void init(const Tab&, double*) {}

  // run f(e, p1, p2) over the stage's lines of the batch's ne elements
  template <int M, int N1, int N2, typename F>
  __device__ __forceinline__ static void lines(int ne, F f) {
    constexpr int N = E * N1 * N2;
    auto one = [&](int t) {
      int e, p1, p2;
      line_map<M, E, N1, N2>(t, e, p1, p2);
      if (e < ne) f(e, p1, p2);
    };
    if constexpr (N <= T) {
      if ((int)threadIdx.x < N) one((int)threadIdx.x);
    } else {
      for (int t = threadIdx.x; t < N; t += T) one(t);
    }
  }

  // X (i, j, k) -> T1 (a, j, k): thread per line (j, k)
  __device__ __forceinline__ static void stage_a(const Tab& tb, int it, const double* xb, double* s1,
                                                 int ne, double*) {
    const double* tab = tb.t[PP ? (it & 1) : 0];
    lines<LP::MA, D, D>(ne, [&](int e, int j, int k) {
      double xr[D], bx[Q];
#pragma unroll
      for (int i = 0; i < D; ++i) xr[i] = xb[LX::at(e, 0, i, j, k)];
      contract_eo<D, Q, +1>(tab + Tab::TB, xr, bx);
#pragma unroll
      for (int a = 0; a < Q; ++a) s1[LT1::at(e, 0, a, j, k)] = bx[a];
      if constexpr (NC == 3) {
        double gx[Q];
        contract_eo<D, Q, -1>(tab + Tab::TG, xr, gx);
#pragma unroll
        for (int a = 0; a < Q; ++a) s1[LT1::at(e, 1, a, j, k)] = gx[a];
      }
    });
  }

  // T1 (a, j, k) -> T2 (a, b, k): thread per line (a, k)
  __device__ __forceinline__ static void stage_b(const Tab& tb, int it, const double* s1, double* s0,
                                                 int ne, double*) {
    const double* tab = tb.t[PP ? (it & 1) : 0];
    lines<LP::MB, Q, D>(ne, [&](int e, int a, int k) {
      double bx[D], c[Q];
#pragma unroll
      for (int j = 0; j < D; ++j) bx[j] = s1[LT1::at(e, 0, a, j, k)];
      if constexpr (NC == 3) {
        double gx[D];
#pragma unroll
        for (int j = 0; j < D; ++j) gx[j] = s1[LT1::at(e, 1, a, j, k)];
        double c2[Q];
        contract_pair<SR, D, Q, +1>(tab + Tab::TB, gx, bx, c, c2);  // comp0 = B_y G_x, comp2 = B_y B_x
#pragma unroll
        for (int b = 0; b < Q; ++b) s0[LT2::at(e, 0, a, b, k)] = c[b];
#pragma unroll
        for (int b = 0; b < Q; ++b) s0[LT2::at(e, 2, a, b, k)] = c2[b];
        contract_eo<D, Q, -1>(tab + Tab::TG, bx, c);  // comp1 = G_y B_x
#pragma unroll
        for (int b = 0; b < Q; ++b) s0[LT2::at(e, 1, a, b, k)] = c[b];
      } else {
        contract_eo<D, Q, +1>(tab + Tab::TB, bx, c);
#pragma unroll
        for (int b = 0; b < Q; ++b) s0[LT2::at(e, 0, a, b, k)] = c[b];
      }
    });
  }

  // T2 (a, b, k) + D -> W (a, b, k): thread per line (a, b); W region sw.
  // MF: D computed from the 1D weights and the element Jacobian, in the PA
  // setup's operation order (fk_setup.cuh pa_data_kernel), so bit-identical.
  // qacc (optional): += sum over this thread's quadrature points of g^T D g,
  // g the reference gradients (BP3) / values (BP1) at the point — the element
  // quadratic form x_e^T A_e x_e, i.e. p.Ap of a CG iteration without a pass
  // over the assembled vectors (fk_api.cu cg_iteration)
  static constexpr bool QF_OK = true;
  template <bool MF = false>
  __device__ __forceinline__ static void stage_c(const Tab& tb, int it, const double* s0,
                                                 const double* db, double* sw, int ne, double*,
                                                 double* qacc = nullptr) {
    const double* tab = tb.t[PP ? (it & 1) : 0];
    constexpr int N = E * Q * Q;
    constexpr int NIT = (N + T - 1) / T;
#pragma unroll
    for (int pass = 0; pass < NIT; ++pass) {
      const int t0 = threadIdx.x + pass * T;
      int e, a, b;
      line_map<LP::MC, E, Q, Q>(t0 < N ? t0 : 0, e, a, b);
      const bool act = t0 < N && e < ne;
      if (!act) e = 0;
      double tin[NC][D];
#pragma unroll
      for (int s = 0; s < NC; ++s)
#pragma unroll
        for (int k = 0; k < D; ++k) tin[s][k] = s0[LT2::at(e, s, a, b, k)];
      if constexpr (IP) __syncthreads();  // every T2 line is in registers: W may overwrite it
      if (!act) continue;
      const double* pe = MF ? nullptr : db + e * G::PS + a + Q * b;
      const double wab = MF ? tb.mfw[b] * tb.mfw[a] : 0.0;
      if constexpr (NC == 3) {
        double g0[Q], g1[Q], g2[Q];
        contract_pair<SR, D, Q, +1>(tab + Tab::TB, tin[0], tin[1], g0, g1);
        contract_eo<D, Q, -1>(tab + Tab::TG, tin[NC - 1], g2);
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const double a0 = g0[c], a1 = g1[c], a2 = g2[c];
          if constexpr (MF) {
            const double wdet = (tb.mfw[c] * wab) * tb.mfc[0];
            g0[c] = (wdet * tb.mfc[1]) * a0;
            g1[c] = (wdet * tb.mfc[2]) * a1;
            g2[c] = (wdet * tb.mfc[3]) * a2;
          } else {
            const double* pc = pe + c * Q * Q;
            const double d00 = pc[0 * Q3], d01 = pc[1 * Q3], d02 = pc[2 * Q3];
            const double d11 = pc[3 * Q3], d12 = pc[4 * Q3], d22 = pc[5 * Q3];
            g0[c] = fma(d02, a2, fma(d01, a1, d00 * a0));
            g1[c] = fma(d12, a2, fma(d11, a1, d01 * a0));
            g2[c] = fma(d22, a2, fma(d12, a1, d02 * a0));
          }
          if (qacc) *qacc = fma(a2, g2[c], fma(a1, g1[c], fma(a0, g0[c], *qacc)));
        }
        double w[D], w1[D];
        contract_pair<SR, Q, D, +1>(tab + Tab::TBT, g0, g1, w, w1);
#pragma unroll
        for (int k = 0; k < D; ++k) sw[LW::at(e, 0, a, b, k)] = w[k];
#pragma unroll
        for (int k = 0; k < D; ++k) sw[LW::at(e, 1, a, b, k)] = w1[k];
        contract_eo<Q, D, -1>(tab + Tab::TGT, g2, w);
#pragma unroll
        for (int k = 0; k < D; ++k) sw[LW::at(e, 2, a, b, k)] = w[k];
      } else {
        double g[Q], w[D];
        contract_eo<D, Q, +1>(tab + Tab::TB, tin[0], g);
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const double a0 = g[c];
          g[c] *= MF ? (tb.mfw[c] * wab) * tb.mfc[0] : pe[c * Q * Q];
          if (qacc) *qacc = fma(a0, g[c], *qacc);
        }
        contract_eo<Q, D, +1>(tab + Tab::TBT, g, w);
#pragma unroll
        for (int k = 0; k < D; ++k) sw[LW::at(e, 0, a, b, k)] = w[k];
      }
    }
  }

  // DR (BP1, pa_pipe.cuh): stage C's PA data in registers, loaded from global
  // at the start of the batch (latency behind stages A and B) instead of a
  // bulk copy into shared memory — D's 2 x 8q^3 bytes of shared-memory
  // traffic per element go away and the CTA needs 8Eq^3 bytes less
  static constexpr int DR_NIT = (E * Q * Q + T - 1) / T;
  struct DRegs {
    double v[DR_NIT][Q];
  };
  __device__ __forceinline__ static void load_d(const double* __restrict__ db, int ne, DRegs& r) {
    static_assert(NC == 1, "PA data in registers: one component (BP1)");
    constexpr int N = E * Q * Q;
#pragma unroll
    for (int pass = 0; pass < DR_NIT; ++pass) {
      const int t0 = threadIdx.x + pass * T;
      int e, a, b;
      line_map<LP::MC, E, Q, Q>(t0 < N ? t0 : 0, e, a, b);
      const bool act = t0 < N && e < ne;
      const double* pe = db + (act ? e : 0) * G::PS + a + Q * b;
#pragma unroll
      for (int c = 0; c < Q; ++c) r.v[pass][c] = act ? __ldcs(pe + c * Q * Q) : 0.0;
    }
  }
  __device__ __forceinline__ static void stage_c_dr(const Tab& tb, int it, const double* s0, const DRegs& r,
                                                    double* sw, int ne, double*) {
    const double* tab = tb.t[PP ? (it & 1) : 0];
    constexpr int N = E * Q * Q;
#pragma unroll
    for (int pass = 0; pass < DR_NIT; ++pass) {
      const int t0 = threadIdx.x + pass * T;
      int e, a, b;
      line_map<LP::MC, E, Q, Q>(t0 < N ? t0 : 0, e, a, b);
      const bool act = t0 < N && e < ne;
      if (!act) e = 0;
      double tin[D];
#pragma unroll
      for (int k = 0; k < D; ++k) tin[k] = s0[LT2::at(e, 0, a, b, k)];
      if constexpr (IP) __syncthreads();
      if (!act) continue;
      double g[Q], w[D];
      contract_eo<D, Q, +1>(tab + Tab::TB, tin, g);
#pragma unroll
      for (int c = 0; c < Q; ++c) g[c] *= r.v[pass][c];
      contract_eo<Q, D, +1>(tab + Tab::TBT, g, w);
#pragma unroll
      for (int k = 0; k < D; ++k) sw[LW::at(e, 0, a, b, k)] = w[k];
    }
  }

  // W (a, b, k) -> R (a, j, k): thread per line (a, k)
  __device__ __forceinline__ static void stage_d(const Tab& tb, int it, const double* sw, double* sr,
                                                 int ne, double*) {
    const double* tab = tb.t[PP ? (it & 1) : 0];
    lines<LP::MD, Q, D>(ne, [&](int e, int a, int k) {
      double wv[Q], r0[D];
#pragma unroll
      for (int b = 0; b < Q; ++b) wv[b] = sw[LW::at(e, 0, a, b, k)];
      if constexpr (NC == 3) {
        double wv2[Q], r1[D], r2[D];
#pragma unroll
        for (int b = 0; b < Q; ++b) wv2[b] = sw[LW::at(e, 2, a, b, k)];
        contract_pair<SR, Q, D, +1>(tab + Tab::TBT, wv, wv2, r0, r2);  // rG = B^T w0, B^T w2
#pragma unroll
        for (int j = 0; j < D; ++j) sr[LR::at(e, 0, a, j, k)] = r0[j];
#pragma unroll
        for (int b = 0; b < Q; ++b) wv[b] = sw[LW::at(e, 1, a, b, k)];
        contract_eo<Q, D, -1>(tab + Tab::TGT, wv, r1);  // G^T w1
#pragma unroll
        for (int j = 0; j < D; ++j) sr[LR::at(e, 1, a, j, k)] = r1[j] + r2[j];
      } else {
        contract_eo<Q, D, +1>(tab + Tab::TBT, wv, r0);  // r = B^T w
#pragma unroll
        for (int j = 0; j < D; ++j) sr[LR::at(e, 0, a, j, k)] = r0[j];
      }
    });
  }

  // stage E with the ids from a functor gid(e, l) (closed-form restriction)
  template <class GidF>
  __device__ __forceinline__ static void stage_e_ids(const Tab& tb, int it, const double* sr, GidF gid,
                                                     double* y, int ne, double*) {
    const double* tab = tb.t[PP ? (it & 1) : 0];
    lines<LP::ME, D, D>(ne, [&](int e, int j, int k) {
      const int g0 = gid(e, j, k);  // id of node (0, j, k); ids along a line are consecutive
      double rv[Q], out[D];
#pragma unroll
      for (int a = 0; a < Q; ++a) rv[a] = sr[LR::at(e, 0, a, j, k)];
      if constexpr (NC == 3) {
        double o2[D];
        contract_eo<Q, D, -1>(tab + Tab::TGT, rv, out);  // G^T rG
#pragma unroll
        for (int a = 0; a < Q; ++a) rv[a] = sr[LR::at(e, 1, a, j, k)];
        contract_eo<Q, D, +1>(tab + Tab::TBT, rv, o2);  // B^T rB
#pragma unroll
        for (int i = 0; i < D; ++i) atomicAdd(y + g0 + i, out[i] + o2[i]);
      } else {
        contract_eo<Q, D, +1>(tab + Tab::TBT, rv, out);
#pragma unroll
        for (int i = 0; i < D; ++i) atomicAdd(y + g0 + i, out[i]);
      }
    });
  }

  // staged scatter (pa_pipe.cuh YS): stage E's line outputs go to the dead W
  // region in the X-buffer layout; the pipeline then issues the RED.F64s in
  // the gather's thread -> node order (consecutive lanes on consecutive nodes
  // of a row: ~3x fewer L2 sectors per warp-wide RED than one line per lane)
  static constexpr bool YS_FITS = XS <= (IP ? P0 : P1);
  __device__ __forceinline__ static void stage_e_stage(const Tab& tb, int it, const double* sr, double* yb,
                                                       int ne, double*) {
    const double* tab = tb.t[PP ? (it & 1) : 0];
    lines<LP::ME, D, D>(ne, [&](int e, int j, int k) {
      double rv[Q], out[D];
#pragma unroll
      for (int a = 0; a < Q; ++a) rv[a] = sr[LR::at(e, 0, a, j, k)];
      if constexpr (NC == 3) {
        double o2[D];
        contract_eo<Q, D, -1>(tab + Tab::TGT, rv, out);  // G^T rG
#pragma unroll
        for (int a = 0; a < Q; ++a) rv[a] = sr[LR::at(e, 1, a, j, k)];
        contract_eo<Q, D, +1>(tab + Tab::TBT, rv, o2);  // B^T rB
#pragma unroll
        for (int i = 0; i < D; ++i) yb[LX::at(e, 0, i, j, k)] = out[i] + o2[i];
      } else {
        contract_eo<Q, D, +1>(tab + Tab::TBT, rv, out);
#pragma unroll
        for (int i = 0; i < D; ++i) yb[LX::at(e, 0, i, j, k)] = out[i];
      }
    });
  }

  // R (a, j, k) -> y (atomic scatter-add): thread per line (j, k)
  __device__ __forceinline__ static void stage_e(const Tab& tb, int it, const double* sr,
                                                 const int* gslot, double* y, int ne, double*) {
    const double* tab = tb.t[PP ? (it & 1) : 0];
    lines<LP::ME, D, D>(ne, [&](int e, int j, int k) {
      const int* g = gslot + e * G::GS + D * (j + D * k);
      double rv[Q], out[D];
#pragma unroll
      for (int a = 0; a < Q; ++a) rv[a] = sr[LR::at(e, 0, a, j, k)];
      if constexpr (NC == 3) {
        double o2[D];
        contract_eo<Q, D, -1>(tab + Tab::TGT, rv, out);  // G^T rG
#pragma unroll
        for (int a = 0; a < Q; ++a) rv[a] = sr[LR::at(e, 1, a, j, k)];
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
