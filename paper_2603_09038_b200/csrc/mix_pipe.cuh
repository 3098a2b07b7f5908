// mix_pipe.cuh — fused partial-assembly apply of the acoustic-gravity block
// operator (feklab/operator.py BlockOperator, strategy FusedPA):
//
//   out_u[r, e] = su * B_u^T (sum_s D[s][r] (grad_ref p)_s)     tau block, :288-301
//   out_p     += sp * G^T (grad_ref^T (sum_r D[s][r] B_u u_r))  v block,   :303-319
//
// p: continuous H1 space of order DP-1 (global dofs, gathered/scattered
// through the E-restriction, mesh.py:130-137); u: 3 discontinuous L2
// components of order DU-1 (element blocks (3, nel, DU^3)); D = dmat
// (operator.py:105-123, 137-144) stored as 9 components [s*3+r][qp].  Both
// blocks contract the same quadrature data, so one pass reads D once (the
// paper's "Fused PA").  TAU / VB select the blocks (the composed normal
// operator apply_fused_normal, :364-387, runs VB then TAU).
//
// Dataflow per element (thread per line, even-odd folded FP64 FMA as in
// pa_dfma_eo.cuh; x, y, z = the reference's cyclic stage order):
//   A  x:  p lines (j,k) -> B_p x, G_p x          u lines (r,j,k) -> B_u x
//   B  y:  p lines (a,k) -> 3 gradient chains      u lines (r,a,k) -> B_u y
//   C  z + D + z^T, lines (a,b):
//        P phase: grad p at the points, t_r = sum_s D_sr g_s, B_u^T z -> W_u
//        U phase: u at the points,  t_s = sum_r D_sr u_r, (B_p^T,B_p^T,G_p^T) z -> W_p
//   D  y^T: u lines (r,a,k) B_u^T                   p lines (a,k): rG = B^T W0, rB = G^T W1 + B^T W2
//   E  x^T: u lines (r,j,k) B_u^T -> out_u (stores) p lines (j,k): G^T rG + B^T rB -> atomics
// Persistent CTAs with the pa_pipe.cuh prefetch pattern: the next batch's p
// gather and u block (cp.async) and gids (bulk copy, three slots) are in
// flight during the current batch, D(b+1) is bulk-copied after stage C(b).
#pragma once

#include "pa_async.cuh"
#include "pa_common.cuh"
#include "pa_dfma_eo.cuh"

namespace fk {

template <int DP, int DU, int Q>
struct __align__(16) MixTables {
  using FBp = Fold<Q, DP>;
  using FBpT = Fold<DP, Q>;
  using FBu = Fold<Q, DU>;
  using FBuT = Fold<DU, Q>;
  static constexpr int TBP = 0, TGP = FBp::SIZE, TBPT = 2 * FBp::SIZE, TGPT = TBPT + FBpT::SIZE;
  static constexpr int TBU = TGPT + FBpT::SIZE, TBUT = TBU + FBu::SIZE, SZ = TBUT + FBuT::SIZE;
  double t[SZ];
  // matrix-free factors (FusedMF): 1D weights, |J|, 1/jac_diag
  double mfw[Q + (Q & 1)];
  double mfc[4];

  void fill_mf(const double* w, double detj, const double* jinv) {
    for (int a = 0; a < Q; ++a) mfw[a] = w[a];
    mfc[0] = detj;
    for (int s = 0; s < 3; ++s) mfc[1 + s] = jinv[s];
  }

  // host: fold the reference tables (row-major q x d)
  void fill(const double* Bp, const double* Gp, const double* Bu) {
    double BpT[Q * DP], GpT[Q * DP], BuT[Q * DU];
    for (int a = 0; a < Q; ++a) {
      for (int i = 0; i < DP; ++i) {
        BpT[i * Q + a] = Bp[a * DP + i];
        GpT[i * Q + a] = Gp[a * DP + i];
      }
      for (int i = 0; i < DU; ++i) BuT[i * Q + a] = Bu[a * DU + i];
    }
    fold_table<Q, DP>(t + TBP, Bp, +1);
    fold_table<Q, DP>(t + TGP, Gp, -1);
    fold_table<DP, Q>(t + TBPT, BpT, +1);
    fold_table<DP, Q>(t + TGPT, GpT, -1);
    fold_table<Q, DU>(t + TBU, Bu, +1);
    fold_table<DU, Q>(t + TBUT, BuT, +1);
  }
};

// Strides of the intermediate buffers, word = c*CS + i1*S1 + i2*S2 + i3*S3
// with (i1, i2, i3) = (a, j, k) for T1/R and (a, b, k) for T2/W.  The
// primary template is the odd-pitch line layout; mix_layouts.cuh specialises
// it with strides searched by tools/mix_strides.py (bank-conflict-free).
template <int CS, int S1, int S2, int S3>
struct SStr {
  static constexpr int cs = CS, s1 = S1, s2 = S2, s3 = S3;
};

template <int DP, int DU, int Q>
struct MixStrides {
  static constexpr int LSP = DP | 1, LSU = DU | 1, LQ = Q | 1;
  using T1P = SStr<Q * DP * LSP, DP * LSP, 1, LSP>;
  using T1U = SStr<Q * DU * LSU, DU * LSU, 1, LSU>;
  using T2P = SStr<Q * Q * LSP, LSP, Q * LSP, 1>;
  using T2U = SStr<Q * Q * LSU, LSU, Q * LSU, 1>;
  using WP = SStr<DP * Q * LQ, LQ, 1, Q * LQ>;
  using WU = SStr<DU * Q * LQ, LQ, 1, Q * LQ>;
  using RP = SStr<DP * DP * LQ, 1, LQ, DP * LQ>;
  using RU = SStr<DU * DU * LQ, 1, LQ, DU * LQ>;
};

}  // namespace fk

#include "mix_layouts.cuh"

namespace fk {

// Shared-memory and global layouts of one (DP, DU, Q) instance.
template <int DP, int DU, int Q>
struct MixLayout {
  using St = MixStrides<DP, DU, Q>;
  static constexpr int LSP = DP | 1, LSU = DU | 1, LQ = Q | 1;
  static constexpr int DP3 = DP * DP * DP, DU3 = DU * DU * DU, Q3 = Q * Q * Q;
  // X buffers
  static constexpr int XPS = odd_up(DP * DP * LSP);
  static constexpr int XUC = DU * DU * LSU, XUS = odd_up(3 * XUC);
  __device__ __forceinline__ static int xp(int e, int i, int j, int k) { return e * XPS + i + LSP * (j + DP * k); }
  __device__ __forceinline__ static int xu(int e, int r, int i, int j, int k) {
    return e * XUS + r * XUC + i + LSU * (j + DU * k);
  }
  template <class S>
  __device__ __forceinline__ static int w(int c, int i1, int i2, int i3) {
    return c * S::cs + i1 * S::s1 + i2 * S::s2 + i3 * S::s3;
  }
  // region 1: T1p (2), T1u (3), later Wp (3), Wu (3)
  static constexpr int OFF_T1U = 2 * St::T1P::cs, OFF_WU = 3 * St::WP::cs;
  static constexpr int R1S = odd_up(cmax(2 * St::T1P::cs + 3 * St::T1U::cs, 3 * St::WP::cs + 3 * St::WU::cs));
  __device__ __forceinline__ static int t1p(int e, int s, int a, int j, int k) {
    return e * R1S + w<typename St::T1P>(s, a, j, k);
  }
  __device__ __forceinline__ static int t1u(int e, int r, int a, int j, int k) {
    return e * R1S + OFF_T1U + w<typename St::T1U>(r, a, j, k);
  }
  __device__ __forceinline__ static int wp(int e, int s, int a, int b, int k) {
    return e * R1S + w<typename St::WP>(s, a, b, k);
  }
  __device__ __forceinline__ static int wu(int e, int r, int a, int b, int k) {
    return e * R1S + OFF_WU + w<typename St::WU>(r, a, b, k);
  }
  // region 0: T2p (3), T2u (3), later Rp (2), Ru (3)
  static constexpr int OFF_T2U = 3 * St::T2P::cs, OFF_RU = 2 * St::RP::cs;
  static constexpr int R0S = odd_up(cmax(3 * St::T2P::cs + 3 * St::T2U::cs, 2 * St::RP::cs + 3 * St::RU::cs));
  __device__ __forceinline__ static int t2p(int e, int s, int a, int b, int k) {
    return e * R0S + w<typename St::T2P>(s, a, b, k);
  }
  __device__ __forceinline__ static int t2u(int e, int r, int a, int b, int k) {
    return e * R0S + OFF_T2U + w<typename St::T2U>(r, a, b, k);
  }
  __device__ __forceinline__ static int rp(int e, int s, int a, int j, int k) {
    return e * R0S + w<typename St::RP>(s, a, j, k);
  }
  __device__ __forceinline__ static int ru(int e, int r, int a, int j, int k) {
    return e * R0S + OFF_RU + w<typename St::RU>(r, a, j, k);
  }
  // staged outputs (YS), region 1 after stage D: p block (X-buffer layout)
  // then the three u blocks, node order within each
  static constexpr int YUO = XPS;
  static_assert(YUO + 3 * XUC <= R1S, "staged outputs must fit in region 1");
  __device__ __forceinline__ static int yp(int e, int i, int j, int k) { return e * R1S + i + LSP * (j + DP * k); }
  __device__ __forceinline__ static int yu(int e, int r, int i, int j, int k) {
    return e * R1S + YUO + r * XUC + i + LSU * (j + DU * k);
  }
  // global: PA data 9 components per point, int32 gather ids
  static constexpr int PS = pa_pad(((9 * Q3 + 1) / 2) * 2, Q);
  static constexpr int GS = ((DP3 + 3) / 4) * 4;
};

template <int DP, int DU, int Q, int E, bool MF = false, bool SX = false>
struct MixSmem {
  static constexpr int NXB = SX ? 1 : 2;  // X buffers (SX: the next gather lands after stage A)
  using L = MixLayout<DP, DU, Q>;
  static constexpr size_t OFF_BAR = 0;  // 1 D barrier + 3 gid barriers
  static constexpr size_t OFF_DB = 32;
  static constexpr size_t OFF_GS = OFF_DB + (MF ? 0ull : 8ull * E * L::PS);
  static constexpr size_t OFF_R0 = OFF_GS + 4ull * 3 * E * L::GS;
  static constexpr size_t OFF_R1 = OFF_R0 + 8ull * E * L::R0S;
  static constexpr size_t OFF_XP = OFF_R1 + 8ull * E * L::R1S;
  static constexpr size_t OFF_XU = OFF_XP + 8ull * NXB * E * L::XPS;
  static constexpr size_t BYTES = OFF_XU + 8ull * NXB * E * L::XUS;
};

struct MixArgs {
  const double* p;  // H1 pressure dofs (TAU input)
  const double* u;  // (3, nel, DU^3) velocity blocks (VB input)
  double* out_u;    // (3, nel, DU^3), overwritten (TAU)
  double* out_p;    // accumulated with atomics (VB)
  const int* gids;
  const double* pa;
  double su, sp;  // output scales (coupling_scale, -coupling_scale for apply)
  int nel;
};

// MF (FusedMF strategy, operator.py:280-286): no dmat traffic — stage C
// recomputes the diagonal w|J|J^-1 of the axis-aligned box from the 1D weights
// in the PA setup's operation order.
//
// YS (staged outputs): stage E writes both blocks' outputs to region 1 (T1/W,
// dead after stage D) in node order; after one barrier out_u is stored
// contiguously across the batch's elements and out_p's RED.F64s go out in
// node order — instead of one x-line per lane, where every warp-wide store /
// RED touches ~32 rows (tools/scatter_bench.cu).
//
// SX (single X buffer): the next batch's gather is issued after stage A has
// consumed this batch's X instead of at the top of the batch — half the X
// shared memory, so one more CTA fits per SM at order 4.
template <int DP, int DU, int Q, int E, int T, bool TAU, bool VB, bool MF = false, bool YS = false,
          bool SX = false>
__global__ void __launch_bounds__(T) mix_pipe_kernel(const __grid_constant__ MixTables<DP, DU, Q> tb,
                                                     const MixArgs arg) {
  using L = MixLayout<DP, DU, Q>;
  using S = MixSmem<DP, DU, Q, E, MF, SX>;
  using Tb = MixTables<DP, DU, Q>;
  constexpr int DP3 = L::DP3, DU3 = L::DU3, Q3 = L::Q3, GS = L::GS, PS = L::PS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar_d = reinterpret_cast<uint64_t*>(smem_raw + S::OFF_BAR);
  uint64_t* bar_g = bar_d + 1;
  double* db = reinterpret_cast<double*>(smem_raw + S::OFF_DB);
  int* gs = reinterpret_cast<int*>(smem_raw + S::OFF_GS);
  double* s0 = reinterpret_cast<double*>(smem_raw + S::OFF_R0);
  double* s1 = reinterpret_cast<double*>(smem_raw + S::OFF_R1);
  double* xpb = reinterpret_cast<double*>(smem_raw + S::OFF_XP);
  double* xub = reinterpret_cast<double*>(smem_raw + S::OFF_XU);
  const double* tab = tb.t;
  const int nel = arg.nel;
  const int nbatch = (nel + E - 1) / E;
  if ((int)blockIdx.x >= nbatch) return;

  if (threadIdx.x == 0) {
    mbar_init(bar_d, 1);
    for (int s = 0; s < 3; ++s) mbar_init(bar_g + s, 1);
    fence_mbar_init();
  }
  for (size_t i = threadIdx.x; i < (S::BYTES - S::OFF_R0) / 8; i += T)
    reinterpret_cast<double*>(smem_raw + S::OFF_R0)[i] = 0.0;
  __syncthreads();

  auto issue_g = [&](int b, int slot) {
    const int e0 = b * E, ne = min(E, nel - e0);
    const uint32_t bytes = 4u * ne * GS;
    mbar_expect_tx(bar_g + slot, bytes);
    bulk_g2s(gs + slot * E * GS, arg.gids + (size_t)e0 * GS, bytes, bar_g + slot);
  };
  auto issue_d = [&](int b) {
    if constexpr (MF) return;
    const int e0 = b * E, ne = min(E, nel - e0);
    const uint32_t bytes = 8u * ne * PS;
    mbar_expect_tx(bar_d, bytes);
    bulk_g2s(db, arg.pa + (size_t)e0 * PS, bytes, bar_d);
  };
  // p gather (TAU) and u block (VB) of batch b into X buffer half `h`
  auto issue_x = [&](int b, int gslot, int h) {
    const int e0 = b * E, ne = min(E, nel - e0);
    if constexpr (TAU) {
      const int* g = gs + gslot * E * GS;
      double* xp = xpb + h * E * L::XPS;
      for (int t = threadIdx.x; t < E * DP3; t += T) {
        const int e = t / DP3, l = t - e * DP3;
        double* dst = xp + L::xp(e, l % DP, (l / DP) % DP, l / (DP * DP));
        if (e < ne) cp_async8(dst, arg.p + g[e * GS + l]);
        else *dst = 0.0;
      }
    }
    if constexpr (VB) {
      double* xu = xub + h * E * L::XUS;
      for (int t = threadIdx.x; t < 3 * E * DU3; t += T) {
        const int r = t / (E * DU3), m = t - r * (E * DU3), e = m / DU3, l = m - e * DU3;
        double* dst = xu + L::xu(e, r, l % DU, (l / DU) % DU, l / (DU * DU));
        if (e < ne) cp_async8(dst, arg.u + ((size_t)r * nel + e0 + e) * DU3 + l);
        else *dst = 0.0;
      }
    }
    cp_async_commit();
  };
  uint32_t ph_g = 0u, ph_d = 0u;
  auto wait_g = [&](int slot) {
    mbar_wait(bar_g + slot, (ph_g >> slot) & 1u);
    ph_g ^= 1u << slot;
  };
  // element-major thread -> (e, line) loop over a stage's lines
  // f(e, l) over a stage's two line groups: l in [0, n1) (first block) and
  // [n1, n1 + n2) (second block).  The groups are laid out phase-major and
  // the second starts on a warp boundary, so no warp runs both code paths.
  auto lines = [&](int ne, int n1, int n2, auto f) {
    const int pad = (E * n1 + 31) & ~31;
    for (int t = threadIdx.x; t < pad + E * n2; t += T) {
      if (t < pad) {
        if (t < E * n1) {
          const int e = t / n1, l = t - e * n1;
          if (e < ne) f(e, l);
        }
      } else {
        const int m = t - pad, e = m / n2, l = n1 + (m - e * n2);
        if (e < ne) f(e, l);
      }
    }
  };
  constexpr int NAP = TAU ? DP * DP : 0, NAU = VB ? 3 * DU * DU : 0;
  constexpr int NBP = TAU ? Q * DP : 0, NBU = VB ? 3 * Q * DU : 0;
  constexpr int NCP = TAU ? Q * Q : 0, NCU = VB ? Q * Q : 0;
  constexpr int NDU = TAU ? 3 * Q * DU : 0, NDP = VB ? Q * DP : 0;

  const int stride = (int)gridDim.x;
  if (threadIdx.x == 0) {
    issue_g(blockIdx.x, 0);
    if ((int)blockIdx.x + stride < nbatch) issue_g(blockIdx.x + stride, 1);
    issue_d(blockIdx.x);
  }
  wait_g(0);
  issue_x(blockIdx.x, 0, 0);

  int it = 0;
  for (int b = blockIdx.x; b < nbatch; b += stride, ++it) {
    const int gslot = it % 3, h = it & 1;
    const int e0 = b * E, ne = min(E, nel - e0);
    const int nb = b + stride, nb2 = nb + stride;
    const double* xp = xpb + (SX ? 0 : h) * E * L::XPS;
    const double* xu = xub + (SX ? 0 : h) * E * L::XUS;
    cp_async_wait_all();
    __syncthreads();
    if (nb < nbatch) {
      if constexpr (!SX) {
        wait_g((it + 1) % 3);
        issue_x(nb, (it + 1) % 3, h ^ 1);
      }
      if (nb2 < nbatch && threadIdx.x == 0) {
        fence_proxy_async();
        issue_g(nb2, (it + 2) % 3);
      }
    }
    // ---- stage A: x contraction
    lines(ne, NAP, NAU, [&](int e, int l) {
      if (TAU && l < NAP) {
        const int j = l % DP, k = l / DP;
        double xr[DP], o[Q];
#pragma unroll
        for (int i = 0; i < DP; ++i) xr[i] = xp[L::xp(e, i, j, k)];
        contract_eo<DP, Q, +1>(tab + Tb::TBP, xr, o);
#pragma unroll
        for (int a = 0; a < Q; ++a) s1[L::t1p(e, 0, a, j, k)] = o[a];
        contract_eo<DP, Q, -1>(tab + Tb::TGP, xr, o);
#pragma unroll
        for (int a = 0; a < Q; ++a) s1[L::t1p(e, 1, a, j, k)] = o[a];
      } else if (VB) {
        const int m = l - NAP, r = m / (DU * DU), jk = m - r * (DU * DU), j = jk % DU, k = jk / DU;
        double xr[DU], o[Q];
#pragma unroll
        for (int i = 0; i < DU; ++i) xr[i] = xu[L::xu(e, r, i, j, k)];
        contract_eo<DU, Q, +1>(tab + Tb::TBU, xr, o);
#pragma unroll
        for (int a = 0; a < Q; ++a) s1[L::t1u(e, r, a, j, k)] = o[a];
      }
    });
    __syncthreads();
    if constexpr (SX) {  // X(b) consumed: gather X(b+1) into the same buffer
      if (nb < nbatch) {
        wait_g((it + 1) % 3);
        issue_x(nb, (it + 1) % 3, 0);
      }
    }
    // ---- stage B: y contraction
    lines(ne, NBP, NBU, [&](int e, int l) {
      if (TAU && l < NBP) {
        const int a = l / DP, k = l % DP;
        double bx[DP], gx[DP], c[Q];
#pragma unroll
        for (int j = 0; j < DP; ++j) {
          bx[j] = s1[L::t1p(e, 0, a, j, k)];
          gx[j] = s1[L::t1p(e, 1, a, j, k)];
        }
        contract_eo<DP, Q, +1>(tab + Tb::TBP, gx, c);  // B_y G_x
#pragma unroll
        for (int b2 = 0; b2 < Q; ++b2) s0[L::t2p(e, 0, a, b2, k)] = c[b2];
        contract_eo<DP, Q, -1>(tab + Tb::TGP, bx, c);  // G_y B_x
#pragma unroll
        for (int b2 = 0; b2 < Q; ++b2) s0[L::t2p(e, 1, a, b2, k)] = c[b2];
        contract_eo<DP, Q, +1>(tab + Tb::TBP, bx, c);  // B_y B_x
#pragma unroll
        for (int b2 = 0; b2 < Q; ++b2) s0[L::t2p(e, 2, a, b2, k)] = c[b2];
      } else if (VB) {
        const int m = l - NBP, r = m / (Q * DU), ak = m - r * (Q * DU), a = ak / DU, k = ak % DU;
        double v[DU], c[Q];
#pragma unroll
        for (int j = 0; j < DU; ++j) v[j] = s1[L::t1u(e, r, a, j, k)];
        contract_eo<DU, Q, +1>(tab + Tb::TBU, v, c);
#pragma unroll
        for (int b2 = 0; b2 < Q; ++b2) s0[L::t2u(e, r, a, b2, k)] = c[b2];
      }
    });
    __syncthreads();
    // ---- stage C: z + D + z^T (D read once for both blocks)
    if constexpr (!MF) {
      mbar_wait(bar_d, ph_d);
      ph_d ^= 1u;
    }
    lines(ne, NCP, NCU, [&](int e, int l) {
      const bool pph = TAU && l < NCP;
      const int m = pph ? l : l - NCP;
      const int a = m % Q, b2 = m / Q;
      const double* pe = MF ? nullptr : db + e * PS + a + Q * b2;
      const double wab = MF ? tb.mfw[b2] * tb.mfw[a] : 0.0;
      // dmat[s][r] at point c (9 components; MF: the box's diagonal)
      auto dm = [&](int c, int s, int r) -> double {
        if constexpr (MF) return s == r ? ((tb.mfw[c] * wab) * tb.mfc[0]) * tb.mfc[1 + s] : 0.0;
        else return pe[c * Q * Q + (s * 3 + r) * Q3];
      };
      if (TAU && pph) {
        double tin[3][DP], g0[Q], g1[Q], g2[Q];
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
          for (int k = 0; k < DP; ++k) tin[s][k] = s0[L::t2p(e, s, a, b2, k)];
        contract_eo<DP, Q, +1>(tab + Tb::TBP, tin[0], g0);
        contract_eo<DP, Q, +1>(tab + Tb::TBP, tin[1], g1);
        contract_eo<DP, Q, -1>(tab + Tb::TGP, tin[2], g2);
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const double x0 = g0[c], x1 = g1[c], x2 = g2[c];
          // t_r = sum_s D[s][r] g_s  (einsum qsr,sq->rq, operator.py:294)
          g0[c] = fma(dm(c, 2, 0), x2, fma(dm(c, 1, 0), x1, dm(c, 0, 0) * x0));
          g1[c] = fma(dm(c, 2, 1), x2, fma(dm(c, 1, 1), x1, dm(c, 0, 1) * x0));
          g2[c] = fma(dm(c, 2, 2), x2, fma(dm(c, 1, 2), x1, dm(c, 0, 2) * x0));
        }
        double w[DU];
        contract_eo<Q, DU, +1>(tab + Tb::TBUT, g0, w);
#pragma unroll
        for (int k = 0; k < DU; ++k) s1[L::wu(e, 0, a, b2, k)] = w[k];
        contract_eo<Q, DU, +1>(tab + Tb::TBUT, g1, w);
#pragma unroll
        for (int k = 0; k < DU; ++k) s1[L::wu(e, 1, a, b2, k)] = w[k];
        contract_eo<Q, DU, +1>(tab + Tb::TBUT, g2, w);
#pragma unroll
        for (int k = 0; k < DU; ++k) s1[L::wu(e, 2, a, b2, k)] = w[k];
      } else if (VB) {
        double tin[3][DU], u0[Q], u1[Q], u2[Q];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int k = 0; k < DU; ++k) tin[r][k] = s0[L::t2u(e, r, a, b2, k)];
        contract_eo<DU, Q, +1>(tab + Tb::TBU, tin[0], u0);
        contract_eo<DU, Q, +1>(tab + Tb::TBU, tin[1], u1);
        contract_eo<DU, Q, +1>(tab + Tb::TBU, tin[2], u2);
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          const double x0 = u0[c], x1 = u1[c], x2 = u2[c];
          // t_s = sum_r D[s][r] u_r  (einsum qsr,rq->sq, operator.py:316)
          u0[c] = fma(dm(c, 0, 2), x2, fma(dm(c, 0, 1), x1, dm(c, 0, 0) * x0));
          u1[c] = fma(dm(c, 1, 2), x2, fma(dm(c, 1, 1), x1, dm(c, 1, 0) * x0));
          u2[c] = fma(dm(c, 2, 2), x2, fma(dm(c, 2, 1), x1, dm(c, 2, 0) * x0));
        }
        double w[DP];
        contract_eo<Q, DP, +1>(tab + Tb::TBPT, u0, w);
#pragma unroll
        for (int k = 0; k < DP; ++k) s1[L::wp(e, 0, a, b2, k)] = w[k];
        contract_eo<Q, DP, +1>(tab + Tb::TBPT, u1, w);
#pragma unroll
        for (int k = 0; k < DP; ++k) s1[L::wp(e, 1, a, b2, k)] = w[k];
        contract_eo<Q, DP, -1>(tab + Tb::TGPT, u2, w);
#pragma unroll
        for (int k = 0; k < DP; ++k) s1[L::wp(e, 2, a, b2, k)] = w[k];
      }
    });
    __syncthreads();
    if (nb < nbatch && threadIdx.x == 0) {
      fence_proxy_async();
      issue_d(nb);
    }
    // ---- stage D: y^T
    lines(ne, NDU, NDP, [&](int e, int l) {
      if (TAU && l < NDU) {
        const int r = l / (Q * DU), ak = l - r * (Q * DU), a = ak % Q, k = ak / Q;
        double v[Q], o[DU];
#pragma unroll
        for (int b2 = 0; b2 < Q; ++b2) v[b2] = s1[L::wu(e, r, a, b2, k)];
        contract_eo<Q, DU, +1>(tab + Tb::TBUT, v, o);
#pragma unroll
        for (int j = 0; j < DU; ++j) s0[L::ru(e, r, a, j, k)] = o[j];
      } else if (VB) {
        const int m = l - NDU, a = m % Q, k = m / Q;
        double v[Q], r0[DP], r1[DP];
#pragma unroll
        for (int b2 = 0; b2 < Q; ++b2) v[b2] = s1[L::wp(e, 0, a, b2, k)];
        contract_eo<Q, DP, +1>(tab + Tb::TBPT, v, r0);  // rG = B^T W0
#pragma unroll
        for (int j = 0; j < DP; ++j) s0[L::rp(e, 0, a, j, k)] = r0[j];
#pragma unroll
        for (int b2 = 0; b2 < Q; ++b2) v[b2] = s1[L::wp(e, 1, a, b2, k)];
        contract_eo<Q, DP, -1>(tab + Tb::TGPT, v, r0);  // G^T W1
#pragma unroll
        for (int b2 = 0; b2 < Q; ++b2) v[b2] = s1[L::wp(e, 2, a, b2, k)];
        contract_eo<Q, DP, +1>(tab + Tb::TBPT, v, r1);  // B^T W2
#pragma unroll
        for (int j = 0; j < DP; ++j) s0[L::rp(e, 1, a, j, k)] = r0[j] + r1[j];
      }
    });
    __syncthreads();
    // ---- stage E: x^T, outputs
    const int* g = gs + gslot * E * GS;
    constexpr int NEU = TAU ? 3 * DU * DU : 0, NEP = VB ? DP * DP : 0;
    if constexpr (YS) {
      lines(ne, NEU, NEP, [&](int e, int l) {
        if (TAU && l < NEU) {
          const int r = l / (DU * DU), jk = l - r * (DU * DU), j = jk % DU, k = jk / DU;
          double v[Q], o[DU];
#pragma unroll
          for (int a = 0; a < Q; ++a) v[a] = s0[L::ru(e, r, a, j, k)];
          contract_eo<Q, DU, +1>(tab + Tb::TBUT, v, o);
#pragma unroll
          for (int i = 0; i < DU; ++i) s1[L::yu(e, r, i, j, k)] = o[i];
        } else if (VB) {
          const int m = l - NEU, j = m % DP, k = m / DP;
          double v[Q], o[DP], o2[DP];
#pragma unroll
          for (int a = 0; a < Q; ++a) v[a] = s0[L::rp(e, 0, a, j, k)];
          contract_eo<Q, DP, -1>(tab + Tb::TGPT, v, o);  // G^T rG
#pragma unroll
          for (int a = 0; a < Q; ++a) v[a] = s0[L::rp(e, 1, a, j, k)];
          contract_eo<Q, DP, +1>(tab + Tb::TBPT, v, o2);  // B^T rB
#pragma unroll
          for (int i = 0; i < DP; ++i) s1[L::yp(e, i, j, k)] = o[i] + o2[i];
        }
      });
      __syncthreads();
      if constexpr (TAU) {  // (3, nel, DU^3): contiguous over the batch for each r
        for (int t = threadIdx.x; t < 3 * E * DU3; t += T) {
          const int r = t / (E * DU3), m = t - r * (E * DU3), e = m / DU3, l = m - e * DU3;
          if (e < ne)
            arg.out_u[((size_t)r * nel + e0 + e) * DU3 + l] =
                arg.su * s1[L::yu(e, r, l % DU, (l / DU) % DU, l / (DU * DU))];
        }
      }
      if constexpr (VB) {
        for (int t = threadIdx.x; t < E * DP3; t += T) {
          const int e = t / DP3, l = t - e * DP3;
          if (e < ne)
            atomicAdd(arg.out_p + g[e * GS + l], arg.sp * s1[L::yp(e, l % DP, (l / DP) % DP, l / (DP * DP))]);
        }
      }
      continue;  // region 1 is next written by the next batch's stage A, after its first barrier
    }
    lines(ne, NEU, NEP, [&](int e, int l) {
      if (TAU && l < NEU) {
        const int r = l / (DU * DU), jk = l - r * (DU * DU), j = jk % DU, k = jk / DU;
        double v[Q], o[DU];
#pragma unroll
        for (int a = 0; a < Q; ++a) v[a] = s0[L::ru(e, r, a, j, k)];
        contract_eo<Q, DU, +1>(tab + Tb::TBUT, v, o);
        double* dst = arg.out_u + ((size_t)r * nel + e0 + e) * DU3 + DU * (j + DU * k);
#pragma unroll
        for (int i = 0; i < DU; ++i) dst[i] = arg.su * o[i];
      } else if (VB) {
        const int m = l - NEU, j = m % DP, k = m / DP;
        double v[Q], o[DP], o2[DP];
#pragma unroll
        for (int a = 0; a < Q; ++a) v[a] = s0[L::rp(e, 0, a, j, k)];
        contract_eo<Q, DP, -1>(tab + Tb::TGPT, v, o);  // G^T rG
#pragma unroll
        for (int a = 0; a < Q; ++a) v[a] = s0[L::rp(e, 1, a, j, k)];
        contract_eo<Q, DP, +1>(tab + Tb::TBPT, v, o2);  // B^T rB
        const int* ge = g + e * GS + DP * (j + DP * k);
#pragma unroll
        for (int i = 0; i < DP; ++i) atomicAdd(arg.out_p + ge[i], arg.sp * (o[i] + o2[i]));
      }
    });
    // the next iteration's barrier (after its cp.async wait) orders stage E
    // reads of R and of this gid slot before anything overwrites them
  }
}

}  // namespace fk
