// pa_eo_ds.cuh — even-odd body with the PA data streamed through a two-slot
// ring of c-plane pairs (D_STREAM; EO cfgs 54-57, BP3 at high orders).
//
// At p >= 5 the BP3 kernels are occupancy-bound: the batch's
// whole PA data (6 q^3 doubles per element, 48 KB at p = 8) sits in shared
// memory through stage C, which caps the CTAs per SM.  Stage C's even-odd
// structure does not need it all at once: for the pair of planes
// (c, q-1-c) a line (a, b) needs its forward row c (E_c +- O_c gives the
// values at c and q-1-c), D at those two planes, and adds the folded pair
// (g'_c +- g'_{q-1-c}) into the accumulators of the transposed contraction
// (E_k += Ne[k][c] xe_c, O_k += No[k][c] xo_c).  So the pipeline keeps two
// pair slots in shared memory (pa_pipe.cuh: one bulk copy per element,
// component and plane, mbarrier per slot, the slot refilled for the pair two
// ahead — across batches — as soon as every thread has passed it).  Same
// sums as DfmaEoBody::stage_c (tensor.py:244-283), accumulated in pair order.
//
// Plane windows: a plane is q^2 doubles at e*PS + m*q^3 + c*q^2; bulk copies
// need 16-byte alignment, so for odd q a window starting one double early
// (phase (m + c) & 1, PS even) is copied and the reader skips the phase.
#pragma once

#include "pa_dfma_eo.cuh"

namespace fk {

template <int D, int Q, int NC, int E_, int T_, class LP, bool PP = true, bool SR = true>
struct EoDsBody : DfmaEoBody<D, Q, NC, E_, T_, LP, PP, SR> {
  using Base = DfmaEoBody<D, Q, NC, E_, T_, LP, PP, SR>;
  using Tab = typename Base::Tab;
  using G = GlobalLayout<D, Q, NC>;
  using LT2 = typename LP::T2;
  using LW = typename LP::W;
  static constexpr int E = E_, T = T_;
  static constexpr bool D_STREAM = true;
  static constexpr bool QF_OK = false;
  static constexpr int NPA = G::NPA, Q2 = Q * Q, Q3 = Q * Q * Q;
  static constexpr int NP = (Q + 1) / 2;              // plane pairs (the last single when q is odd)
  static constexpr int PLP = ((Q2 + 1) / 2) * 2;      // ring pitch of a plane window (even: 16 B)
  static constexpr int SLOT = E * NPA * 2 * PLP;      // doubles per ring slot
  static_assert(E * Q * Q <= T, "one stage-C line per thread");
  static_assert(Q2 % 2 == 0 || G::PS > NPA * Q3, "plane windows must stay inside the element's PA data");

  // window of plane (e, m, c): first double relative to the batch's PA base,
  // its length (doubles, even) and the reader's phase
  __device__ __forceinline__ static int win_phase(int m, int c) { return (m * Q3 + c * Q2) & 1; }
  __device__ __forceinline__ static int win_off(int e, int m, int c) {
    return e * G::PS + m * Q3 + c * Q2 - win_phase(m, c);
  }
  __device__ __forceinline__ static int win_len(int m, int c) { return (win_phase(m, c) + Q2 + 1) & ~1; }
  __device__ __forceinline__ static int slot_at(int e, int m, int h) { return ((e * NPA + m) * 2 + h) * PLP; }

  // stage C over the pairs: wait(s) -> slot base of pair s once its copies
  // landed (all threads), release(s): CTA barrier + refill (pipeline)
  template <class WaitF, class RelF>
  __device__ __forceinline__ static void stage_c_ds(const Tab& tb, int it, const double* s0, double* sw, int ne,
                                                    WaitF wait, RelF release) {
    const double* tab = tb.t[PP ? (it & 1) : 0];
    using FF = Fold<Q, D>;  // forward rows: out c, in k
    using FB = Fold<D, Q>;  // transposed rows: out k', in c
    constexpr int HF = FF::HI > 0 ? FF::HI : 1, HB = FB::HO;
    constexpr int N = E * Q * Q;
    int e, a, b;
    line_map<LP::MC, E, Q, Q>((int)threadIdx.x < N ? (int)threadIdx.x : 0, e, a, b);
    const bool act = (int)threadIdx.x < N && e < ne;
    if (!act) e = 0;
    double xe[NC][HF], xo[NC][HF], xm[NC];
#pragma unroll
    for (int s = 0; s < NC; ++s) {
      double tin[D];
#pragma unroll
      for (int k = 0; k < D; ++k) tin[k] = s0[LT2::at(e, s, a, b, k)];
      eo_fold<D>(tin, xe[s], xo[s]);
      xm[s] = tin[FF::HI < D ? FF::HI : 0];
    }
    double Ea[NC][HB], Oa[NC][HB];
#pragma unroll
    for (int s = 0; s < NC; ++s)
#pragma unroll
      for (int r = 0; r < HB; ++r) Ea[s][r] = Oa[s][r] = 0.0;
    const int ab = a + Q * b;
#pragma unroll 1
    for (int p = 0; p < NP; ++p) {
      const double* slot = wait(p);
      if (act) {
        const int c0 = p, c1 = Q - 1 - p;
        const bool two = c0 != c1;
        // forward row p: values at c0 (h = 0) and c1 (h = 1)
        double g[2][NC];
        {
          double row[FF::RL];
          ld_row(tab + Tab::TB + p * FF::RP, row);
#pragma unroll
          for (int s = 0; s < (NC == 3 ? 2 : 1); ++s) {
            double Ev, Ov;
            eo_row<D, FF::RL, FF::HI>(row, xe[s], xo[s], xm[s], Ev, Ov);
            g[0][s] = Ev + Ov;
            g[1][s] = Ev - Ov;
          }
          if constexpr (NC == 3) {
            ld_row(tab + Tab::TG + p * FF::RP, row);
            double Ev, Ov;
            eo_row<D, FF::RL, FF::HI>(row, xe[2], xo[2], xm[2], Ev, Ov);
            g[0][2] = Ev + Ov;
            g[1][2] = Ov - Ev;
          }
        }
        // D at the two planes
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two) break;
          const int c = h ? c1 : c0;
          auto dv = [&](int m) { return slot[slot_at(e, m, h) + win_phase(m, c) + ab]; };
          if constexpr (NC == 3) {
            const double a0 = g[h][0], a1 = g[h][1], a2 = g[h][2];
            const double d00 = dv(0), d01 = dv(1), d02 = dv(2), d11 = dv(3), d12 = dv(4), d22 = dv(5);
            g[h][0] = fma(d02, a2, fma(d01, a1, d00 * a0));
            g[h][1] = fma(d12, a2, fma(d11, a1, d01 * a0));
            g[h][2] = fma(d22, a2, fma(d12, a1, d02 * a0));
          } else {
            g[h][0] *= dv(0);
          }
        }
        // transposed contraction over c: fold the pair, accumulate
#pragma unroll
        for (int s = 0; s < NC; ++s) {
          const double* tt = tab + ((NC == 3 && s == 2) ? Tab::TGT : Tab::TBT);
          if (two) {
            const double ve = g[0][s] + g[1][s], vo = g[0][s] - g[1][s];
#pragma unroll
            for (int r = 0; r < HB; ++r) {
              Ea[s][r] = fma(tt[r * FB::RP + p], ve, Ea[s][r]);
              Oa[s][r] = fma(tt[r * FB::RP + FB::HI + p], vo, Oa[s][r]);
            }
          } else {  // middle plane (q odd)
#pragma unroll
            for (int r = 0; r < HB; ++r) Ea[s][r] = fma(tt[r * FB::RP + 2 * FB::HI], g[0][s], Ea[s][r]);
          }
        }
      }
      release(p);
    }
    if (!act) return;
#pragma unroll
    for (int s = 0; s < NC; ++s) {
      const bool neg = NC == 3 && s == 2;
      double w[D];
#pragma unroll
      for (int r = 0; r < HB; ++r) {
        w[r] = Ea[s][r] + Oa[s][r];
        if (r != D - 1 - r) w[D - 1 - r] = neg ? (Oa[s][r] - Ea[s][r]) : (Ea[s][r] - Oa[s][r]);
      }
#pragma unroll
      for (int k = 0; k < D; ++k) sw[LW::at(e, s, a, b, k)] = w[k];
    }
  }
};

}  // namespace fk
