// mix_inst.cu — instantiation of the acoustic-gravity kernels for ONE order
// (compiled once per order with -DFK_MIX_P=<order_p>; the build runs them in
// parallel).  Exports fk_mix_register_p<order_p>().
#include "mix_kernels.h"

#ifndef FK_MIX_P
#error "compile with -DFK_MIX_P=<order_p>"
#endif

namespace fk {
namespace {

template <int DP, int DU, int Q, int CFG>
struct MixGeom {
  static constexpr int NA = DP * DP + 3 * DU * DU, NB = Q * DP + 3 * Q * DU, NC = 2 * Q * Q;
  static constexpr int NMAX = NB > NA ? (NB > NC ? NB : NC) : (NA > NC ? NA : NC);
  static constexpr int EB = CFG == 1 ? 384 : CFG == 2 ? 96 : CFG == 3 ? 288 : 192;
  static constexpr int E = EB / NMAX > 0 ? EB / NMAX : 1;
  // one thread per line of the widest stage, the two blocks' lines of a stage
  // laid out warp-aligned (mix_pipe.cuh lines())
  static constexpr int PA_ = mix_round32(E * DP * DP) + E * 3 * DU * DU;
  static constexpr int PB_ = mix_round32(E * Q * DP) + E * 3 * Q * DU;
  static constexpr int PC_ = mix_round32(E * Q * Q) + E * Q * Q;
  static constexpr int PD_ = mix_round32(E * 3 * Q * DU) + E * Q * DP;
  static constexpr int PE_ = mix_round32(E * 3 * DU * DU) + E * DP * DP;
  static constexpr int TL = cmax5(PA_, PB_, PC_, PD_, PE_);
  static constexpr int T = mix_round32(TL) > 384 ? 384 : mix_round32(TL);
};

// cfgs 4-7: the geometries of cfgs 0-3 with staged outputs (mix_pipe.cuh YS);
// cfgs 8-11: the same geometries with one X buffer (SX); cfgs 12-15: both
template <int DP, int DU, int Q, int CFG>
void mix_launch(const MixKernel&, const double* Bp, const double* Gp, const double* Bu,
                const double* w, double detj, const double* jinv, const MixArgs& a, int mode,
                int blocks, cudaStream_t s) {
  using G = MixGeom<DP, DU, Q, CFG % 4>;
  constexpr bool YS = CFG / 4 == 1 || CFG / 4 == 3, SX = CFG / 4 >= 2;
  MixTables<DP, DU, Q> tb;
  tb.fill(Bp, Gp, Bu);
  tb.fill_mf(w, detj, jinv);
  const size_t smem = MixSmem<DP, DU, Q, G::E, false, SX>::BYTES;
  if (mode == MIX_BOTH)
    mix_pipe_kernel<DP, DU, Q, G::E, G::T, true, true, false, YS, SX><<<blocks, G::T, smem, s>>>(tb, a);
  else if (mode == MIX_TAU)
    mix_pipe_kernel<DP, DU, Q, G::E, G::T, true, false, false, YS, SX><<<blocks, G::T, smem, s>>>(tb, a);
  else if (mode == MIX_VB)
    mix_pipe_kernel<DP, DU, Q, G::E, G::T, false, true, false, YS, SX><<<blocks, G::T, smem, s>>>(tb, a);
  else
    mix_pipe_kernel<DP, DU, Q, G::E, G::T, true, true, true, YS, SX>
        <<<blocks, G::T, MixSmem<DP, DU, Q, G::E, true, SX>::BYTES, s>>>(tb, a);
}

template <int P, int CFG>
MixKernel mix_entry() {
  constexpr int DP = P + 1, DU = P, Q = P + 1;
  using G = MixGeom<DP, DU, Q, CFG % 4>;
  constexpr bool YS = CFG / 4 == 1 || CFG / 4 == 3, SX = CFG / 4 >= 2;
  using L = MixLayout<DP, DU, Q>;
  MixKernel k;
  k.dp = DP;
  k.du = DU;
  k.q = Q;
  k.cfg = CFG;
  k.E = G::E;
  k.T = G::T;
  k.ps = L::PS;
  k.gs = L::GS;
  k.smem = MixSmem<DP, DU, Q, G::E, false, SX>::BYTES;
  k.smem_mf = MixSmem<DP, DU, Q, G::E, true, SX>::BYTES;
  k.f_both = reinterpret_cast<const void*>(&mix_pipe_kernel<DP, DU, Q, G::E, G::T, true, true, false, YS, SX>);
  k.f_tau = reinterpret_cast<const void*>(&mix_pipe_kernel<DP, DU, Q, G::E, G::T, true, false, false, YS, SX>);
  k.f_vb = reinterpret_cast<const void*>(&mix_pipe_kernel<DP, DU, Q, G::E, G::T, false, true, false, YS, SX>);
  k.f_mf = reinterpret_cast<const void*>(&mix_pipe_kernel<DP, DU, Q, G::E, G::T, true, true, true, YS, SX>);
  k.launch = &mix_launch<DP, DU, Q, CFG>;
  return k;
}

template <int P>
void mix_add(std::vector<MixKernel>& v) {
  v.push_back(mix_entry<P, 0>());
  v.push_back(mix_entry<P, 1>());
  v.push_back(mix_entry<P, 2>());
  v.push_back(mix_entry<P, 3>());
  v.push_back(mix_entry<P, 4>());
  v.push_back(mix_entry<P, 5>());
  v.push_back(mix_entry<P, 6>());
  v.push_back(mix_entry<P, 7>());
  v.push_back(mix_entry<P, 8>());
  v.push_back(mix_entry<P, 9>());
  v.push_back(mix_entry<P, 10>());
  v.push_back(mix_entry<P, 11>());
  v.push_back(mix_entry<P, 12>());
  v.push_back(mix_entry<P, 13>());
  v.push_back(mix_entry<P, 14>());
  v.push_back(mix_entry<P, 15>());
}

}  // namespace
}  // namespace fk

#define FK_MCAT2(a, b) a##b
#define FK_MCAT(a, b) FK_MCAT2(a, b)

void FK_MCAT(fk_mix_register_p, FK_MIX_P)(std::vector<fk::MixKernel>& out) { fk::mix_add<FK_MIX_P>(out); }
