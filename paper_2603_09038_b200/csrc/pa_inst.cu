// pa_inst.cu — explicit instantiation of the fused kernels for ONE order.
// Compiled once per order with -DFK_P=<p> (the build runs the eight
// compilations in parallel); each object exports fk_register_p<p>().
//
// Several launch geometries (elements per CTA E, threads T) are compiled per
// (kind, p, q, variant) and selectable by (variant, cfg) (fk_op_set_config,
// FK_CFG) for the tuning sweeps recorded in DESIGN.md; FK_VARIANT_AUTO picks
// the measured best per order (fk_api.cu kAutoVar*/kAutoCfg*).
#include <cstring>

#include "fk_internal.h"
#include "pa_diag.cuh"
#include "pa_dfma.cuh"
#include "pa_dfma_eo.cuh"
#include "pa_eo_layouts.cuh"
#include "pa_dmma.cuh"
#include "pa_dmma_map.cuh"
#include "pa_dmma_warp.cuh"
#include "pa_eo_bcd.cuh"
#include "pa_eo_ds.cuh"
#include "pa_eo_tpe.cuh"
#include "pa_eo_dmmac.cuh"
#include "pa_pipe.cuh"

#ifndef FK_P
#error "compile with -DFK_P=<order>"
#endif

namespace fk {
namespace {

constexpr int round32(int n) { return ((n + 31) / 32) * 32; }
// stage C (q^2 lines per element) is the heaviest: E*q^2 lines ~ 288
constexpr int base_E(int Q) { return (288 / (Q * Q)) > 0 ? (288 / (Q * Q)) : 1; }

// round-up multiplier for n / d = (umulhi(n, m) + n) >> s, exact for n < 2^31
// (Granlund-Montgomery; pa_pipe.cuh fast_div)
void div_magic(int d, unsigned& m, int& s) {
  s = 0;
  while ((1ll << s) < d) ++s;
  m = (unsigned)((((1ull << 32) * ((1ull << s) - (unsigned long long)d)) / (unsigned long long)d) + 1);
}

StructIds struct_ids(const OpView& v) {
  StructIds sid{v.nx, v.ny, v.p, (int)v.npx, (int)v.npy, (long long)v.e0, 0u, 0u, 0, 0, v.qf};
  if (v.nx > 0 && v.ny > 0) {
    div_magic(v.nx, sid.mnx, sid.snx);
    div_magic(v.ny, sid.mny, sid.sny);
  }
  return sid;
}

template <int D, int Q, int NC, class Body, bool PERSIST, bool DG, bool MF = false, int GM = 0,
          bool SX = false, bool XP = false, bool QF = false, bool YS = false, bool DR = false>
void launch_pipe(const OpView& v, const double* x, double* y, int blocks, cudaStream_t s) {
  typename Body::Tab tb;
  Body::fill(tb, v.B, v.G);
  if constexpr (MF) Body::fill_mf(tb, v.w, v.detj, v.jinv);
  const StructIds sid = struct_ids(v);
  pa_pipe_kernel<D, Q, NC, Body, PERSIST, DG, MF, GM, SX, XP, QF, YS, DR>
      <<<blocks, Body::T, PipeSmem<D, Q, NC, Body, DG || MF, GM, SX>::BYTES, s>>>(
          tb, x, y, v.gids, v.pa, v.ebits, v.nel, sid);
}

template <int D, int Q, int NC>
void launch_diag(const OpView& v, double* diag, int64_t nel, int blocks, cudaStream_t s) {
  Tables<D, Q> tb;
  std::memcpy(tb.B, v.B, sizeof(tb.B));
  std::memcpy(tb.G, v.G, sizeof(tb.G));
  diagonal_kernel<D, Q, NC><<<blocks, 128, 0, s>>>(tb, diag, v.gids, v.pa, nel);
}

template <int D, int Q, int NC, int W>
void launch_warp_dmma(const OpView& v, const double* x, double* y, int blocks, cudaStream_t s) {
  Tables<D, Q> tb;
  std::memcpy(tb.B, v.B, sizeof(tb.B));
  std::memcpy(tb.G, v.G, sizeof(tb.G));
  const StructIds sid = struct_ids(v);
  dmma_warp_kernel<D, Q, NC, W><<<blocks, 32 * W, WarpDmmaKernel<D, Q, NC, W>::SMEM, s>>>(
      tb, x, y, v.pa, v.ebits, v.nel, sid);
}

template <int D, int Q, int W, int MINB>
void launch_tpe(const OpView& v, const double* x, double* y, int blocks, cudaStream_t s) {
  FoldTables<D, Q> tb;
  DfmaEoBody<D, Q, 1, 1, 32, EoLayDefault<D, Q, 1, false>>::fill(tb, v.B, v.G);
  const StructIds sid = struct_ids(v);
  tpe_kernel<D, Q, W, MINB><<<blocks, 32 * W, TpeLayout<D, Q, W>::SMEM, s>>>(tb, x, y, v.pa, v.ebits, v.nel, sid);
}

// thread-per-element BP1 (pa_eo_tpe.cuh): closed-form ids, 32 elements per
// warp; MINB = CTAs per SM the register allocation must allow
template <int D, int Q, int W, int MINB = 1>
KernelEntry tpe_entry(int cfg) {
  KernelEntry k;
  k.nc = 1;
  k.d = D;
  k.q = Q;
  k.variant = FK_VARIANT_EO;
  k.cfg = cfg;
  k.E = 32 * W;
  k.T = 32 * W;
  k.persist = true;
  k.structured = true;
  k.smem = TpeLayout<D, Q, W>::SMEM;
  k.func = reinterpret_cast<const void*>(&tpe_kernel<D, Q, W, MINB>);
  k.launch = &launch_tpe<D, Q, W, MINB>;
  k.diag = &launch_diag<D, Q, 1>;
  k.diag_func = reinterpret_cast<const void*>(&diagonal_kernel<D, Q, 1>);
  return k;
}

// warp-per-element DMMA (pa_dmma_warp.cuh): closed-form ids, D through L2
template <int D, int Q, int NC, int W>
KernelEntry warp_dmma_entry(int cfg) {
  KernelEntry k;
  k.nc = NC;
  k.d = D;
  k.q = Q;
  k.variant = FK_VARIANT_DMMA;
  k.cfg = cfg;
  k.E = W;
  k.T = 32 * W;
  k.persist = true;
  k.structured = true;
  k.smem = WarpDmmaKernel<D, Q, NC, W>::SMEM;
  k.func = reinterpret_cast<const void*>(&dmma_warp_kernel<D, Q, NC, W>);
  k.launch = &launch_warp_dmma<D, Q, NC, W>;
  k.diag = &launch_diag<D, Q, NC>;
  k.diag_func = reinterpret_cast<const void*>(&diagonal_kernel<D, Q, NC>);
  return k;
}


// Geometries that CG may select (fk_api.cu: kAutoCfg3 / kAutoCfgMF3 for q = p+2
// and the array-map tables of the deterministic mode) get a twin instance with
// the element quadratic form compiled in (QF, CG's p.Ap); every other launch
// runs the kernel without it (measured 1-3% faster than a runtime switch).
constexpr bool qf_cfg(int variant, int cfg) {
  return variant == FK_VARIANT_EO
             ? (cfg == 1 || cfg == 2 || cfg == 11 || cfg == 14 || cfg == 18 || cfg == 23 ||
                cfg == 25 || cfg == 35)
             : variant == FK_VARIANT_MF ? (cfg == 2 || cfg == 5 || cfg == 6 || cfg == 7 || cfg == 8 ||
                                           cfg == 10)
                                        : false;
}

template <int V, int CFG, int D, int Q, int NC, class Body, bool PERSIST = true, bool DG = false,
          bool MF = false, int GM = 0, bool SX = false, bool XP = false, bool YS = false,
          bool DR = false>
KernelEntry entry() {
  constexpr int variant = V, cfg = CFG;
  KernelEntry k;
  k.nc = NC;
  k.d = D;
  k.q = Q;
  k.variant = variant;
  k.cfg = cfg;
  k.E = Body::E;
  k.T = Body::T;
  k.persist = PERSIST;
  k.structured = GM == 1;
  if constexpr (NC == 3 && Q == D + 1 && PERSIST && !DR && HasQf<Body>::value && qf_cfg(V, CFG))
  {
    k.launch_qf = &launch_pipe<D, Q, NC, Body, PERSIST, DG, MF, GM, SX, XP, true, YS, DR>;
    k.func_qf = reinterpret_cast<const void*>(&pa_pipe_kernel<D, Q, NC, Body, PERSIST, DG, MF, GM, SX, XP, true, YS, DR>);
  }
  k.smem = PipeSmem<D, Q, NC, Body, DG || MF, GM, SX>::BYTES;
  k.func = reinterpret_cast<const void*>(&pa_pipe_kernel<D, Q, NC, Body, PERSIST, DG, MF, GM, SX, XP, false, YS, DR>);
  k.launch = &launch_pipe<D, Q, NC, Body, PERSIST, DG, MF, GM, SX, XP, false, YS, DR>;
  k.diag = &launch_diag<D, Q, NC>;
  k.diag_func = reinterpret_cast<const void*>(&diagonal_kernel<D, Q, NC>);
  return k;
}

template <int D, int Q, int NC, int E, bool IP, bool PP, bool SR = true>
using TunedEo =
    DfmaEoBody<D, Q, NC, E, round32(E * Q * Q), EoLayTuned<D, Q, NC, E, round32(E * Q * Q), IP>, PP, SR>;

// nine tuned even-odd geometries from cfg c0: (E2, E1) x (smem D, D via L2) x
// (W over T1, W over T2), then E0 in place
template <int D, int Q, int NC, bool PP, int C0>
void add_tuned_eo(std::vector<KernelEntry>& out) {
  constexpr int E0 = base_E(Q);
  constexpr int E1 = E0 / 2 > 0 ? E0 / 2 : 1;
  constexpr int E2 = E0 / 4 > 0 ? E0 / 4 : 1;
  out.push_back(entry<FK_VARIANT_EO, C0 + 0, D, Q, NC, TunedEo<D, Q, NC, E2, false, PP>, true>());
  out.push_back(entry<FK_VARIANT_EO, C0 + 1, D, Q, NC, TunedEo<D, Q, NC, E1, false, PP>, true>());
  out.push_back(entry<FK_VARIANT_EO, C0 + 2, D, Q, NC, TunedEo<D, Q, NC, E2, false, PP>, true, true>());
  out.push_back(entry<FK_VARIANT_EO, C0 + 3, D, Q, NC, TunedEo<D, Q, NC, E1, false, PP>, true, true>());
  out.push_back(entry<FK_VARIANT_EO, C0 + 4, D, Q, NC, TunedEo<D, Q, NC, E2, true, PP>, true>());
  out.push_back(entry<FK_VARIANT_EO, C0 + 5, D, Q, NC, TunedEo<D, Q, NC, E1, true, PP>, true>());
  out.push_back(entry<FK_VARIANT_EO, C0 + 6, D, Q, NC, TunedEo<D, Q, NC, E2, true, PP>, true, true>());
  out.push_back(entry<FK_VARIANT_EO, C0 + 7, D, Q, NC, TunedEo<D, Q, NC, E1, true, PP>, true, true>());
  out.push_back(entry<FK_VARIANT_EO, C0 + 8, D, Q, NC, TunedEo<D, Q, NC, E0, true, PP>, true>());
}

// Compiled launch geometries (cfg index per variant), measured per order in
// the sweeps (profiles/r01_sweep_*).
template <int D, int Q, int NC>
void add_all(std::vector<KernelEntry>& out) {
  constexpr int E0 = base_E(Q);
  constexpr int E1 = E0 / 2 > 0 ? E0 / 2 : 1;
  constexpr int E2 = E0 / 4 > 0 ? E0 / 4 : 1;
  using F1 = DfmaBody<D, Q, NC, E1, round32(E1 * Q * Q), 1>;
  using F2 = DfmaBody<D, Q, NC, E2, round32(E2 * Q * Q), 1>;
  using F1x2 = DfmaBody<D, Q, NC, E1, round32((E1 * Q * Q + 1) / 2), 2>;
  out.push_back(entry<FK_VARIANT_DFMA, 0, D, Q, NC, F2, true>());
  out.push_back(entry<FK_VARIANT_DFMA, 1, D, Q, NC, F1, true>());
  out.push_back(entry<FK_VARIANT_DFMA, 2, D, Q, NC, F2, true, true>());   // D via L2, not smem
  out.push_back(entry<FK_VARIANT_DFMA, 3, D, Q, NC, F1, true, true>());
  out.push_back(entry<FK_VARIANT_DFMA, 4, D, Q, NC, F1x2, true>());       // 2 lines per thread
  out.push_back(entry<FK_VARIANT_DFMA, 5, D, Q, NC, F2, false>());        // one batch per CTA
  out.push_back(entry<FK_VARIANT_DMMA, 0, D, Q, NC, DmmaBody<D, Q, NC, E1, 128>, true>());
  out.push_back(entry<FK_VARIANT_DMMA, 1, D, Q, NC, DmmaBody<D, Q, NC, E0, 256>, true>());
  out.push_back(entry<FK_VARIANT_DMMA, 2, D, Q, NC, DmmaBody<D, Q, NC, E1, 128>, true, true>());
  // cfgs 6-8: smaller footprints for occupancy (D via L2): one element per CTA
  // with 4 or 8 warps, two elements with 8 warps
  out.push_back(entry<FK_VARIANT_DMMA, 6, D, Q, NC, DmmaBody<D, Q, NC, 1, 128>, true, true>());
  out.push_back(entry<FK_VARIANT_DMMA, 7, D, Q, NC, DmmaBody<D, Q, NC, 1, 256>, true, true>());
  out.push_back(entry<FK_VARIANT_DMMA, 8, D, Q, NC, DmmaBody<D, Q, NC, E1, 256>, true, true>());
  // cfgs 12-14: even-odd FMA stages A, B, D, E with stage C on DMMA
  // (pa_eo_dmmac.cuh; d, q <= 8): E2 / E1 array-map geometries and the
  // closed-form single-X precomputed-gather geometry of eo33
  if constexpr (D <= 8 && Q <= 8) {
    constexpr int E0c = base_E(Q);
    constexpr int E1c = E0c / 2 > 0 ? E0c / 2 : 1;
    constexpr int E2c = E0c / 4 > 0 ? E0c / 4 : 1;
    using HC2 = EoDmmaCBody<D, Q, NC, E2c, round32(E2c * Q * Q),
                            EoLayTuned<D, Q, NC, E2c, round32(E2c * Q * Q), false>, false>;
    using HC1 = EoDmmaCBody<D, Q, NC, E1c, round32(E1c * Q * Q),
                            EoLayTuned<D, Q, NC, E1c, round32(E1c * Q * Q), false>, false>;
    using HC2s = EoDmmaCBody<D, Q, NC, E2c, round32(E2c * Q * Q),
                             EoLayTuned<D, Q, NC, E2c, round32(E2c * Q * Q), false>, true, false>;
    out.push_back(entry<FK_VARIANT_DMMA, 12, D, Q, NC, HC2, true>());
    out.push_back(entry<FK_VARIANT_DMMA, 13, D, Q, NC, HC1, true>());
    out.push_back(entry<FK_VARIANT_DMMA, 14, D, Q, NC, HC2s, true, false, false, 1, true, true>());
  }
  // cfgs 9-11: one warp per element, stages chained in registers (d, q <= 8)
  if constexpr (D <= 8 && Q <= 8) {
    out.push_back(warp_dmma_entry<D, Q, NC, 4>(9));
    out.push_back(warp_dmma_entry<D, Q, NC, 8>(10));
    out.push_back(warp_dmma_entry<D, Q, NC, 2>(11));
  }
  // cfgs 3-5: the paper's per-element DMMA dataflow on the reference's shipped
  // conflict-free tile maps (pa_dmma_map.cuh): p = 3, q = 5 only, 1 / 2 / 4
  // elements (4 warps each) per CTA
  if constexpr (D == 4 && Q == 5) {
    out.push_back(entry<FK_VARIANT_DMMA, 3, D, Q, NC, DmmaMapBody<NC, 1>, true>());
    out.push_back(entry<FK_VARIANT_DMMA, 4, D, Q, NC, DmmaMapBody<NC, 2>, true>());
    out.push_back(entry<FK_VARIANT_DMMA, 5, D, Q, NC, DmmaMapBody<NC, 4>, true>());
  }
  using F0 = DfmaBody<D, Q, NC, E0, round32(E0 * Q * Q), 1>;
  out.push_back(entry<FK_VARIANT_DFMA, 6, D, Q, NC, F0, true>());
  // even-odd bodies.  cfg 0: the line layout of the first EO kernels (reference
  // point); cfgs 1-9: smem layouts searched by tools/smem_strides.py
  // (pa_eo_layouts.cuh) with ping-pong tables; cfgs 10-18: the same with a
  // static table copy (see DfmaEoBody PP).
  using O2 = DfmaEoBody<D, Q, NC, E2, round32(E2 * Q * Q), EoLayDefault<D, Q, NC, false>>;
  out.push_back(entry<FK_VARIANT_EO, 0, D, Q, NC, O2, true>());
  add_tuned_eo<D, Q, NC, true, 1>(out);
  add_tuned_eo<D, Q, NC, false, 10>(out);
  // closed-form restriction (no id traffic, 1 int per element per slot) with a
  // single X buffer: less smem per CTA -> more CTAs per SM
  out.push_back(entry<FK_VARIANT_EO, 19, D, Q, NC, TunedEo<D, Q, NC, E2, true, true>, true, false, false, 1, true>());
  out.push_back(entry<FK_VARIANT_EO, 20, D, Q, NC, TunedEo<D, Q, NC, E2, false, true>, true, false, false, 1, true>());
  out.push_back(entry<FK_VARIANT_EO, 21, D, Q, NC, TunedEo<D, Q, NC, E2, true, true>, true, false, false, 1, false>());
  out.push_back(entry<FK_VARIANT_EO, 22, D, Q, NC, TunedEo<D, Q, NC, E2, true, false>, true, false, false, 1, true>());
  out.push_back(entry<FK_VARIANT_EO, 23, D, Q, NC, TunedEo<D, Q, NC, E1, false, false>, true, false, false, 1, true>());
  out.push_back(entry<FK_VARIANT_EO, 24, D, Q, NC, TunedEo<D, Q, NC, E0, true, false>, true, false, false, 1, true>());
  // cfgs 25-31: cfgs 2, 10, 14, 18, 19, 23, 24 with the gather slots precomputed (XP)
  out.push_back(entry<FK_VARIANT_EO, 25, D, Q, NC, TunedEo<D, Q, NC, E1, false, true>, true, false, false, 0, false, true>());
  out.push_back(entry<FK_VARIANT_EO, 26, D, Q, NC, TunedEo<D, Q, NC, E2, false, false>, true, false, false, 0, false, true>());
  out.push_back(entry<FK_VARIANT_EO, 27, D, Q, NC, TunedEo<D, Q, NC, E2, true, false>, true, false, false, 0, false, true>());
  out.push_back(entry<FK_VARIANT_EO, 28, D, Q, NC, TunedEo<D, Q, NC, E0, true, false>, true, false, false, 0, false, true>());
  out.push_back(entry<FK_VARIANT_EO, 29, D, Q, NC, TunedEo<D, Q, NC, E2, true, true>, true, false, false, 1, true, true>());
  out.push_back(entry<FK_VARIANT_EO, 30, D, Q, NC, TunedEo<D, Q, NC, E1, false, false>, true, false, false, 1, true, true>());
  out.push_back(entry<FK_VARIANT_EO, 31, D, Q, NC, TunedEo<D, Q, NC, E0, true, false>, true, false, false, 1, true, true>());
  // cfg 32: cfg 29 with separate table-row loads per component (SR off)
  out.push_back(entry<FK_VARIANT_EO, 32, D, Q, NC, TunedEo<D, Q, NC, E2, true, true, false>, true, false, false, 1, true, true>());
  // cfgs 33-35: more SR-off closed-form geometries (33: W over T1; 34: two X
  // buffers; 35: E1 elements per CTA, the BP3 p=4 default)
  out.push_back(entry<FK_VARIANT_EO, 33, D, Q, NC, TunedEo<D, Q, NC, E2, false, true, false>, true, false, false, 1, true, true>());
  out.push_back(entry<FK_VARIANT_EO, 34, D, Q, NC, TunedEo<D, Q, NC, E2, true, true, false>, true, false, false, 1, false, true>());
  out.push_back(entry<FK_VARIANT_EO, 35, D, Q, NC, TunedEo<D, Q, NC, E1, true, true, false>, true, false, false, 1, true, true>());
  // cfgs 36-39: one-warp CTAs (T = 32): a CTA barrier is one warp's, up to 32
  // CTAs per SM hide each other's latency; lines over E = 1 / 2 / 4 elements
  // in several passes (layouts searched for T = 32, pa_eo_layouts.cuh);
  // closed-form ids, single X, precomputed gather as cfg 30
  if constexpr (Q == D + 1) {
    using W1 = DfmaEoBody<D, Q, NC, 1, 32, EoLayTuned<D, Q, NC, 1, 32, false>, false>;
    out.push_back(entry<FK_VARIANT_EO, 36, D, Q, NC, W1, true, false, false, 1, true, true>());
    if constexpr (NC == 1) {
      using W2 = DfmaEoBody<D, Q, NC, 2, 32, EoLayTuned<D, Q, NC, 2, 32, false>, false>;
      using W4 = DfmaEoBody<D, Q, NC, 4, 32, EoLayTuned<D, Q, NC, 4, 32, false>, false>;
      out.push_back(entry<FK_VARIANT_EO, 37, D, Q, NC, W2, true, false, false, 1, true, true>());
      out.push_back(entry<FK_VARIANT_EO, 38, D, Q, NC, W4, true, false, false, 1, true, true>());
      // 39: E = 2 with two X buffers (next gather issued before stage A)
      out.push_back(entry<FK_VARIANT_EO, 39, D, Q, NC, W2, true, false, false, 1, false, true>());
    }
  }
  // cfgs 40-45: staged scatter (YS) twins of cfgs 30, 35, 23, 24, 31, 29 —
  // stage E's outputs through shared memory so the RED.F64s go out in node
  // order (tools/scatter_bench.cu: 300 vs 154 G RED/s at p = 4); geometries
  // whose X layout does not fit in the W region are not compiled
  if constexpr (Q == D + 1) {
    using Y30 = TunedEo<D, Q, NC, E1, false, false>;
    using Y35 = TunedEo<D, Q, NC, E1, true, true, false>;
    using Y24 = TunedEo<D, Q, NC, E0, true, false>;
    using Y29 = TunedEo<D, Q, NC, E2, true, true>;
    if constexpr (Y30::YS_FITS) {
      out.push_back(entry<FK_VARIANT_EO, 40, D, Q, NC, Y30, true, false, false, 1, true, true, true>());
      out.push_back(entry<FK_VARIANT_EO, 42, D, Q, NC, Y30, true, false, false, 1, true, false, true>());
    }
    if constexpr (Y35::YS_FITS)
      out.push_back(entry<FK_VARIANT_EO, 41, D, Q, NC, Y35, true, false, false, 1, true, true, true>());
    if constexpr (Y24::YS_FITS) {
      out.push_back(entry<FK_VARIANT_EO, 43, D, Q, NC, Y24, true, false, false, 1, true, false, true>());
      out.push_back(entry<FK_VARIANT_EO, 44, D, Q, NC, Y24, true, false, false, 1, true, true, true>());
    }
    if constexpr (Y29::YS_FITS)
      out.push_back(entry<FK_VARIANT_EO, 45, D, Q, NC, Y29, true, false, false, 1, true, true, true>());
    // cfgs 46-49 (BP1): cfgs 40, 41, 43, 44 with stage C's PA data loaded
    // into registers at the start of the batch (DR) instead of bulk-copied to
    // shared memory
    if constexpr (NC == 1) {
      if constexpr (Y30::YS_FITS)
        out.push_back(entry<FK_VARIANT_EO, 46, D, Q, NC, Y30, true, true, false, 1, true, true, true, true>());
      if constexpr (Y35::YS_FITS)
        out.push_back(entry<FK_VARIANT_EO, 47, D, Q, NC, Y35, true, true, false, 1, true, true, true, true>());
      if constexpr (Y24::YS_FITS) {
        out.push_back(entry<FK_VARIANT_EO, 48, D, Q, NC, Y24, true, true, false, 1, true, false, true, true>());
        out.push_back(entry<FK_VARIANT_EO, 49, D, Q, NC, Y24, true, true, false, 1, true, true, true, true>());
      }
    }
  }
  // cfgs 50-53 (BP1): stages B, C, D fused in registers (pa_eo_bcd.cuh), E =
  // 4 / 8 / 16 / 2 elements per CTA, one thread per (element, a) slab; staged
  // scatter, closed-form ids, single X, precomputed gather
  if constexpr (NC == 1 && Q == D + 1) {
    using B4 = EoBcdBody<D, Q, 4, round32(4 * Q)>;
    using B8 = EoBcdBody<D, Q, 8, round32(8 * Q)>;
    using B16 = EoBcdBody<D, Q, 16, round32(16 * Q)>;
    using B2 = EoBcdBody<D, Q, 2, round32(2 * Q)>;
    out.push_back(entry<FK_VARIANT_EO, 50, D, Q, NC, B4, true, false, false, 1, true, true, true>());
    out.push_back(entry<FK_VARIANT_EO, 51, D, Q, NC, B8, true, false, false, 1, true, true, true>());
    out.push_back(entry<FK_VARIANT_EO, 52, D, Q, NC, B16, true, false, false, 1, true, true, true>());
    out.push_back(entry<FK_VARIANT_EO, 53, D, Q, NC, B2, true, false, false, 1, true, true, true>());
  }
  // cfgs 54-57 (BP3, p >= 4): PA data streamed through a two-slot ring of
  // c-plane pairs (pa_eo_ds.cuh) instead of the batch's whole D in shared
  // memory: 54 / 55 one element per CTA (W over T1 / in place), 56 two
  // elements, 57 = 54 without the precomputed gather
  if constexpr (NC == 3 && Q == D + 1 && D >= 5) {
    constexpr int T1e = round32(Q * Q), T2e = round32(2 * Q * Q);
    using S54 = EoDsBody<D, Q, NC, 1, T1e, EoLayTuned<D, Q, NC, 1, T1e, false>, false>;
    using S55 = EoDsBody<D, Q, NC, 1, T1e, EoLayTuned<D, Q, NC, 1, T1e, true>, false>;
    using S56 = EoDsBody<D, Q, NC, 2, T2e, EoLayTuned<D, Q, NC, 2, T2e, false>, false>;
    out.push_back(entry<FK_VARIANT_EO, 54, D, Q, NC, S54, true, false, false, 1, true, true>());
    out.push_back(entry<FK_VARIANT_EO, 55, D, Q, NC, S55, true, false, false, 1, true, true>());
    out.push_back(entry<FK_VARIANT_EO, 56, D, Q, NC, S56, true, false, false, 1, true, true>());
    out.push_back(entry<FK_VARIANT_EO, 57, D, Q, NC, S54, true, false, false, 1, true, false>());
  }
  // cfgs 58-61 (BP1, p <= 2): one thread per element, all stages in
  // registers (pa_eo_tpe.cuh), 4 / 2 warps per CTA; 60-61 with the register
  // allocation capped for 3 / 6 CTAs per SM
  if constexpr (NC == 1 && Q == D + 1 && D <= 3) {
    out.push_back(tpe_entry<D, Q, 4>(58));
    out.push_back(tpe_entry<D, Q, 2>(59));
    out.push_back(tpe_entry<D, Q, 4, 3>(60));  // registers capped for 3 CTAs (12 warps) per SM
    out.push_back(tpe_entry<D, Q, 2, 6>(61));
  }
  // p = 3: T2 is 100 doubles per thread; 2 / 1 warps per CTA (33 KB of PA
  // slots per warp)
  if constexpr (NC == 1 && Q == D + 1 && D == 4) {
    out.push_back(tpe_entry<D, Q, 2>(58));
    out.push_back(tpe_entry<D, Q, 1>(59));
  }
  // matrix-free (FK_VARIANT_MF): even-odd tuned bodies, D recomputed in stage C
  using M2 = TunedEo<D, Q, NC, E2, false, true>;
  using M1 = TunedEo<D, Q, NC, E1, false, true>;
  using M2i = TunedEo<D, Q, NC, E2, true, true>;
  using M0i = TunedEo<D, Q, NC, E0, true, true>;
  using M2s = TunedEo<D, Q, NC, E2, false, false>;
  using M1s = TunedEo<D, Q, NC, E1, false, false>;
  using M2is = TunedEo<D, Q, NC, E2, true, false>;
  using M0is = TunedEo<D, Q, NC, E0, true, false>;
  out.push_back(entry<FK_VARIANT_MF, 0, D, Q, NC, M2, true, false, true>());
  out.push_back(entry<FK_VARIANT_MF, 1, D, Q, NC, M1, true, false, true>());
  out.push_back(entry<FK_VARIANT_MF, 2, D, Q, NC, M2i, true, false, true>());
  out.push_back(entry<FK_VARIANT_MF, 3, D, Q, NC, M0i, true, false, true>());
  out.push_back(entry<FK_VARIANT_MF, 4, D, Q, NC, M2s, true, false, true>());
  out.push_back(entry<FK_VARIANT_MF, 5, D, Q, NC, M1s, true, false, true>());
  out.push_back(entry<FK_VARIANT_MF, 6, D, Q, NC, M2is, true, false, true>());
  out.push_back(entry<FK_VARIANT_MF, 7, D, Q, NC, M0is, true, false, true>());
  // mf8-9: closed-form ids (GM 1) and precomputed gather slots (XP); with the
  // static-table three-component bodies XP costs registers, so BP1 only gains
  // (profiles/r01_sweep_v20_mf_xp.jsonl)
  out.push_back(entry<FK_VARIANT_MF, 8, D, Q, NC, M1s, true, false, true, 1, false, true>());
  out.push_back(entry<FK_VARIANT_MF, 9, D, Q, NC, M0is, true, false, true, 1, false, true>());
  // mf10: the BP3 p=4 PA default's body (cfg 35) without the PA stream
  out.push_back(entry<FK_VARIANT_MF, 10, D, Q, NC, TunedEo<D, Q, NC, E1, true, true, false>, true, false, true, 1, true, true>());
}

}  // namespace
}  // namespace fk

#define FK_CAT2(a, b) a##b
#define FK_CAT(a, b) FK_CAT2(a, b)

void FK_CAT(fk_register_p, FK_P)(std::vector<fk::KernelEntry>& out) {
  constexpr int D = FK_P + 1;
  fk::add_all<D, FK_P + 2, 3>(out);
  fk::add_all<D, FK_P + 2, 1>(out);
  fk::add_all<D, FK_P + 1, 3>(out);
  fk::add_all<D, FK_P + 1, 1>(out);
}
