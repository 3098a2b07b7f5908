// pa_inst.cu — explicit instantiation of the fused kernels for ONE order.
// Compiled once per order with -DFK_P=<p> (the build runs the eight
// compilations in parallel); each object exports fk_register_p<p>().
#include <cstring>

#include "fk_internal.h"
#include "pa_diag.cuh"
#include "pa_dfma.cuh"
#if FK_HAVE_DMMA
#include "pa_dmma.cuh"
#endif

#ifndef FK_P
#error "compile with -DFK_P=<order>"
#endif

namespace fk {
namespace {

// Launch geometry: E elements per CTA so that E*q^2 lines (stage C, the
// heaviest) fill whole warps, T = E*q^2 rounded up to a warp multiple.
constexpr int pick_E(int Q) { return (288 / (Q * Q)) > 0 ? (288 / (Q * Q)) : 1; }
constexpr int pick_T(int Q) { return ((pick_E(Q) * Q * Q + 31) / 32) * 32; }

template <int D, int Q, int NC>
void launch_dfma(const OpView& v, const double* x, double* y, int blocks, cudaStream_t s) {
  constexpr int E = pick_E(Q), T = pick_T(Q);
  Tables<D, Q> tb;
  std::memcpy(tb.B, v.B, sizeof(tb.B));
  std::memcpy(tb.G, v.G, sizeof(tb.G));
  pa_dfma_kernel<D, Q, NC, E, T><<<blocks, T, LineLayout<D, Q, NC>::smem_bytes(E), s>>>(
      tb, x, y, v.gids, v.pa, v.mask, v.nel);
}

template <int D, int Q, int NC>
void launch_diag(const OpView& v, double* diag, int64_t nel, int blocks, cudaStream_t s) {
  Tables<D, Q> tb;
  std::memcpy(tb.B, v.B, sizeof(tb.B));
  std::memcpy(tb.G, v.G, sizeof(tb.G));
  diagonal_kernel<D, Q, NC><<<blocks, 128, 0, s>>>(tb, diag, v.gids, v.pa, nel);
}

template <int D, int Q, int NC>
KernelEntry entry_dfma() {
  constexpr int E = pick_E(Q), T = pick_T(Q);
  KernelEntry k;
  k.nc = NC;
  k.d = D;
  k.q = Q;
  k.variant = FK_VARIANT_DFMA;
  k.E = E;
  k.T = T;
  k.smem = LineLayout<D, Q, NC>::smem_bytes(E);
  k.func = reinterpret_cast<const void*>(&pa_dfma_kernel<D, Q, NC, E, T>);
  k.launch = &launch_dfma<D, Q, NC>;
  k.diag = &launch_diag<D, Q, NC>;
  return k;
}

#if FK_HAVE_DMMA
template <int D, int Q, int NC>
void launch_dmma(const OpView& v, const double* x, double* y, int blocks, cudaStream_t s) {
  using K = DmmaConfig<D, Q, NC>;
  Tables<D, Q> tb;
  std::memcpy(tb.B, v.B, sizeof(tb.B));
  std::memcpy(tb.G, v.G, sizeof(tb.G));
  pa_dmma_kernel<D, Q, NC><<<blocks, K::T, K::smem_bytes(), s>>>(tb, x, y, v.gids, v.pa, v.mask,
                                                                  v.nel);
}

template <int D, int Q, int NC>
KernelEntry entry_dmma() {
  using K = DmmaConfig<D, Q, NC>;
  KernelEntry k;
  k.nc = NC;
  k.d = D;
  k.q = Q;
  k.variant = FK_VARIANT_DMMA;
  k.E = K::E;
  k.T = K::T;
  k.smem = K::smem_bytes();
  k.func = reinterpret_cast<const void*>(&pa_dmma_kernel<D, Q, NC>);
  k.launch = &launch_dmma<D, Q, NC>;
  return k;
}
#endif

}  // namespace
}  // namespace fk

#define FK_CAT2(a, b) a##b
#define FK_CAT(a, b) FK_CAT2(a, b)

extern "C++" void FK_CAT(fk_register_p, FK_P)(std::vector<fk::KernelEntry>& out) {
  constexpr int D = FK_P + 1;
  out.push_back(fk::entry_dfma<D, FK_P + 2, 3>());
  out.push_back(fk::entry_dfma<D, FK_P + 1, 3>());
  out.push_back(fk::entry_dfma<D, FK_P + 2, 1>());
  out.push_back(fk::entry_dfma<D, FK_P + 1, 1>());
#if FK_HAVE_DMMA
  out.push_back(fk::entry_dmma<D, FK_P + 2, 3>());
  out.push_back(fk::entry_dmma<D, FK_P + 2, 1>());
#endif
}
