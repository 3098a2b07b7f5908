// mix_kernels.h — registry entry of one compiled acoustic-gravity kernel
// instance (mix_inst.cu, one translation unit per order) and the C-ABI side
// (fk_mixed.cu).
#pragma once

#include <cstddef>
#include <vector>

#include <cuda_runtime.h>

#include "mix_pipe.cuh"

namespace fk {

struct MixKernel {
  int dp = 0, du = 0, q = 0, cfg = 0, E = 0, T = 0, ps = 0, gs = 0;
  size_t smem = 0, smem_mf = 0;
  const void* f_both = nullptr;
  const void* f_tau = nullptr;
  const void* f_vb = nullptr;
  const void* f_mf = nullptr;  // FusedMF apply (both blocks, no dmat traffic)
  void (*launch)(const MixKernel&, const double* Bp, const double* Gp, const double* Bu,
                 const double* w, double detj, const double* jinv, const MixArgs& a, int mode,
                 int blocks, cudaStream_t s) = nullptr;
};

enum { MIX_BOTH = 0, MIX_TAU = 1, MIX_VB = 2, MIX_BOTH_MF = 3 };
constexpr int kMixCfgs = 16;  // 0-3 geometries, 4-7 with staged outputs (YS), 8-11 with one X buffer (SX), 12-15 both

constexpr int mix_round32(int n) { return (n + 31) / 32 * 32; }
constexpr int cmax5(int a, int b, int c, int d, int e) {
  return fk::cmax(fk::cmax(a, b), fk::cmax(c, fk::cmax(d, e)));
}

// Launch geometries: E ~ EB / NMAX elements per CTA (NMAX = lines of the
// widest stage), one thread per line of the widest stage (measured: fewer
// threads, e.g. one per stage-C line, is slower at every order)

}  // namespace fk

// per-order registration (mix_inst.cu compiled with -DFK_MIX_P=2..8)
void fk_mix_register_p2(std::vector<fk::MixKernel>&);
void fk_mix_register_p3(std::vector<fk::MixKernel>&);
void fk_mix_register_p4(std::vector<fk::MixKernel>&);
void fk_mix_register_p5(std::vector<fk::MixKernel>&);
void fk_mix_register_p6(std::vector<fk::MixKernel>&);
void fk_mix_register_p7(std::vector<fk::MixKernel>&);
void fk_mix_register_p8(std::vector<fk::MixKernel>&);
