// fk_cg.cuh — device-resident Jacobi-PCG pieces (MFEM CGSolver semantics).
//
// All scalars stay on the device; one iteration is
//   apply(p -> Ap), with den = p.Ap formed inside the fused kernel as the sum
//     of element quadratic forms g^T D g at the quadrature points (EO bodies;
//     other kernels: a dot pass) ; alpha = nom/den
//   r -= alpha Ap ; bn = r.(dinv r)                   (one pass, z not stored)
//   hist[it] = sqrt(bn) ; beta = bn/nom ; nom = bn
//   x += alpha p ; p = dinv r + beta p                (one pass)
// and is captured once into a CUDA graph that is replayed `iters` times.
// Vector traffic per iteration: 32 + 48 B/dof (was 16 + 64 + 24 with the
// separate dot, the stored z and the x update in the residual pass).
// Reductions are deterministic: fixed grid, fixed per-block order, the last
// block to finish sums the block partials in index order.
#pragma once

#include <cstdint>

namespace fk {

enum ScalarSlot { S_NOM = 0, S_DEN = 1, S_BN = 2, S_STOP = 3, S_ALPHA = 4, S_BETA = 5, S_DOT = 6 };
enum IntSlot { I_DONE = 0, I_IT = 1, I_ACT = 2 };  // I_ACT: this iteration updates x, r

constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Block-reduce v; block partial to partials[blockIdx.x]; the last block sums
// the partials in order and writes *out (then resets the counter).
__device__ __forceinline__ void reduce_finish(double v, double* partials, unsigned* counter,
                                              double* out) {
  __shared__ double sw[kRedThreads / 32];
  __shared__ bool last;
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sw[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kRedThreads / 32; ++i) s += sw[i];
    partials[blockIdx.x] = s;
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double s = 0.0;
    if (threadIdx.x < 32) {
      // fixed order: lane l sums partials l, l+32, ... then a fixed shuffle tree
      for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) s += ((volatile double*)partials)[i];
      s = warp_sum(s);
      if (threadIdx.x == 0) {
        *out = s;
        *counter = 0u;
      }
    }
  }
}

__global__ void __launch_bounds__(kRedThreads) dot_kernel(const double* __restrict__ a,
                                                          const double* __restrict__ b,
                                                          int64_t n0, int64_t n1,
                                                          double* partials, unsigned* counter,
                                                          double* out) {
  double s = 0.0;
  for (int64_t i = n0 + blockIdx.x * (int64_t)kRedThreads + threadIdx.x; i < n1;
       i += (int64_t)gridDim.x * kRedThreads)
    s = fma(a[i], b[i], s);
  reduce_finish(s, partials, counter, out);
}

// x = 0, r = b, p = dinv*b; partial r.(dinv r) over [n0, n1)
__global__ void __launch_bounds__(kRedThreads) cg_init_kernel(
    const double* __restrict__ b, double* __restrict__ x, double* __restrict__ r,
    double* __restrict__ p, const double* __restrict__ dinv, int64_t n, int64_t n0,
    double* partials, unsigned* counter, double* out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kRedThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kRedThreads) {
    const double bi = b[i], zi = dinv[i] * bi;
    x[i] = 0.0;
    r[i] = bi;
    p[i] = zi;
    if (i >= n0) s = fma(bi, zi, s);
  }
  reduce_finish(s, partials, counter, out);
}

// *out = sum of the n per-CTA quadratic-form partials, fixed order (one CTA)
__global__ void __launch_bounds__(kRedThreads) qf_sum_kernel(const double* __restrict__ part,
                                                             int64_t n, double* out) {
  __shared__ double sw[kRedThreads / 32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kRedThreads) s += part[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) t += sw[w];
    *out = t;
  }
}

__global__ void cg_start_kernel(double* scal, int* iscal, double* hist, double rtol) {
  const double nom = scal[S_NOM];
  hist[0] = sqrt(nom);
  scal[S_STOP] = rtol * rtol * nom;
  iscal[I_IT] = 0;
  // MFEM CGSolver: converged when nom <= max(rtol^2 nom0, abs_tol^2), abs_tol
  // = 0 — an exactly zero residual stops even with rtol = 0
  iscal[I_DONE] = (nom <= rtol * rtol * nom) ? 1 : 0;
}

__global__ void cg_alpha_kernel(double* scal, int* iscal) {
  iscal[I_ACT] = 0;
  if (iscal[I_DONE]) return;
  const double den = scal[S_DEN];
  if (den == 0.0) {  // MFEM breaks on p.Ap == 0 (no 0/0 update)
    iscal[I_DONE] = 1;
    return;
  }
  scal[S_ALPHA] = scal[S_NOM] / den;
  iscal[I_ACT] = 1;
}

// r -= alpha Ap ; partial r.(dinv r) over [n0, n)
__global__ void __launch_bounds__(kRedThreads) cg_residual_kernel(
    double* __restrict__ r, const double* __restrict__ Ap, const double* __restrict__ dinv,
    int64_t n, int64_t n0, const double* scal, const int* iscal, double* partials,
    unsigned* counter, double* out) {
  if (!iscal[I_ACT]) return;  // uniform across the grid
  const double alpha = scal[S_ALPHA];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kRedThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kRedThreads) {
    const double ri = fma(-alpha, Ap[i], r[i]);
    r[i] = ri;
    if (i >= n0) s = fma(ri, dinv[i] * ri, s);
  }
  reduce_finish(s, partials, counter, out);
}

__global__ void cg_finish_kernel(double* scal, int* iscal, double* hist) {
  if (iscal[I_DONE]) return;
  const double bn = scal[S_BN];
  const int it = iscal[I_IT] + 1;
  iscal[I_IT] = it;
  hist[it] = sqrt(bn);
  scal[S_BETA] = bn / scal[S_NOM];
  scal[S_NOM] = bn;
  if (bn <= scal[S_STOP]) iscal[I_DONE] = 1;
}

// x += alpha p (this iteration ran) ; p = dinv r + beta p (unless converged)
__global__ void cg_step_kernel(double* __restrict__ x, double* __restrict__ p,
                               const double* __restrict__ r, const double* __restrict__ dinv,
                               int64_t n, const double* scal, const int* iscal) {
  if (!iscal[I_ACT]) return;
  const double alpha = scal[S_ALPHA], beta = scal[S_BETA];
  const bool dir = !iscal[I_DONE];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double pi = p[i];
    x[i] = fma(alpha, pi, x[i]);
    if (dir) p[i] = fma(beta, pi, dinv[i] * r[i]);
  }
}

// ---- closed-form Jacobi on the box (fk_op_diagonal's box path, fk_setup.cuh) ----
// diag(gi, gj, gk) = sum_s c_s F^x_s(gi) F^y_s(gj) F^z_s(gk) from host-built
// 1D factor tables (the z table assembled over the GLOBAL element layers, so
// shared planes need no exchange and every rank holds the same bits), with
// every product and sum rounded separately (no FMA contraction: the result
// does not depend on the compiler's choices); 1 on the essential (box-face)
// dofs.  (Computing dinv inside the CG passes from these tables instead of
// reading a dinv vector was measured slower: the FP64 division and the index
// decomposition cost more than the 16 B/dof they save.)
struct BoxDiag {
  const double* tab;  // [FBx FGx | FBy FGy | FBz FGz], z over the rank's planes
  int npx, npy, npz;  // local planes
  int nc;
  double c0, c1, c2, cm;
  int dirichlet;
  int z0p, npzg;      // first global plane of the rank, global planes
  unsigned mx, my;    // fast division by npx, npy (pa_pipe.cuh fast_div)
  int sx, sy;
};

__device__ __forceinline__ double box_diag_at(const BoxDiag& b, int i, int j, int k) {
  const double* bx = b.tab;
  const double* gx = bx + b.npx;
  const double* by = gx + b.npx;
  const double* gy = by + b.npy;
  const double* bz = gy + b.npy;
  const double* gz = bz + b.npz;
  if (b.nc == 3) {
    const double t0 = __dmul_rn(b.c0, __dmul_rn(__dmul_rn(gx[i], by[j]), bz[k]));
    const double t1 = __dmul_rn(b.c1, __dmul_rn(__dmul_rn(bx[i], gy[j]), bz[k]));
    const double t2 = __dmul_rn(b.c2, __dmul_rn(__dmul_rn(bx[i], by[j]), gz[k]));
    return __dadd_rn(__dadd_rn(t0, t1), t2);
  }
  return __dmul_rn(b.cm, __dmul_rn(__dmul_rn(bx[i], by[j]), bz[k]));
}

__device__ __forceinline__ bool box_ess(const BoxDiag& b, int i, int j, int k) {
  if (!b.dirichlet) return false;
  const int kg = b.z0p + k;
  return i == 0 || i == b.npx - 1 || j == 0 || j == b.npy - 1 || kg == 0 || kg == b.npzg - 1;
}

__global__ void diag_box_rn_kernel(double* __restrict__ diag, const BoxDiag b, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int tt = (int)t;
    const int row = (int)((__umulhi((unsigned)tt, b.mx) + (unsigned)tt) >> b.sx);
    const int i = tt - row * b.npx;
    const int k = (int)((__umulhi((unsigned)row, b.my) + (unsigned)row) >> b.sy);
    const int j = row - k * b.npy;
    diag[t] = box_ess(b, i, j, k) ? 1.0 : box_diag_at(b, i, j, k);
  }
}

__global__ void recip_kernel(double* __restrict__ out, const double* __restrict__ in, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = 1.0 / in[i];
}

}  // namespace fk
