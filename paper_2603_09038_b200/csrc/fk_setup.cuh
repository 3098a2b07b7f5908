// fk_setup.cuh — setup-time kernels: E-restriction, PA data, Dirichlet data,
// assembled diagonal.  None of these is on the per-apply hot path.
#pragma once

#include <cstdint>

#include "fk_internal.h"
#include "pa_common.cuh"

namespace fk {

// Closed form of h1_restriction (feklab/mesh.py:157-164) for a z-slab:
// local element e = ex + nx*(ey + ny*ez_l), local node l = i + d*(j + d*k):
//   id = (ex*p + i) + npx*((ey*p + j) + npy*(ez_l*p + k))      (slab-local)
// The slab-local id plus dof_offset = z0*p*npx*npy is the reference's global id.
// Rows are padded to gs int32 (16-byte multiples for the bulk copies);
// padding entries hold a valid id (0) and are never used.
// colour = 1: row s holds element colour_element(s) (deterministic mode,
// fk_internal.h).
__global__ void restriction_kernel(int* __restrict__ gids, int nx, int ny, int nzl, int p,
                                   int64_t npx, int64_t npy, int64_t gs, int colour) {
  const int d = p + 1, d3 = d * d * d;
  const int64_t total = (int64_t)nx * ny * nzl * gs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / gs;
    const int l = (int)(t - row * gs);
    if (l >= d3) {
      gids[t] = 0;
      continue;
    }
    const int64_t e = colour ? colour_element(row, nx, ny, nzl) : row;
    const int i = l % d, j = (l / d) % d, k = l / (d * d);
    const int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / ((int64_t)nx * ny);
    gids[t] = (int)((ex * p + i) + npx * ((ey * p + j) + npy * (ez * p + k)));
  }
}

// Per-element Dirichlet bits: bit l of element e set iff its node l is essential.
__global__ void ebits_kernel(uint32_t* __restrict__ bits, const int* __restrict__ gids,
                             const unsigned char* __restrict__ mask, int64_t nel, int d3,
                             int64_t gs, int64_t ms) {
  const int64_t total = nel * ms;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / ms;
    const int w = (int)(t - e * ms);
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b) {
      const int l = w * 32 + b;
      if (l < d3 && mask[gids[e * gs + l]]) v |= 1u << b;
    }
    bits[t] = v;
  }
}

// PA data (operator.py:132-134 + SURVEY.md §8a row a10):
//   wdet(a,b,c) = (w_c * (w_b * w_a)) * detJ       (np.kron(w, np.kron(w, w)) * detJ)
//   BP1: D = wdet
//   BP3: D = wdet * J^-1 J^-T, stored as the 6 symmetric components
//        (00, 01, 02, 11, 12, 22); on the axis-aligned box the off-diagonal
//        components are zero and D_ss = wdet * (jinv_s * jinv_s).
// Layout: pa[e][comp][qp], qp = a + q*(b + q*c) (x fastest), element-major.
__global__ void pa_data_kernel(double* __restrict__ pa, int64_t nel, int q, int npa, int64_t ps,
                               const double* __restrict__ w, double detj, double ji0, double ji1,
                               double ji2) {
  const int q3 = q * q * q;
  const int64_t total = nel * q3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / q3;
    const int qp = (int)(t - e * q3);
    const int a = qp % q, b = (qp / q) % q, c = qp / (q * q);
    const double w3 = w[c] * (w[b] * w[a]);
    const double wdet = w3 * detj;
    double* o = pa + e * ps + qp;
    if (qp == 0 && ps > (int64_t)npa * q3) pa[e * ps + npa * q3] = 0.0;  // stride padding
    if (npa == 1) {
      o[0] = wdet;
    } else {
      o[0 * q3] = wdet * (ji0 * ji0);
      o[1 * q3] = 0.0;
      o[2 * q3] = 0.0;
      o[3 * q3] = wdet * (ji1 * ji1);
      o[4 * q3] = 0.0;
      o[5 * q3] = wdet * (ji2 * ji2);
    }
  }
}

// Essential (Dirichlet) dofs: every node on the six faces of the global box.
// For a z-slab only the global bottom/top planes count as z-faces.
__global__ void dirichlet_kernel(unsigned char* __restrict__ mask, int* __restrict__ ess,
                                 unsigned long long* __restrict__ n_ess, int64_t npx, int64_t npy,
                                 int64_t npz_local, int64_t gk0, int64_t npz_global) {
  const int64_t total = npx * npy * npz_local;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = t % npx, gj = (t / npx) % npy, gk = t / (npx * npy) + gk0;
    const bool on = gi == 0 || gi == npx - 1 || gj == 0 || gj == npy - 1 || gk == 0 ||
                    gk == npz_global - 1;
    mask[t] = on ? 1 : 0;
    if (on) ess[atomicAdd(n_ess, 1ull)] = (int)t;
  }
}

// y[ess] = x[ess]  (constrained operator, diagonal one)
__global__ void ess_copy_kernel(double* __restrict__ y, const double* __restrict__ x,
                                const int* __restrict__ ess, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int id = ess[t];
    y[id] = x[id];
  }
}

__global__ void ess_set_kernel(double* __restrict__ y, const int* __restrict__ ess, int64_t n,
                               double v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    y[ess[t]] = v;
}

}  // namespace fk
