// fk_mixed.cu — C-ABI of the acoustic-gravity block operator (include/fk.h,
// fk_mix_*): setup of the PA data and lumped mass diagonals, the fused
// FusedPA apply (mix_pipe.cuh), the composed normal operator, the lumped mass
// inverse and a device RK4 driver.  Reference: feklab/operator.py:105-193
// (QuadData / setup_quad_data), :221-397 (BlockOperator), :506-531 (rk4_step).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fk_error.h"
#include "fk_internal.h"
#include "mix_kernels.h"

namespace {

using fk::MixArgs;
using fk::MixKernel;
using fk::MIX_BOTH;
using fk::MIX_TAU;
using fk::MIX_VB;
using fk::MIX_BOTH_MF;
using fk::kMixCfgs;

// Compiled (order_p, order_u, q): the paper's H1(p) x L2(p-1) pairs with
// q = p+1 (the reference default is p=4, u=3, q=5, operator.py:227-229).
constexpr int kMixMaxP = 8;

const std::vector<MixKernel>& mix_registry() {
  static const std::vector<MixKernel> reg = [] {
    std::vector<MixKernel> v;
    fk_mix_register_p2(v);
    fk_mix_register_p3(v);
    fk_mix_register_p4(v);
    fk_mix_register_p5(v);
    fk_mix_register_p6(v);
    fk_mix_register_p7(v);
    fk_mix_register_p8(v);
    return v;
  }();
  return reg;
}

const int kMixAutoCfg[9] = {0, 0, 8, 3, 10, 10, 8, 8, 4};  // single-X twins, r02_ab_mix_sx.log; order 8 staged outputs, r02_ab_bcd_p3.log

int grid_for(int64_t n, int threads, int num_sms) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms * 8));
}

// E-restriction of the H1 pressure space (mesh.py:157-164), rows padded to gs
__global__ void mix_restriction_kernel(int* __restrict__ gids, int nx, int ny, int nz, int p,
                                       int64_t npx, int64_t npy, int64_t gs) {
  const int d = p + 1, d3 = d * d * d;
  const int64_t total = (int64_t)nx * ny * nz * gs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / gs;
    const int l = (int)(t - e * gs);
    if (l >= d3) {
      gids[t] = 0;
      continue;
    }
    const int i = l % d, j = (l / d) % d, k = l / (d * d);
    const int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / ((int64_t)nx * ny);
    gids[t] = (int)((ex * p + i) + npx * ((ey * p + j) + npy * (ez * p + k)));
  }
}

// dmat (operator.py:137-144, 171-175): dm[e][s*3+r][qp] = wdet(qp) * Jinv[s][r]
// with wdet = kron(w, kron(w, w)) * detJ and Jinv = diag(1/jac_diag).
__global__ void mix_pa_kernel(double* __restrict__ pa, int64_t nel, int q, int64_t ps, double w0,
                              double w1, double w2, double w3, double w4, double w5, double w6,
                              double w7, double w8, double detj, double j0, double j1, double j2) {
  const double w[9] = {w0, w1, w2, w3, w4, w5, w6, w7, w8};
  const double jinv[3] = {j0, j1, j2};
  const int q3 = q * q * q;
  const int64_t total = nel * ps;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / ps;
    const int k = (int)(t - e * ps);
    double v = 0.0;
    if (k < 9 * q3) {
      const int comp = k / q3, qp = k - comp * q3;
      const int s = comp / 3, r = comp % 3;
      const int a = qp % q, b = (qp / q) % q, c = qp / (q * q);
      if (s == r) v = (w[c] * (w[b] * w[a])) * detj * jinv[s];
    }
    pa[t] = v;
  }
}

// lump_p = scatter_add(kinv[e] * lump_ref_p) (operator.py:185-188)
__global__ void mix_lump_p_kernel(double* __restrict__ lump_p, const int* __restrict__ gids,
                                  const double* __restrict__ kinv, const double* __restrict__ ref,
                                  int64_t nel, int d3, int64_t gs) {
  const int64_t total = nel * d3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / d3;
    const int l = (int)(t - e * d3);
    atomicAdd(lump_p + gids[e * gs + l], kinv[e] * ref[l]);
  }
}

// lump_u[e][l] = rho[e] * lump_ref_u[l] (operator.py:184)
__global__ void mix_lump_u_kernel(double* __restrict__ lump_u, const double* __restrict__ rho,
                                  const double* __restrict__ ref, int64_t nel, int du3) {
  const int64_t total = nel * du3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / du3;
    lump_u[t] = rho[e] * ref[t - e * du3];
  }
}

// k = -r / lump (rk4 rhs: negate, then apply_mass_inverse, operator.py:512-516)
__global__ void mix_minv_kernel(double* __restrict__ ku, const double* __restrict__ ru,
                                const double* __restrict__ lump_u, int64_t nu, int64_t nel_du3,
                                double* __restrict__ kp, const double* __restrict__ rp,
                                const double* __restrict__ lump_p, int64_t np, double sign) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nu + np;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < nu) ku[t] = (sign * ru[t]) / lump_u[t - (t >= nel_du3 ? (t >= 2 * nel_du3 ? 2 : 1) : 0) * nel_du3];
    else kp[t - nu] = (sign * rp[t - nu]) / lump_p[t - nu];
  }
}

// One fused RK4 stage update (rk4_step, operator.py:506-531) on [u | p]:
//   k    = ((-r) + f) / lump                (rhs negation, forcing, apply_mass_inverse)
//   acc' = (first ? y : acc) + c_acc * k    (the final lincomb, accumulated in
//                                            the reference's left-to-right order)
//   ynext = y + c_next * k                  (next stage state; skipped if c_next == 0)
// Every multiply and add separately rounded, like NumPy.  k is never stored.
__global__ void mix_rk4_stage_kernel(const double* __restrict__ r, const double* __restrict__ lump_u,
                                     int64_t nu, int64_t nel_du3, const double* __restrict__ lump_p,
                                     const double* y, const double* acc_in, double* acc_out,
                                     double* __restrict__ ynext, double c_acc, double c_next,
                                     int first, int64_t n, const double* __restrict__ f) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    // u is (3, nel, du^3): its lumped entry is lump_u[t - r nel du^3] (no 64-bit modulo)
    const double lump = t < nu ? lump_u[t - (t >= nel_du3 ? (t >= 2 * nel_du3 ? 2 : 1) : 0) * nel_du3]
                               : lump_p[t - nu];
    const double k = (f ? __dadd_rn(-r[t], f[t]) : -r[t]) / lump;
    const double yt = y[t];
    acc_out[t] = __dadd_rn(first ? yt : acc_in[t], __dmul_rn(c_acc, k));
    if (c_next != 0.0) ynext[t] = __dadd_rn(yt, __dmul_rn(c_next, k));
  }
}

// ---- boundary terms (operator.py:400-470) --------------------------------------
// Face tables: 1D consistent face mass m1 = Bp^T W Bp (dp x dp) and its row
// sums l1 = Bp^T w; the 2D face mass is kron(m1, m1), the face lump kron(l1, l1)
// (_init_boundary_terms :420-427).  Face node (a, b): first in-plane index
// fastest (_face_local_indices :201-210).
struct FaceTabs {
  double m1[81];
  double l1[9];
};

// element-local node of face node (a, b) on face (axis, side)
__device__ __forceinline__ int face_node(int axis, int side, int d, int a, int b) {
  const int lay = side ? d - 1 : 0;
  return axis == 0 ? lay + d * (a + d * b) : axis == 1 ? a + d * (lay + d * b) : a + d * (b + d * lay);
}

// Absorbing lateral faces (_apply_absorbing :432-439):
//   out_p[face] += cs * (area / Z_e) * (kron(m1, m1) p_face),  Z_e = rho sqrt(1/(rho kinv)).
// Faces in blocks: x-low, x-high (ny nz each), y-low, y-high (nx nz each); one
// thread per (face, node).
__global__ void mix_absorb_kernel(const __grid_constant__ FaceTabs ft, double* __restrict__ out_p,
                                  const double* __restrict__ p, const int* __restrict__ gids,
                                  int64_t gs, const double* __restrict__ rho,
                                  const double* __restrict__ kinv, int nx, int ny, int nz, int d,
                                  double area_x, double area_y, double cs) {
  const int64_t fx = (int64_t)ny * nz, fy = (int64_t)nx * nz, nf = 2 * (fx + fy);
  const int d2 = d * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nf * d2;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t f = t / d2;
    const int node = (int)(t - f * d2), a = node % d, b = node / d;
    int axis, side;
    int64_t e;
    if (f < 2 * fx) {
      axis = 0;
      side = (int)(f / fx);
      f -= side * fx;
      e = (side ? nx - 1 : 0) + (int64_t)nx * (f % ny + (int64_t)ny * (f / ny));
    } else {
      f -= 2 * fx;
      axis = 1;
      side = (int)(f / fy);
      f -= side * fy;
      e = f % nx + (int64_t)nx * ((side ? ny - 1 : 0) + (int64_t)ny * (f / nx));
    }
    const int* g = gids + e * gs;
    double acc = 0.0;
    for (int bb = 0; bb < d; ++bb) {
      double row = 0.0;
      for (int aa = 0; aa < d; ++aa) row = fma(ft.m1[a * d + aa], p[g[face_node(axis, side, d, aa, bb)]], row);
      acc = fma(ft.m1[b * d + bb], row, acc);
    }
    const double z = rho[e] * sqrt(1.0 / (rho[e] * kinv[e]));
    atomicAdd(out_p + g[face_node(axis, side, d, a, b)], cs * (((axis == 0 ? area_x : area_y) / z) * acc));
  }
}

// Free-surface lumped mass (:268-276): lump_p[top face] += (1/(rho g)) (area l1_b l1_a)
__global__ void mix_surface_lump_kernel(const __grid_constant__ FaceTabs ft, double* __restrict__ lump_p,
                                        const int* __restrict__ gids, int64_t gs,
                                        const double* __restrict__ rho, int nx, int ny, int nz, int d,
                                        double area, double g) {
  const int64_t nf = (int64_t)nx * ny;
  const int d2 = d * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nf * d2;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = t / d2;
    const int node = (int)(t - f * d2), a = node % d, b = node / d;
    const int64_t e = f + nf * (nz - 1);
    atomicAdd(lump_p + gids[e * gs + face_node(2, 1, d, a, b)],
              (1.0 / (rho[e] * g)) * (area * (ft.l1[b] * ft.l1[a])));
  }
}

// bottom_face_load (:441-460): load[bottom face] += area * (kron(m1, m1) vals_f)
__global__ void mix_bottom_load_kernel(const __grid_constant__ FaceTabs ft, double* __restrict__ load,
                                       const double* __restrict__ vals, const int* __restrict__ gids,
                                       int64_t gs, int nx, int ny, int d, double area) {
  const int64_t nf = (int64_t)nx * ny;
  const int d2 = d * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nf * d2;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = t / d2;
    const int node = (int)(t - f * d2), a = node % d, b = node / d;
    const double* v = vals + f * d2;
    double acc = 0.0;
    for (int bb = 0; bb < d; ++bb) {
      double row = 0.0;
      for (int aa = 0; aa < d; ++aa) row = fma(ft.m1[a * d + aa], v[aa + d * bb], row);
      acc = fma(ft.m1[b * d + bb], row, acc);
    }
    atomicAdd(load + gids[f * gs + face_node(2, 0, d, a, b)], area * acc);
  }
}

// sum_i x_i m[a][i], ascending i, separately rounded (contract_cyclic, tensor.py:177-210)
void host_chain_t(const double* m /* q x d row-major: m[a*d+i] */, int q, int d, std::vector<double>& x,
                  int n0, int n1, int n2) {
  // one cyclic stage with M^T (d x q): out(j,k,i') = sum_a M[a][i'] x(a,j,k)
  std::vector<double> out((size_t)n1 * n2 * d, 0.0);
  for (int jk = 0; jk < n1 * n2; ++jk)
    for (int ip = 0; ip < d; ++ip) {
      double acc = 0.0;
      for (int a = 0; a < n0; ++a) acc = acc + x[(size_t)jk * n0 + a] * m[a * d + ip];
      out[(size_t)ip * n1 * n2 + jk] = acc;
    }
  x.swap(out);
  (void)q;
}

}  // namespace

struct fk_mix {
  fk_mix_desc desc{};
  int dp = 0, du = 0, q = 0;
  int64_t nel = 0, ndof_p = 0, npx = 0, npy = 0;
  std::vector<double> Bp, Gp, Bu, w, rho, kinv;
  const MixKernel* kern = nullptr;
  cudaStream_t stream = nullptr;
  int device = 0, num_sms = 0, blocks = 0, blocks_mf = 0;
  bool is_setup = false;
  int* gids = nullptr;
  double* pa = nullptr;
  double* lump_u = nullptr;  // (nel, du^3)
  double* lump_p = nullptr;  // ndof_p
  double* zbuf = nullptr;    // fused-normal intermediate (ndof_p)
  double* rk = nullptr;      // rk4 work: 4 stage vectors, stage state, residual, state
  cudaEvent_t ev[4] = {};
  // boundary terms
  FaceTabs face{};
  double* rho_d = nullptr;   // per-element density / inverse bulk modulus (device)
  double* kinv_d = nullptr;
};

namespace {

int64_t nu_of(const fk_mix* m) { return 3 * m->nel * m->du * m->du * m->du; }

int mix_launch_mode(fk_mix* m, const double* u, const double* p, double* out_u, double* out_p,
                    int mode, double su, double sp, cudaStream_t s) {
  MixArgs a;
  a.p = p;
  a.u = u;
  a.out_u = out_u;
  a.out_p = out_p;
  a.gids = m->gids;
  a.pa = m->pa;
  a.su = su;
  a.sp = sp;
  a.nel = (int)m->nel;
  const double jinv[3] = {1.0 / m->desc.jac_diag[0], 1.0 / m->desc.jac_diag[1],
                          1.0 / m->desc.jac_diag[2]};
  m->kern->launch(*m->kern, m->Bp.data(), m->Gp.data(), m->Bu.data(), m->w.data(),
                  m->desc.jac_det, jinv, a, mode, mode == MIX_BOTH_MF ? m->blocks_mf : m->blocks, s);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}

// out = A [u; p] (BlockOperator.apply): out_p zeroed, then one fused launch
int mix_apply_dev(fk_mix* m, const double* u, const double* p, double* out_u, double* out_p,
                  cudaStream_t s) {
  FK_CUDA(cudaMemsetAsync(out_p, 0, sizeof(double) * m->ndof_p, s));
  const double cs = m->desc.coupling_scale;
  FK_TRY(mix_launch_mode(m, u, p, out_u, out_p, m->desc.matrix_free ? MIX_BOTH_MF : MIX_BOTH, cs,
                         -cs, s));
  if (m->desc.absorbing) {
    const int nx = m->desc.nx, ny = m->desc.ny, nz = m->desc.nz, d = m->dp;
    const int64_t work = 2 * ((int64_t)ny * nz + (int64_t)nx * nz) * d * d;
    const double* jd = m->desc.jac_diag;  // h/2: area of an x face (h_y/2)(h_z/2)
    mix_absorb_kernel<<<grid_for(work, 256, m->num_sms), 256, 0, s>>>(
        m->face, out_p, p, m->gids, m->kern->gs, m->rho_d, m->kinv_d, nx, ny, nz, d, jd[1] * jd[2],
        jd[0] * jd[2], cs);
    FK_CUDA(cudaGetLastError());
  }
  return FK_OK;
}

}  // namespace

extern "C" {

int fk_mix_create(fk_mix** out, const fk_mix_desc* d) {
  if (out == nullptr || d == nullptr) return fk_fail(FK_EINVAL, "null argument");
  *out = nullptr;
  // order_u >= 1: a GLL rule needs two points (tensor.py:29-41)
  if (d->order_p < 2 || d->order_p > kMixMaxP)
    return fk_fail(FK_EUNSUPPORTED, "order_p=%d outside 2..%d", d->order_p, kMixMaxP);
  if (d->order_u != d->order_p - 1 || d->num_quad_1d != d->order_p + 1)
    return fk_fail(FK_EUNSUPPORTED,
                   "compiled spaces are H1(p) x L2(p-1) with q = p+1; got order_p=%d order_u=%d q=%d",
                   d->order_p, d->order_u, d->num_quad_1d);
  if (d->nx < 1 || d->ny < 1 || d->nz < 1)
    return fk_fail(FK_EINVAL, "mesh dimensions %d x %d x %d do not match a box", d->nx, d->ny, d->nz);
  if (!(d->jac_det > 0.0) || !(d->jac_diag[0] > 0.0) || !(d->jac_diag[1] > 0.0) ||
      !(d->jac_diag[2] > 0.0))
    return fk_fail(FK_EINVAL, "non-positive Jacobian determinant in element 0");
  if (d->Bp == nullptr || d->Gp == nullptr || d->Bu == nullptr || d->w == nullptr)
    return fk_fail(FK_EINVAL, "basis tables Bp, Gp, Bu, w are required");
  // the fused kernel folds the 1D tables even-odd (mix_pipe.cuh)
  if (!fk::mirror_symmetric(d->Bp, d->Gp, d->num_quad_1d, d->order_p + 1) ||
      !fk::mirror_symmetric(d->Bu, nullptr, d->num_quad_1d, d->order_u + 1))
    return fk_fail(FK_EUNSUPPORTED, "the block operator kernels need mirror-symmetric basis tables "
                                    "(symmetric nodes and quadrature points)");
  if (d->surface_gravity < 0.0 || !(d->surface_gravity == d->surface_gravity))
    return fk_fail(FK_EINVAL, "surface gravity must be positive");
  fk_mix* m = new fk_mix();
  m->desc = *d;
  m->dp = d->order_p + 1;
  m->du = d->order_u + 1;
  m->q = d->num_quad_1d;
  m->nel = (int64_t)d->nx * d->ny * d->nz;
  m->npx = (int64_t)d->nx * d->order_p + 1;
  m->npy = (int64_t)d->ny * d->order_p + 1;
  m->ndof_p = m->npx * m->npy * ((int64_t)d->nz * d->order_p + 1);
  if (m->ndof_p >= ((int64_t)1 << 31) || m->nel >= ((int64_t)1 << 31) - 64) {
    delete m;
    return fk_fail(FK_EINVAL, "problem too large for int32 dof ids");
  }
  m->Bp.assign(d->Bp, d->Bp + m->q * m->dp);
  m->Gp.assign(d->Gp, d->Gp + m->q * m->dp);
  m->Bu.assign(d->Bu, d->Bu + m->q * m->du);
  m->w.assign(d->w, d->w + m->q);
  m->rho.resize(m->nel);
  m->kinv.resize(m->nel);
  for (int64_t e = 0; e < m->nel; ++e) {
    const double r = d->rho ? d->rho[e] : d->rho_scalar;
    const double k = d->bulk ? d->bulk[e] : d->bulk_scalar;
    if (!(r > 0.0) || !(k > 0.0)) {
      delete m;
      return fk_fail(FK_EINVAL, "density and bulk modulus must be positive");
    }
    m->rho[e] = r;
    m->kinv[e] = 1.0 / k;
  }
  int cfg = kMixAutoCfg[d->order_p];
  if (const char* c = std::getenv("FK_MIX_CFG")) cfg = std::atoi(c);
  if (cfg < 0 || cfg >= kMixCfgs) {
    delete m;
    return fk_fail(FK_EUNSUPPORTED, "no mixed launch config %d", cfg);
  }
  for (const auto& k : mix_registry())
    if (k.dp == m->dp && k.du == m->du && k.q == m->q && k.cfg == cfg) m->kern = &k;
  if (m->kern == nullptr) {
    delete m;
    return fk_fail(FK_EUNSUPPORTED, "no kernel for order_p=%d", d->order_p);
  }
  m->device = d->device;
  m->stream = static_cast<cudaStream_t>(d->stream);
  *out = m;
  return FK_OK;
}

int fk_mix_setup(fk_mix* m) {
  if (m == nullptr) return fk_fail(FK_EINVAL, "null handle");
  FkDeviceGuard g(m->device);
  cudaStream_t s = m->stream;
  FK_CUDA(cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, m->device));
  const MixKernel& k = *m->kern;
  const int dp3 = m->dp * m->dp * m->dp, du3 = m->du * m->du * m->du, q = m->q;
  if (m->gids == nullptr) FK_CUDA(cudaMalloc(&m->gids, sizeof(int) * (m->nel * k.gs + 16)));
  mix_restriction_kernel<<<grid_for(m->nel * k.gs, 256, m->num_sms), 256, 0, s>>>(
      m->gids, m->desc.nx, m->desc.ny, m->desc.nz, m->desc.order_p, m->npx, m->npy, k.gs);
  FK_CUDA(cudaGetLastError());
  if (m->pa == nullptr) FK_CUDA(cudaMalloc(&m->pa, sizeof(double) * (m->nel * k.ps + 16)));
  double w9[9] = {0};
  for (int i = 0; i < q; ++i) w9[i] = m->w[i];
  mix_pa_kernel<<<grid_for(m->nel * k.ps, 256, m->num_sms), 256, 0, s>>>(
      m->pa, m->nel, q, k.ps, w9[0], w9[1], w9[2], w9[3], w9[4], w9[5], w9[6], w9[7], w9[8],
      m->desc.jac_det, 1.0 / m->desc.jac_diag[0], 1.0 / m->desc.jac_diag[1],
      1.0 / m->desc.jac_diag[2]);
  FK_CUDA(cudaGetLastError());
  // lumped diagonals: lump_ref = apply_basis_transpose_3d(basis, wdet_ref) on the host
  std::vector<double> wdet((size_t)q * q * q);
  for (int c = 0; c < q; ++c)
    for (int b = 0; b < q; ++b)
      for (int a = 0; a < q; ++a) wdet[a + q * (b + q * c)] = (m->w[c] * (m->w[b] * m->w[a])) * m->desc.jac_det;
  auto lump_ref = [&](const std::vector<double>& B, int d) {
    std::vector<double> x = wdet;
    host_chain_t(B.data(), q, d, x, q, q, q);
    host_chain_t(B.data(), q, d, x, q, q, d);
    host_chain_t(B.data(), q, d, x, q, d, d);
    return x;  // (d, d, d) x fastest
  };
  std::vector<double> lu = lump_ref(m->Bu, m->du), lp = lump_ref(m->Bp, m->dp);
  double* d_ref = nullptr;
  FK_CUDA(cudaMalloc(&d_ref, sizeof(double) * (du3 + dp3)));
  if (m->rho_d == nullptr) FK_CUDA(cudaMalloc(&m->rho_d, sizeof(double) * m->nel));
  if (m->kinv_d == nullptr) FK_CUDA(cudaMalloc(&m->kinv_d, sizeof(double) * m->nel));
  double* d_rho = m->rho_d;
  double* d_kinv = m->kinv_d;
  // face tables m1 = Bp^T W Bp, l1 = Bp^T w (_init_boundary_terms, operator.py:420-427)
  for (int i = 0; i < m->dp; ++i) {
    double l = 0.0;
    for (int a2 = 0; a2 < q; ++a2) l += m->Bp[a2 * m->dp + i] * m->w[a2];
    m->face.l1[i] = l;
    for (int j = 0; j < m->dp; ++j) {
      double s2 = 0.0;
      for (int a2 = 0; a2 < q; ++a2) s2 += m->Bp[a2 * m->dp + i] * (m->w[a2] * m->Bp[a2 * m->dp + j]);
      m->face.m1[i * m->dp + j] = s2;
    }
  }
  FK_CUDA(cudaMemcpyAsync(d_ref, lu.data(), sizeof(double) * du3, cudaMemcpyHostToDevice, s));
  FK_CUDA(cudaMemcpyAsync(d_ref + du3, lp.data(), sizeof(double) * dp3, cudaMemcpyHostToDevice, s));
  FK_CUDA(cudaMemcpyAsync(d_rho, m->rho.data(), sizeof(double) * m->nel, cudaMemcpyHostToDevice, s));
  FK_CUDA(cudaMemcpyAsync(d_kinv, m->kinv.data(), sizeof(double) * m->nel, cudaMemcpyHostToDevice, s));
  if (m->lump_u == nullptr) FK_CUDA(cudaMalloc(&m->lump_u, sizeof(double) * m->nel * du3));
  if (m->lump_p == nullptr) FK_CUDA(cudaMalloc(&m->lump_p, sizeof(double) * m->ndof_p));
  mix_lump_u_kernel<<<grid_for(m->nel * du3, 256, m->num_sms), 256, 0, s>>>(m->lump_u, d_rho, d_ref,
                                                                            m->nel, du3);
  FK_CUDA(cudaMemsetAsync(m->lump_p, 0, sizeof(double) * m->ndof_p, s));
  mix_lump_p_kernel<<<grid_for(m->nel * dp3, 256, m->num_sms), 256, 0, s>>>(
      m->lump_p, m->gids, d_kinv, d_ref + du3, m->nel, dp3, k.gs);
  FK_CUDA(cudaGetLastError());
  if (m->desc.surface_gravity > 0.0) {  // after the volume lump, as the reference
    const int64_t work = (int64_t)m->desc.nx * m->desc.ny * m->dp * m->dp;
    mix_surface_lump_kernel<<<grid_for(work, 256, m->num_sms), 256, 0, s>>>(
        m->face, m->lump_p, m->gids, k.gs, d_rho, m->desc.nx, m->desc.ny, m->desc.nz, m->dp,
        m->desc.jac_diag[0] * m->desc.jac_diag[1], m->desc.surface_gravity);
    FK_CUDA(cudaGetLastError());
  }
  FK_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_ref);
  for (const void* f : {k.f_both, k.f_tau, k.f_vb})
    FK_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem));
  FK_CUDA(cudaFuncSetAttribute(k.f_mf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem_mf));
  int occ = 0, occ_mf = 0;
  FK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k.f_both, k.T, k.smem));
  FK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_mf, k.f_mf, k.T, k.smem_mf));
  if (occ < 1 || occ_mf < 1)
    return fk_fail(FK_EUNSUPPORTED, "mixed kernel does not fit on an SM (smem %zu)", k.smem);
  const int64_t nbatch = (m->nel + k.E - 1) / k.E;
  m->blocks = (int)std::max<int64_t>(1, std::min<int64_t>(nbatch, (int64_t)occ * m->num_sms));
  m->blocks_mf = (int)std::max<int64_t>(1, std::min<int64_t>(nbatch, (int64_t)occ_mf * m->num_sms));
  // test hook (as fk_api.cu): cap the persistent grid so small meshes run
  // several batches per CTA (the cross-batch gather / id prefetches)
  if (const char* c = std::getenv("FK_MAX_BLOCKS")) {
    const int cap = std::max(1, std::atoi(c));
    m->blocks = std::min(m->blocks, cap);
    m->blocks_mf = std::min(m->blocks_mf, cap);
  }
  for (auto& e : m->ev) FK_CUDA(cudaEventCreate(&e));
  m->is_setup = true;
  return FK_OK;
}

int fk_mix_get_info(const fk_mix* m, fk_mix_info* info) {
  if (m == nullptr || info == nullptr) return fk_fail(FK_EINVAL, "null argument");
  info->nel = m->nel;
  info->ndof_p = m->ndof_p;
  info->ndof_u = nu_of(m);
  info->pa_bytes = (int64_t)sizeof(double) * m->nel * m->kern->ps;
  info->elems_per_block = m->kern->E;
  info->threads_per_block = m->kern->T;
  info->blocks = m->desc.matrix_free ? m->blocks_mf : m->blocks;
  info->smem_bytes = (int64_t)m->kern->smem;
  return FK_OK;
}

int fk_mix_apply(fk_mix* m, const double* u, const double* p, double* out_u, double* out_p) {
  if (m == nullptr || u == nullptr || p == nullptr || out_u == nullptr || out_p == nullptr)
    return fk_fail(FK_EINVAL, "null argument");
  if (!m->is_setup) return fk_fail(FK_EINVAL, "fk_mix_setup has not been called");
  FkDeviceGuard g(m->device);
  return mix_apply_dev(m, u, p, out_u, out_p, m->stream);
}

int fk_mix_fused_normal(fk_mix* m, const double* u, double* out_u) {
  if (m == nullptr || u == nullptr || out_u == nullptr) return fk_fail(FK_EINVAL, "null argument");
  if (!m->is_setup) return fk_fail(FK_EINVAL, "fk_mix_setup has not been called");
  FkDeviceGuard g(m->device);
  if (m->zbuf == nullptr) FK_CUDA(cudaMalloc(&m->zbuf, sizeof(double) * m->ndof_p));
  FK_CUDA(cudaMemsetAsync(m->zbuf, 0, sizeof(double) * m->ndof_p, m->stream));
  // z = sum_e G^T v_e(u) (operator.py:375-380), then out = tau(G z) (:381-386)
  FK_TRY(mix_launch_mode(m, u, nullptr, nullptr, m->zbuf, MIX_VB, 1.0, 1.0, m->stream));
  return mix_launch_mode(m, nullptr, m->zbuf, out_u, nullptr, MIX_TAU, 1.0, 1.0, m->stream);
}

int fk_mix_mass_inverse(fk_mix* m, const double* ru, const double* rp, double* u, double* p) {
  if (m == nullptr || ru == nullptr || rp == nullptr || u == nullptr || p == nullptr)
    return fk_fail(FK_EINVAL, "null argument");
  if (!m->is_setup) return fk_fail(FK_EINVAL, "fk_mix_setup has not been called");
  FkDeviceGuard g(m->device);
  const int64_t nu = nu_of(m), du3 = m->du * m->du * m->du;
  mix_minv_kernel<<<grid_for(nu + m->ndof_p, 256, m->num_sms), 256, 0, m->stream>>>(
      u, ru, m->lump_u, nu, m->nel * du3, p, rp, m->lump_p, m->ndof_p, 1.0);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}

static int mix_rk4(fk_mix* m, double* u, double* p, double dt, int steps, const double* f0,
                   const double* fh, const double* f1) {
  if (m == nullptr || u == nullptr || p == nullptr) return fk_fail(FK_EINVAL, "null argument");
  if (!m->is_setup) return fk_fail(FK_EINVAL, "fk_mix_setup has not been called");
  if (!(dt > 0.0)) return fk_fail(FK_EINVAL, "dt must be positive, got %g", dt);
  if (steps < 0) return fk_fail(FK_EINVAL, "steps must be >= 0");
  FkDeviceGuard g(m->device);
  const int64_t nu = nu_of(m), n = nu + m->ndof_p, du3 = m->du * m->du * m->du;
  // work vectors [u | p]: y (state), acc (final lincomb), ytmp (stage state), r (residual)
  if (m->rk == nullptr) FK_CUDA(cudaMalloc(&m->rk, sizeof(double) * 4 * n));
  double* y = m->rk;
  double* acc = m->rk + n;
  double* ytmp = m->rk + 2 * n;
  double* res = m->rk + 3 * n;
  cudaStream_t s = m->stream;
  const int gb = grid_for(n, 256, m->num_sms);
  // one stage: r = A x, then the fused k / acc / next-state update
  auto stage = [&](const double* x, double c_acc, double c_next, int first, double* acc_out,
                   const double* f) -> int {
    FK_TRY(mix_apply_dev(m, x, x + nu, res, res + nu, s));
    mix_rk4_stage_kernel<<<gb, 256, 0, s>>>(res, m->lump_u, nu, m->nel * du3, m->lump_p, y, acc,
                                            acc_out, ytmp, c_acc, c_next, first, n, f);
    FK_CUDA(cudaGetLastError());
    return FK_OK;
  };
  FK_CUDA(cudaMemcpyAsync(y, u, sizeof(double) * nu, cudaMemcpyDeviceToDevice, s));
  FK_CUDA(cudaMemcpyAsync(y + nu, p, sizeof(double) * m->ndof_p, cudaMemcpyDeviceToDevice, s));
  for (int st = 0; st < steps; ++st) {
    FK_TRY(stage(y, dt / 6, dt / 2, 1, acc, f0));     // k1 = rhs(t)
    FK_TRY(stage(ytmp, dt / 3, dt / 2, 0, acc, fh));  // k2 = rhs(t + dt/2)
    FK_TRY(stage(ytmp, dt / 3, dt, 0, acc, fh));      // k3 = rhs(t + dt/2)
    FK_TRY(stage(ytmp, dt / 6, 0.0, 0, y, f1));       // k4 = rhs(t + dt): y = acc + dt/6 k4
  }
  FK_CUDA(cudaMemcpyAsync(u, y, sizeof(double) * nu, cudaMemcpyDeviceToDevice, s));
  FK_CUDA(cudaMemcpyAsync(p, y + nu, sizeof(double) * m->ndof_p, cudaMemcpyDeviceToDevice, s));
  return FK_OK;
}

int fk_mix_rk4(fk_mix* m, double* u, double* p, double dt, int steps) {
  return mix_rk4(m, u, p, dt, steps, nullptr, nullptr, nullptr);
}

int fk_mix_rk4_forced(fk_mix* m, double* u, double* p, double dt, const double* f0,
                      const double* fh, const double* f1) {
  return mix_rk4(m, u, p, dt, 1, f0, fh, f1);
}

int fk_mix_bottom_load(fk_mix* m, const double* vals, double* load) {
  if (m == nullptr || vals == nullptr || load == nullptr) return fk_fail(FK_EINVAL, "null argument");
  if (!m->is_setup) return fk_fail(FK_EINVAL, "fk_mix_setup has not been called");
  FkDeviceGuard g(m->device);
  FK_CUDA(cudaMemsetAsync(load, 0, sizeof(double) * m->ndof_p, m->stream));
  const int64_t work = (int64_t)m->desc.nx * m->desc.ny * m->dp * m->dp;
  mix_bottom_load_kernel<<<grid_for(work, 256, m->num_sms), 256, 0, m->stream>>>(
      m->face, load, vals, m->gids, m->kern->gs, m->desc.nx, m->desc.ny, m->dp,
      m->desc.jac_diag[0] * m->desc.jac_diag[1]);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}

int fk_mix_lumped(fk_mix* m, double* lump_u, double* lump_p) {
  if (m == nullptr || lump_u == nullptr || lump_p == nullptr) return fk_fail(FK_EINVAL, "null argument");
  if (!m->is_setup) return fk_fail(FK_EINVAL, "fk_mix_setup has not been called");
  FkDeviceGuard g(m->device);
  const int64_t du3 = m->du * m->du * m->du;
  FK_CUDA(cudaMemcpyAsync(lump_u, m->lump_u, sizeof(double) * m->nel * du3, cudaMemcpyDeviceToDevice,
                          m->stream));
  FK_CUDA(cudaMemcpyAsync(lump_p, m->lump_p, sizeof(double) * m->ndof_p, cudaMemcpyDeviceToDevice,
                          m->stream));
  return FK_OK;
}

int fk_mix_restriction(fk_mix* m, int64_t* host_out) {
  if (m == nullptr || host_out == nullptr) return fk_fail(FK_EINVAL, "null argument");
  if (!m->is_setup) return fk_fail(FK_EINVAL, "fk_mix_setup has not been called");
  FkDeviceGuard g(m->device);
  const int dp3 = m->dp * m->dp * m->dp, gs = m->kern->gs;
  std::vector<int> buf((size_t)m->nel * gs);
  FK_CUDA(cudaMemcpyAsync(buf.data(), m->gids, sizeof(int) * buf.size(), cudaMemcpyDeviceToHost, m->stream));
  FK_CUDA(cudaStreamSynchronize(m->stream));
  for (int64_t e = 0; e < m->nel; ++e)
    for (int l = 0; l < dp3; ++l) host_out[e * dp3 + l] = buf[(size_t)e * gs + l];
  return FK_OK;
}

int fk_mix_time_apply(fk_mix* m, const double* u, const double* p, double* out_u, double* out_p,
                      int reps, double* ms_apply, double* ms_kernel) {
  if (m == nullptr || reps < 1) return fk_fail(FK_EINVAL, "bad argument");
  if (!m->is_setup) return fk_fail(FK_EINVAL, "fk_mix_setup has not been called");
  FkDeviceGuard g(m->device);
  std::vector<cudaEvent_t> ev(3 * (size_t)reps);
  for (auto& e : ev) FK_CUDA(cudaEventCreate(&e));
  const double cs = m->desc.coupling_scale;
  for (int r = 0; r < reps; ++r) {
    FK_CUDA(cudaEventRecord(ev[3 * r], m->stream));
    FK_CUDA(cudaMemsetAsync(out_p, 0, sizeof(double) * m->ndof_p, m->stream));
    FK_CUDA(cudaEventRecord(ev[3 * r + 1], m->stream));
    FK_TRY(mix_launch_mode(m, u, p, out_u, out_p, m->desc.matrix_free ? MIX_BOTH_MF : MIX_BOTH, cs,
                           -cs, m->stream));
    FK_CUDA(cudaEventRecord(ev[3 * r + 2], m->stream));
  }
  FK_CUDA(cudaEventSynchronize(ev.back()));
  double ta = 0.0, tk = 0.0;
  for (int r = 0; r < reps; ++r) {
    float a = 0.f, k = 0.f;
    FK_CUDA(cudaEventElapsedTime(&a, ev[3 * r], ev[3 * r + 2]));
    FK_CUDA(cudaEventElapsedTime(&k, ev[3 * r + 1], ev[3 * r + 2]));
    ta += a;
    tk += k;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (ms_apply) *ms_apply = ta / reps;
  if (ms_kernel) *ms_kernel = tk / reps;
  return FK_OK;
}

int fk_mix_destroy(fk_mix* m) {
  if (m == nullptr) return FK_OK;
  FkDeviceGuard g(m->device);
  cudaFree(m->gids);
  cudaFree(m->pa);
  cudaFree(m->lump_u);
  cudaFree(m->lump_p);
  cudaFree(m->zbuf);
  cudaFree(m->rk);
  for (auto& e : m->ev)
    if (e) cudaEventDestroy(e);
  cudaFree(m->rho_d);
  cudaFree(m->kinv_d);
  delete m;
  return FK_OK;
}

}  // extern "C"
