// fk_api.cu — the C-ABI (include/fk.h): handle lifecycle, setup, apply,
// diagonal, device CG, z-slab exchange.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fk_cg.cuh"
#include "fk_comm.h"
#include "fk_error.h"
#include "fk_internal.h"
#include "fk_setup.cuh"

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------

static thread_local std::string g_last_error;

int fk_fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}
#define fail fk_fail

namespace {

using DeviceGuard = FkDeviceGuard;

std::vector<fk::KernelEntry>& registry() {
  static std::vector<fk::KernelEntry> reg;
  static std::once_flag once;
  std::call_once(once, [] { fk::register_kernels(reg); });
  return reg;
}

int grid_for(int64_t n, int threads, int num_sms) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms * 8;
  return (int)std::max<int64_t>(1, std::min(b, cap));
}

// Per-order automatic choice (FK_VARIANT_AUTO): variant and launch geometry
// with the highest measured GDOF/s in the p-sweep on B200.
// The FP64-FMA line kernels win at every order on sm_100a: DMMA and DFMA share
// the 37 TFLOP/s FP64 pipe, and DMMA's 8x8x4 padding wastes 14-88% of it at
// these shapes.
// (variant, cfg) per order, best of profiles/r01_sweep_v21_shared_rows.jsonl
// (BP3; one box, every candidate geometry incl. the precomputed-gather cfgs
// 25-31, shared table rows) and r01_sweep_v19_xp.jsonl (BP1); BP3 p=4 from
// the repeated A/Bs r01_ab_p4_cfg29_32.log and r01_ab_p4_cfg32_35.log (cfg 35:
// four elements per CTA, W over T2, no shared rows, closed-form ids, one X
// buffer, precomputed gather: +6% over cfg 32 over 1000 applies);
// tools/auto_table.py.  Structured-id geometries (eo19-24, 29-49) fall back
// to cfg 0 when the caller passes its own gather map
constexpr int D_ = FK_VARIANT_DFMA, O_ = FK_VARIANT_EO;
const int kAutoVar3[9] = {D_, O_, O_, O_, O_, O_, O_, O_, O_};
const int kAutoCfg3[9] = {0, 19, 35, 35, 35, 25, 14, 18, 23};  // every p by 200-apply A/B: r01_ab_orders_*.log
const int kAutoVar1[9] = {D_, O_, O_, O_, O_, O_, O_, O_, O_};
const int kAutoCfg1[9] = {0, 58, 58, 51, 40, 47, 47, 43, 45};  // p <= 2: thread per element, r02_ab_tpe.log; p = 3: fused B-C-D, r02_ab_bcd_p3.log; p >= 4: staged scatter, r02_ab_bp1_ys.log

int auto_variant(int nc, int p, int q) {
  (void)q;
  if (p < 1 || p > 8) return FK_VARIANT_DFMA;
  return nc == 3 ? kAutoVar3[p] : kAutoVar1[p];
}

// matrix-free geometry per order (best of profiles/r01_sweep_v24_mf10.jsonl, the
// earlier r01_sweep_v14_mf / v20_mf_xp where the new geometries do not win;
// BP3 p=4 mf10 +6% over mf5 in a repeated A/B, r01_ab_mf_p4_cfg5_10.log)
const int kAutoCfgMF3[9] = {0, 8, 10, 10, 10, 10, 6, 5, 6};
const int kAutoCfgMF1[9] = {0, 3, 9, 8, 10, 10, 10, 10, 4};
int auto_cfg_mf(int nc, int p) {
  if (p < 1 || p > 8) return 0;
  return nc == 3 ? kAutoCfgMF3[p] : kAutoCfgMF1[p];
}

int auto_cfg(int nc, int p) {
  if (p < 1 || p > 8) return 0;
  return nc == 3 ? kAutoCfg3[p] : kAutoCfg1[p];
}

// Fastest geometry that reads the gather-id array (no closed-form ids) per
// order: the deterministic mode (colour-ordered rows) and user maps.  Best
// array-map entries of profiles/r01_sweep_f6.jsonl.
const int kArrayCfg3[9] = {0, 1, 1, 2, 1, 1, 1, 18, 11};
const int kArrayCfg1[9] = {0, 28, 28, 28, 25, 25, 26, 15, 27};
const int kArrayCfgMF3[9] = {0, 5, 7, 5, 5, 5, 6, 2, 2};
const int kArrayCfgMF1[9] = {0, 3, 3, 3, 0, 5, 4, 4, 6};
int array_cfg(int nc, int p, int variant) {
  if (p < 1 || p > 8) return 0;
  if (variant == FK_VARIANT_MF) return nc == 3 ? kArrayCfgMF3[p] : kArrayCfgMF1[p];
  if (variant == FK_VARIANT_EO) return nc == 3 ? kArrayCfg3[p] : kArrayCfg1[p];
  return 0;
}

// the kernel must read op->gids (user map, or colour-ordered rows)
bool needs_array_map(const fk_op* op) { return !op->host_gids.empty() || op->colour; }

fk::OpView view(const fk_op* op) {
  fk::OpView v;
  v.B = op->B;
  v.G = op->G;
  v.gids = op->gids;
  v.pa = op->pa;
  v.ebits = op->ebits;
  v.nel = (int)op->nel;
  v.w = op->w;
  v.detj = op->desc.jac_det;
  for (int s = 0; s < 3; ++s) v.jinv[s] = op->jinv[s];
  v.nx = op->desc.nx;
  v.ny = op->desc.ny;
  v.p = op->p;
  v.npx = op->npx;
  v.npy = op->npy;
  v.e0 = 0;
  return v;
}

// Even-odd folding needs B[q-1-a][d-1-i] = B[a][i] and G[q-1-a][d-1-i] = -G[a][i]
// (symmetric nodes and points, as Basis1D.nodal produces, tensor.py:101-119).
// The folded kernels use one half of each mirror pair, i.e. the tables are
// symmetrised.  Basis1D.nodal's monomial-coefficient tables are themselves
// only symmetric to their rounding: up to 41 / 59 ulp of max|B| at p = 8
// (q = 9 / 10; 2 ulp at p = 4), the same size as their deviation from exact
// Lagrange values (7.5e-15 at p = 8).  The gate admits that
// rounding (128 ulp of the table maximum) and nothing coarser, so the
// symmetrisation moves no entry by more than 64 ulp of max|B|.
bool tables_symmetric(const fk_op* op) {
  return fk::mirror_symmetric(op->B, op->G, op->q, op->d);
}

int select_kernel(fk_op* op, int variant) {
  int v = variant == FK_VARIANT_AUTO ? auto_variant(op->nc, op->p, op->q) : variant;
  if ((v == FK_VARIANT_EO || v == FK_VARIANT_MF) && !tables_symmetric(op)) {
    if (variant != FK_VARIANT_AUTO)
      return fail(FK_EUNSUPPORTED, "even-odd / matrix-free variants need symmetric basis tables");
    v = FK_VARIANT_DFMA;
  }
  const fk::KernelEntry* k = nullptr;
  if (op->cfg >= 0) k = fk::find_kernel_cfg(op->nc, op->d, op->q, v, op->cfg);
  else if (variant == FK_VARIANT_AUTO) k = fk::find_kernel_cfg(op->nc, op->d, op->q, v, auto_cfg(op->nc, op->p));
  else if (variant == FK_VARIANT_MF) k = fk::find_kernel_cfg(op->nc, op->d, op->q, v, auto_cfg_mf(op->nc, op->p));
  if (k == nullptr) k = fk::find_kernel(op->nc, op->d, op->q, v);
  if (k != nullptr && k->structured && needs_array_map(op)) {
    if (op->cfg >= 0)
      return fail(FK_EUNSUPPORTED, "launch config %d uses the closed-form box restriction; "
                                   "%s", op->cfg, op->colour ? "the deterministic mode orders elements by colour"
                                                             : "a user gather map was given");
    k = fk::find_kernel_cfg(op->nc, op->d, op->q, v, array_cfg(op->nc, op->p, v));
    if (k == nullptr || k->structured) k = fk::find_kernel(op->nc, op->d, op->q, v);  // cfg 0: array map
  }
  if (k == nullptr)
    return fail(FK_EUNSUPPORTED, "no %s kernel compiled for kind=%d p=%d q=%d",
                v == FK_VARIANT_DMMA ? "DMMA" : v == FK_VARIANT_EO ? "even-odd" : v == FK_VARIANT_MF ? "matrix-free" : "DFMA",
                op->desc.kind, op->p, op->q);
  {
    int max_smem = 0;
    DeviceGuard g(op->device);
    FK_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, op->device));
    if (k->smem > (size_t)max_smem) {
      if (op->cfg >= 0)
        return fail(FK_EUNSUPPORTED, "launch config %d needs %zu B shared memory (> %d)", op->cfg,
                    k->smem, max_smem);
      // default geometry too large: first compiled geometry of this variant
      // that fits (and reads the user's gather map if there is one)
      const fk::KernelEntry* alt = nullptr;
      for (const auto& t : registry()) {
        if (t.nc != op->nc || t.d != op->d || t.q != op->q || t.variant != v) continue;
        if (t.structured && needs_array_map(op)) continue;
        if (t.smem <= (size_t)max_smem) {
          alt = &t;
          break;
        }
      }
      if (alt == nullptr) return fail(FK_EUNSUPPORTED, "no launch config fits in shared memory");
      k = alt;
    }
  }
  if (op->is_setup) {
    DeviceGuard g(op->device);
    FK_CUDA(cudaFuncSetAttribute(k->func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)k->smem));
    if (k->func_qf)
      FK_CUDA(cudaFuncSetAttribute(k->func_qf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)k->smem));
    int occ = 0;
    FK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k->func, k->T, k->smem));
    if (occ < 1) return fail(FK_EUNSUPPORTED, "fused kernel does not fit on an SM (smem %zu)", k->smem);
    const int64_t nbatch = (op->nel + k->E - 1) / k->E;
    int max_blocks = occ * op->num_sms;
    if (op->block_cap > 0) max_blocks = std::min(max_blocks, op->block_cap);
    op->max_blocks = max_blocks;
    op->blocks = k->persist
                     ? (int)std::max<int64_t>(1, std::min<int64_t>(nbatch, (int64_t)max_blocks))
                     : (int)std::max<int64_t>(1, nbatch);
  }
  // committed only now: a failed selection leaves the previous kernel in place
  op->kern = k;
  op->variant = v;
  return FK_OK;
}

int launch_range(fk_op* op, const double* x, double* y, int64_t e0, int64_t ne, cudaStream_t s);

// The fused kernel over every local element (y already zeroed): one launch,
// or in the deterministic mode one launch per colour in colour order.
int launch_all(fk_op* op, const double* x, double* y, cudaStream_t s) {
  if (op->colour) {
    for (int c = 0; c < 8; ++c)
      FK_TRY(launch_range(op, x, y, op->colour_off[c], op->colour_off[c + 1] - op->colour_off[c], s));
    return FK_OK;
  }
  fk::OpView v = view(op);
  if (op->qf_on) v.qf = op->qf_part + (size_t)op->qf_seg++ * op->max_blocks;
  (op->qf_on ? op->kern->launch_qf : op->kern->launch)(v, x, y, op->blocks, s);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}

int launch_local(fk_op* op, const double* x, double* y) {
  FK_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * op->ndof, op->stream));
  return launch_all(op, x, y, op->stream);
}

// Fused kernel over local elements [e0, e0 + ne) (gids / PA data offset views).
int launch_range(fk_op* op, const double* x, double* y, int64_t e0, int64_t ne, cudaStream_t s) {
  if (ne <= 0) return FK_OK;
  fk::OpView v = view(op);
  v.gids += e0 * op->gs;
  v.pa += e0 * op->ps;
  v.e0 = e0;
  if (v.ebits) v.ebits += e0 * op->ms;
  v.nel = (int)ne;
  if (op->qf_on) v.qf = op->qf_part + (size_t)op->qf_seg++ * op->max_blocks;
  const int64_t nb = (ne + op->kern->E - 1) / op->kern->E;
  const int blocks =
      (int)std::max<int64_t>(1, op->kern->persist ? std::min<int64_t>(nb, op->max_blocks) : nb);
  (op->qf_on ? op->kern->launch_qf : op->kern->launch)(v, x, y, blocks, s);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}

// Multi-rank apply with the interface exchange overlapped:
// boundary element layers first, then the plane exchange runs while the
// interior layers (which never touch an interface plane) compute; the
// received partial sums are added after the join.
int apply_overlapped(fk_op* op, const double* x, double* y) {
  const int64_t nxy = (int64_t)op->desc.nx * op->desc.ny;
  FK_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * op->ndof, op->stream));
  FK_TRY(launch_range(op, x, y, 0, nxy, op->stream));
  FK_TRY(launch_range(op, x, y, op->nel - nxy, nxy, op->stream));
  if (fk::p2p(op)) {
    // peer memory: the plane stores are issued in stream order before the
    // interior kernel (a few µs of NVLink stores that never wait behind the
    // persistent grid); the data lands in the neighbours' mailboxes while the
    // interior layers run, and the add waits on the arrival flags after them
    FK_TRY(fk::exchange_post(op, y, op->stream));
    FK_TRY(launch_range(op, x, y, nxy, op->nel - 2 * nxy, op->stream));
    return fk::exchange_finish(op, y, op->stream);
  }
  FK_CUDA(cudaEventRecord(op->ev_bnd, op->stream));
  FK_CUDA(cudaStreamWaitEvent(op->comm_stream, op->ev_bnd, 0));
  FK_TRY(fk::exchange_post(op, y, op->comm_stream));
  FK_CUDA(cudaEventRecord(op->ev_xchg, op->comm_stream));
  FK_TRY(launch_range(op, x, y, nxy, op->nel - 2 * nxy, op->stream));
  FK_CUDA(cudaStreamWaitEvent(op->stream, op->ev_xchg, 0));
  return fk::exchange_finish(op, y, op->stream);
}

int apply_full(fk_op* op, const double* x, double* y, cudaStream_t s_override = nullptr) {
  cudaStream_t saved = op->stream;
  if (s_override) op->stream = s_override;
  int rc = FK_OK;
  if (fk::multi_rank(op) && op->desc.nz_local >= 3 && !op->colour) {
    rc = apply_overlapped(op, x, y);
  } else {
    rc = launch_local(op, x, y);
    if (rc == FK_OK && op->comm) rc = fk::exchange_interface(op, y, op->stream);
  }
  if (rc == FK_OK && op->desc.dirichlet && op->n_ess > 0) {
    fk::ess_copy_kernel<<<grid_for(op->n_ess, 256, op->num_sms), 256, 0, op->stream>>>(
        y, x, op->ess, op->n_ess);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = fail(FK_ECUDA, "ess_copy_kernel: %s", cudaGetErrorString(e));
  }
  op->stream = saved;
  return rc;
}

}  // namespace

// With CUDA lazy module loading (the default since CUDA 12.2) the first launch
// of a kernel may need a context synchronisation; if a peer rank's exchange
// kernel is spinning on this device at that moment (a loopback group, or any
// rank waiting for a neighbour), that synchronisation never completes.  So a
// multi-rank operator loads, at setup, every kernel its apply / diagonal /
// dot / CG paths can launch (cudaFuncGetAttributes forces the load).
static int preload_kernels(const fk_op* op) {
  const void* ks[] = {reinterpret_cast<const void*>(&fk::ess_copy_kernel),
                      reinterpret_cast<const void*>(&fk::ess_set_kernel),
                      reinterpret_cast<const void*>(&fk::dot_kernel),
                      reinterpret_cast<const void*>(&fk::cg_init_kernel),
                      reinterpret_cast<const void*>(&fk::cg_start_kernel),
                      reinterpret_cast<const void*>(&fk::cg_alpha_kernel),
                      reinterpret_cast<const void*>(&fk::cg_residual_kernel),
                      reinterpret_cast<const void*>(&fk::cg_finish_kernel),
                      reinterpret_cast<const void*>(&fk::cg_step_kernel),
                      reinterpret_cast<const void*>(&fk::qf_sum_kernel),
                      reinterpret_cast<const void*>(&fk::recip_kernel),
                      reinterpret_cast<const void*>(&fk::diag_box_rn_kernel)};
  cudaFuncAttributes a;
  for (const void* k : ks) FK_CUDA(cudaFuncGetAttributes(&a, k));
  for (const auto& k : registry()) {
    if (k.nc != op->nc || k.d != op->d || k.q != op->q) continue;
    FK_CUDA(cudaFuncGetAttributes(&a, k.func));
    if (k.func_qf) FK_CUDA(cudaFuncGetAttributes(&a, k.func_qf));
    if (k.diag_func) FK_CUDA(cudaFuncGetAttributes(&a, k.diag_func));
  }
  return fk::preload_comm_kernels();
}

// reduction scratch (block partials, last-block counters, CG scalars); made at
// setup so that dots and CG solves allocate nothing while peers may be waiting
static int ensure_reduce_ws(fk_op* op) {
  if (op->partials == nullptr) {
    FK_CUDA(cudaMalloc(&op->partials, sizeof(double) * 4096));
    FK_CUDA(cudaMalloc(&op->counter, sizeof(unsigned) * 4));
    FK_CUDA(cudaMemsetAsync(op->counter, 0, sizeof(unsigned) * 4, op->stream));
    FK_CUDA(cudaMalloc(&op->scal, sizeof(double) * 16 + sizeof(int) * 8));
    FK_CUDA(cudaMemsetAsync(op->scal, 0, sizeof(double) * 16 + sizeof(int) * 8, op->stream));
  }
  return FK_OK;
}

int fk_set_error(int code, const char* msg) { return fail(code, "%s", msg); }

void fk_register_p1(std::vector<fk::KernelEntry>&);
void fk_register_p2(std::vector<fk::KernelEntry>&);
void fk_register_p3(std::vector<fk::KernelEntry>&);
void fk_register_p4(std::vector<fk::KernelEntry>&);
void fk_register_p5(std::vector<fk::KernelEntry>&);
void fk_register_p6(std::vector<fk::KernelEntry>&);
void fk_register_p7(std::vector<fk::KernelEntry>&);
void fk_register_p8(std::vector<fk::KernelEntry>&);

namespace fk {
void register_kernels(std::vector<KernelEntry>& out) {
  fk_register_p1(out);
  fk_register_p2(out);
  fk_register_p3(out);
  fk_register_p4(out);
  fk_register_p5(out);
  fk_register_p6(out);
  fk_register_p7(out);
  fk_register_p8(out);
}

const KernelEntry* find_kernel(int nc, int d, int q, int variant) {
  for (const auto& k : registry())
    if (k.nc == nc && k.d == d && k.q == q && k.variant == variant) return &k;
  return nullptr;
}

const KernelEntry* find_kernel_cfg(int nc, int d, int q, int variant, int cfg) {
  for (const auto& k : registry())
    if (k.nc == nc && k.d == d && k.q == q && k.variant == variant && k.cfg == cfg) return &k;
  return nullptr;
}
}  // namespace fk

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------

extern "C" {

int fk_version(void) { return FK_API_VERSION; }

const char* fk_last_error(void) { return g_last_error.c_str(); }

int fk_op_create(fk_op** out, const fk_op_desc* d) {
  if (out == nullptr || d == nullptr) return fail(FK_EINVAL, "null argument");
  *out = nullptr;
  if (d->kind != FK_KIND_MASS && d->kind != FK_KIND_DIFFUSION)
    return fail(FK_EINVAL, "kind %d is not FK_KIND_MASS (1) or FK_KIND_DIFFUSION (3)", d->kind);
  if (d->p < 1 || d->p > 8) return fail(FK_EUNSUPPORTED, "order p=%d outside 1..8", d->p);
  if (d->q != d->p + 1 && d->q != d->p + 2)
    return fail(FK_EUNSUPPORTED, "num_quad_1d=%d must be p+1 or p+2 for p=%d", d->q, d->p);
  if (d->nx < 1 || d->ny < 1 || d->nz_local < 1 || d->z0_layer < 0 ||
      d->z0_layer + d->nz_local > d->nz_global)
    return fail(FK_EINVAL, "mesh dimensions nx=%d ny=%d nz_local=%d z0=%d nz_global=%d do not match",
                d->nx, d->ny, d->nz_local, d->z0_layer, d->nz_global);
  if (!(d->jac_det > 0.0) || !(d->jac_diag[0] > 0.0) || !(d->jac_diag[1] > 0.0) ||
      !(d->jac_diag[2] > 0.0))
    return fail(FK_EINVAL, "non-positive Jacobian");
  if (d->B == nullptr || d->G == nullptr || d->w == nullptr)
    return fail(FK_EINVAL, "basis tables B, G, w are required");
  if (d->variant < FK_VARIANT_AUTO || d->variant > FK_VARIANT_LAST)
    return fail(FK_EINVAL, "unknown variant %d", d->variant);

  fk_op* op = new fk_op();
  op->desc = *d;
  op->p = d->p;
  op->d = d->p + 1;
  op->q = d->q;
  op->nc = d->kind == FK_KIND_DIFFUSION ? 3 : 1;
  op->npa = d->kind == FK_KIND_DIFFUSION ? 6 : 1;
  op->npx = (int64_t)d->nx * d->p + 1;
  op->npy = (int64_t)d->ny * d->p + 1;
  op->npz_local = (int64_t)d->nz_local * d->p + 1;
  op->npz_global = (int64_t)d->nz_global * d->p + 1;
  op->nel = (int64_t)d->nx * d->ny * d->nz_local;
  op->ndof = op->npx * op->npy * op->npz_local;
  op->ndof_global = op->npx * op->npy * op->npz_global;
  op->dof_offset = (int64_t)d->z0_layer * d->p * op->npx * op->npy;
  if (op->ndof >= (int64_t)1 << 31 || op->nel * op->d * op->d * op->d >= ((int64_t)1 << 40)) {
    delete op;
    return fail(FK_EINVAL, "local problem too large for int32 dof ids (%lld dofs)",
                (long long)(op->ndof));
  }
  if (op->nel >= ((int64_t)1 << 31) - 64) {
    delete op;
    return fail(FK_EINVAL, "too many local elements");
  }
  const int qd = op->q * op->d;
  std::memcpy(op->B, d->B, sizeof(double) * qd);
  std::memcpy(op->G, d->G, sizeof(double) * qd);
  std::memcpy(op->w, d->w, sizeof(double) * op->q);
  for (int s = 0; s < 3; ++s) op->jinv[s] = 1.0 / d->jac_diag[s];
  if (d->gather_ids != nullptr) {
    const int64_t n = op->nel * op->d * op->d * op->d;
    op->host_gids.resize(n);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t g = d->gather_ids[i] - op->dof_offset;
      if (g < 0 || g >= op->ndof) {
        delete op;
        return fail(FK_EINVAL, "gather_ids[%lld]=%lld outside this rank's dofs", (long long)i,
                    (long long)d->gather_ids[i]);
      }
      op->host_gids[i] = (int)g;
    }
  }
  op->colour = d->deterministic != 0;
  if (op->colour && d->gather_ids != nullptr) {
    delete op;
    return fail(FK_EUNSUPPORTED, "the deterministic mode orders the box's elements by colour; "
                                 "it does not take a user gather map");
  }
  for (int c = 0; c < 8; ++c)
    op->colour_off[c + 1] = op->colour_off[c] + fk::colour_count(c, d->nx, d->ny, d->nz_local);
  op->device = d->device;
  op->stream = static_cast<cudaStream_t>(d->stream);
  op->comm = d->comm;
  {
    DeviceGuard g(op->device);
    cudaError_t e = cudaDeviceGetAttribute(&op->num_sms, cudaDevAttrMultiProcessorCount, op->device);
    if (e != cudaSuccess) {
      delete op;
      return fail(FK_ECUDA, "device %d: %s", d->device, cudaGetErrorString(e));
    }
  }
  int rc = select_kernel(op, d->variant);
  if (rc != FK_OK) {
    delete op;
    return rc;
  }
  *out = op;
  return FK_OK;
}

int fk_op_setup(fk_op* op) {
  if (op == nullptr) return fail(FK_EINVAL, "null handle");
  DeviceGuard g(op->device);
  const int d3 = op->d * op->d * op->d, q3 = op->q * op->q * op->q;
  cudaStream_t s = op->stream;
  op->ps = fk::pa_stride(op->npa, op->q);
  op->gs = fk::gid_stride(op->d);
  op->ms = fk::bits_stride(op->d);
  if (const char* c = std::getenv("FK_CFG")) op->cfg = std::atoi(c);
  // test hook: cap the persistent grid so small meshes run several batches per
  // CTA (exercises the cross-batch prefetch pipeline of pa_pipe.cuh)
  if (const char* c = std::getenv("FK_MAX_BLOCKS")) op->block_cap = std::max(1, std::atoi(c));
  if (op->gids == nullptr) FK_CUDA(cudaMalloc(&op->gids, sizeof(int) * (op->nel * op->gs + 16)));
  if (op->host_gids.empty()) {
    fk::restriction_kernel<<<grid_for(op->nel * op->gs, 256, op->num_sms), 256, 0, s>>>(
        op->gids, op->desc.nx, op->desc.ny, op->desc.nz_local, op->p, op->npx, op->npy, op->gs,
        op->colour ? 1 : 0);
    FK_CUDA(cudaGetLastError());
  } else {
    std::vector<int> padded(op->nel * op->gs, 0);
    for (int64_t e = 0; e < op->nel; ++e)
      std::memcpy(&padded[e * op->gs], &op->host_gids[e * d3], sizeof(int) * d3);
    FK_CUDA(cudaMemcpyAsync(op->gids, padded.data(), sizeof(int) * padded.size(),
                            cudaMemcpyHostToDevice, s));
    FK_CUDA(cudaStreamSynchronize(s));
  }
  // PA data, padded element stride (+64 bytes slack for 16-byte-granular copies)
  if (op->pa == nullptr) FK_CUDA(cudaMalloc(&op->pa, sizeof(double) * op->nel * op->ps + 64));
  double* dw = nullptr;
  FK_CUDA(cudaMalloc(&dw, sizeof(double) * op->q));
  FK_CUDA(cudaMemcpyAsync(dw, op->w, sizeof(double) * op->q, cudaMemcpyHostToDevice, s));
  fk::pa_data_kernel<<<grid_for(op->nel * q3, 256, op->num_sms), 256, 0, s>>>(
      op->pa, op->nel, op->q, op->npa, op->ps, dw, op->desc.jac_det, op->jinv[0], op->jinv[1],
      op->jinv[2]);
  FK_CUDA(cudaGetLastError());
  if (op->desc.dirichlet) {
    if (op->mask == nullptr) FK_CUDA(cudaMalloc(&op->mask, op->ndof));
    const int64_t ring = 2 * (op->npx + op->npy) * op->npz_local + 2 * op->npx * op->npy;
    if (op->ess == nullptr) FK_CUDA(cudaMalloc(&op->ess, sizeof(int) * (ring + 16)));
    unsigned long long* dn = nullptr;
    FK_CUDA(cudaMalloc(&dn, sizeof(unsigned long long)));
    FK_CUDA(cudaMemsetAsync(dn, 0, sizeof(unsigned long long), s));
    fk::dirichlet_kernel<<<grid_for(op->ndof, 256, op->num_sms), 256, 0, s>>>(
        op->mask, op->ess, dn, op->npx, op->npy, op->npz_local,
        (int64_t)op->desc.z0_layer * op->p, op->npz_global);
    FK_CUDA(cudaGetLastError());
    unsigned long long hn = 0;
    FK_CUDA(cudaMemcpyAsync(&hn, dn, sizeof(hn), cudaMemcpyDeviceToHost, s));
    FK_CUDA(cudaStreamSynchronize(s));
    op->n_ess = (int64_t)hn;
    cudaFree(dn);
    if (op->ebits == nullptr) FK_CUDA(cudaMalloc(&op->ebits, sizeof(uint32_t) * (op->nel * op->ms + 16)));
    fk::ebits_kernel<<<grid_for(op->nel * op->ms, 256, op->num_sms), 256, 0, s>>>(
        op->ebits, op->gids, op->mask, op->nel, d3, op->gs, op->ms);
    FK_CUDA(cudaGetLastError());
  }
  FK_CUDA(cudaStreamSynchronize(s));
  cudaFree(dw);
  if (op->ev0 == nullptr) {
    FK_CUDA(cudaEventCreate(&op->ev0));
    FK_CUDA(cudaEventCreate(&op->ev1));
    FK_CUDA(cudaEventCreate(&op->ev2));
    FK_CUDA(cudaEventCreate(&op->ev3));
  }
  if (op->comm) FK_TRY(fk::comm_setup(op));
  if (fk::multi_rank(op)) FK_TRY(preload_kernels(op));
  FK_TRY(ensure_reduce_ws(op));
  FK_CUDA(cudaStreamSynchronize(s));
  op->is_setup = true;
  return select_kernel(op, op->desc.variant);
}

int fk_op_destroy(fk_op* op) {
  if (op == nullptr) return FK_OK;
  DeviceGuard g(op->device);
  cudaFree(op->gids);
  cudaFree(op->pa);
  cudaFree(op->mask);
  cudaFree(op->ebits);
  cudaFree(op->ess);
  cudaFree(op->stage_x);
  cudaFree(op->stage_y);
  cudaFree(op->work);
  cudaFree(op->scal);
  cudaFree(op->partials);
  cudaFree(op->counter);
  cudaFree(op->hist);
  cudaFree(op->qf_part);
  cudaFree(op->diag_tab);
  cudaFree(op->halo);
  if (op->comm_stream) cudaStreamDestroy(op->comm_stream);
  if (op->ev_bnd) cudaEventDestroy(op->ev_bnd);
  if (op->ev_xchg) cudaEventDestroy(op->ev_xchg);
  if (op->ev0) cudaEventDestroy(op->ev0);
  if (op->ev1) cudaEventDestroy(op->ev1);
  if (op->ev2) cudaEventDestroy(op->ev2);
  if (op->ev3) cudaEventDestroy(op->ev3);
  if (op->cg_stream) cudaStreamDestroy(op->cg_stream);
  if (op->h2d) cudaStreamDestroy(op->h2d);
  if (op->d2h) cudaStreamDestroy(op->d2h);
  for (auto& e : op->chunk_ev)
    if (e) cudaEventDestroy(e);
  delete op;
  return FK_OK;
}

int fk_op_get_info(const fk_op* op, fk_op_info* info) {
  if (op == nullptr || info == nullptr) return fail(FK_EINVAL, "null argument");
  info->ndof_local = op->ndof;
  info->nel_local = op->nel;
  info->dof_offset = op->dof_offset;
  info->ndof_global = op->ndof_global;
  info->pa_bytes = (int64_t)sizeof(double) * op->nel * op->npa * op->q * op->q * op->q;
  info->variant = op->variant;
  info->elems_per_block = op->kern ? op->kern->E : 0;
  info->threads_per_block = op->kern ? op->kern->T : 0;
  info->blocks = op->blocks;
  info->cfg = op->kern ? op->kern->cfg : -1;
  return FK_OK;
}

// Switch variant / launch geometry; on failure the handle keeps the kernel,
// variant and cfg it had (select_kernel commits only when it succeeds).
static int reselect(fk_op* op, int variant, int cfg) {
  const int old_cfg = op->cfg;
  op->cfg = cfg;
  int rc = select_kernel(op, variant);
  if (rc != FK_OK) {
    op->cfg = old_cfg;
    return rc;
  }
  op->desc.variant = variant;
  return FK_OK;
}

int fk_op_set_variant(fk_op* op, int variant) {
  if (op == nullptr) return fail(FK_EINVAL, "null handle");
  if (variant < FK_VARIANT_AUTO || variant > FK_VARIANT_LAST)
    return fail(FK_EINVAL, "unknown variant %d", variant);
  return reselect(op, variant, -1);
}

int fk_op_set_config(fk_op* op, int variant, int cfg) {
  if (op == nullptr) return fail(FK_EINVAL, "null handle");
  if (variant < FK_VARIANT_DFMA || variant > FK_VARIANT_LAST || cfg < 0)
    return fail(FK_EINVAL, "bad variant %d / cfg %d", variant, cfg);
  if (fk::find_kernel_cfg(op->nc, op->d, op->q, variant, cfg) == nullptr)
    return fail(FK_EUNSUPPORTED, "no launch config %d for variant %d", cfg, variant);
  return reselect(op, variant, cfg);
}

int fk_op_restriction(fk_op* op, int64_t* host_out) {
  if (op == nullptr || host_out == nullptr) return fail(FK_EINVAL, "null argument");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  DeviceGuard g(op->device);
  const int d3 = op->d * op->d * op->d;
  std::vector<int> tmp(op->nel * op->gs);
  FK_CUDA(cudaMemcpyAsync(tmp.data(), op->gids, sizeof(int) * tmp.size(), cudaMemcpyDeviceToHost,
                          op->stream));
  FK_CUDA(cudaStreamSynchronize(op->stream));
  for (int64_t s = 0; s < op->nel; ++s) {
    // rows are in the reference's element order except in the colour order
    const int64_t e = op->colour ? fk::colour_element(s, op->desc.nx, op->desc.ny, op->desc.nz_local) : s;
    for (int l = 0; l < d3; ++l) host_out[e * d3 + l] = (int64_t)tmp[s * op->gs + l] + op->dof_offset;
  }
  return FK_OK;
}

int fk_op_pa_data(fk_op* op, double* host_out) {
  if (op == nullptr || host_out == nullptr) return fail(FK_EINVAL, "null argument");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  DeviceGuard g(op->device);
  const size_t row = sizeof(double) * op->npa * op->q * op->q * op->q;
  FK_CUDA(cudaMemcpy2DAsync(host_out, row, op->pa, sizeof(double) * op->ps, row, op->nel,
                            cudaMemcpyDeviceToHost, op->stream));
  FK_CUDA(cudaStreamSynchronize(op->stream));
  return FK_OK;
}

int fk_op_apply(fk_op* op, const double* x, double* y) {
  if (op == nullptr || x == nullptr || y == nullptr) return fail(FK_EINVAL, "null argument");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  if (x == y) return fail(FK_EINVAL, "in-place apply is not supported (x == y)");
  DeviceGuard g(op->device);
  return apply_full(op, x, y);
}

int fk_op_apply_local(fk_op* op, const double* x, double* y) {
  if (op == nullptr || x == nullptr || y == nullptr) return fail(FK_EINVAL, "null argument");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  DeviceGuard g(op->device);
  return launch_local(op, x, y);
}

int fk_op_apply_host(fk_op* op, const double* xh, double* yh) {
  if (op == nullptr || xh == nullptr || yh == nullptr) return fail(FK_EINVAL, "null argument");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  DeviceGuard g(op->device);
  const size_t bytes = sizeof(double) * op->ndof;
  if (op->stage_x == nullptr) {
    FK_CUDA(cudaMalloc(&op->stage_x, bytes));
    FK_CUDA(cudaMalloc(&op->stage_y, bytes));
  }
  const int nzl = op->desc.nz_local;
  if (op->comm != nullptr || op->desc.dirichlet || op->colour || nzl < 4 || op->kern == nullptr) {
    FK_CUDA(cudaMemcpyAsync(op->stage_x, xh, bytes, cudaMemcpyHostToDevice, op->stream));
    FK_TRY(apply_full(op, op->stage_x, op->stage_y));
    FK_CUDA(cudaMemcpyAsync(yh, op->stage_y, bytes, cudaMemcpyDeviceToHost, op->stream));
    FK_CUDA(cudaStreamSynchronize(op->stream));
    return FK_OK;
  }
  // z-chunk pipeline: chunk c's x planes go up while chunk c-1 computes and the
  // completed y planes of chunk c-2 come down (PCIe is full duplex).  Dof
  // planes are z-slowest (mesh.py:164): chunk of element layers [z0, z1) reads
  // planes [z0 p, z1 p] and finalises every plane below z1 p.
  if (op->h2d == nullptr) {
    FK_CUDA(cudaStreamCreateWithFlags(&op->h2d, cudaStreamNonBlocking));
    FK_CUDA(cudaStreamCreateWithFlags(&op->d2h, cudaStreamNonBlocking));
    for (auto& e : op->chunk_ev) FK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  int K = std::min(nzl, 8);  // tools/pcie_probe.py: 8 ramped chunks measured best
  if (const char* c = std::getenv("FK_HOST_CHUNKS")) K = std::max(1, std::min({nzl, std::atoi(c), 15}));
  const int64_t P = op->npx * op->npy, nxy = (int64_t)op->desc.nx * op->desc.ny;
  const int p = op->p;
  FK_CUDA(cudaEventRecord(op->chunk_ev[30], op->stream));  // order after prior work
  FK_CUDA(cudaStreamWaitEvent(op->h2d, op->chunk_ev[30], 0));
  FK_CUDA(cudaMemsetAsync(op->stage_y, 0, bytes, op->stream));
  int64_t x_done = 0, y_done = 0;
  // chunk boundaries on a smoothstep ramp: small first and last chunks shorten
  // the pipeline fill (H2D before the first compute) and drain (compute + D2H
  // after the last H2D); FK_HOST_RAMP=0 gives uniform chunks
  const char* ramp_env = std::getenv("FK_HOST_RAMP");
  const bool ramp = !(ramp_env && ramp_env[0] == '0');
  auto zb = [&](int c) {
    if (c <= 0) return 0;
    if (c >= K) return nzl;
    const double t = (double)c / K, f = ramp ? t * t * (3.0 - 2.0 * t) : t;
    return std::min(nzl, std::max(1, (int)std::lround(f * nzl)));
  };
  // FK_HOST_TRACE=1: timing events per chunk and stream, printed to stderr
  // (tools/pcie_probe.py; diagnosis only)
  const bool trace = std::getenv("FK_HOST_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto tmark = [&](cudaStream_t s) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    tev.push_back(e);
  };
  tmark(op->stream);
  for (int c = 0; c < K; ++c) {
    const int z0 = zb(c), z1 = zb(c + 1);
    if (z1 <= z0) continue;
    const int64_t x_hi = (int64_t)z1 * p + 1;
    FK_CUDA(cudaMemcpyAsync(op->stage_x + x_done * P, xh + x_done * P,
                            sizeof(double) * (x_hi - x_done) * P, cudaMemcpyHostToDevice, op->h2d));
    x_done = x_hi;
    tmark(op->h2d);
    FK_CUDA(cudaEventRecord(op->chunk_ev[2 * c], op->h2d));
    FK_CUDA(cudaStreamWaitEvent(op->stream, op->chunk_ev[2 * c], 0));
    tmark(op->stream);
    FK_TRY(launch_range(op, op->stage_x, op->stage_y, (int64_t)z0 * nxy, (int64_t)(z1 - z0) * nxy,
                        op->stream));
    tmark(op->stream);
    FK_CUDA(cudaEventRecord(op->chunk_ev[2 * c + 1], op->stream));
    FK_CUDA(cudaStreamWaitEvent(op->d2h, op->chunk_ev[2 * c + 1], 0));
    const int64_t y_hi = (z1 == nzl) ? op->npz_local : (int64_t)z1 * p;
    FK_CUDA(cudaMemcpyAsync(yh + y_done * P, op->stage_y + y_done * P,
                            sizeof(double) * (y_hi - y_done) * P, cudaMemcpyDeviceToHost, op->d2h));
    y_done = y_hi;
    tmark(op->d2h);
  }
  FK_CUDA(cudaStreamSynchronize(op->d2h));
  if (trace) {
    cudaDeviceSynchronize();
    std::string line = "[fk host trace ms] ";
    for (size_t i = 1; i < tev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      const char* kind = (i - 1) % 4 == 0 ? "h2d" : (i - 1) % 4 == 1 ? "cs" : (i - 1) % 4 == 2 ? "ce" : "d2h";
      char b[48];
      snprintf(b, sizeof(b), "%s%zu=%.3f ", kind, (i - 1) / 4, ms);
      line += b;
    }
    fprintf(stderr, "%s\n", line.c_str());
    for (auto e : tev) cudaEventDestroy(e);
  }
  return FK_OK;
}

// 1D factor tables of the closed-form box diagonal (fk_cg.cuh BoxDiag):
// f(i) = sum_a w_a T[a][i]^2 (T = B, G), assembled over the elements holding
// a node: x and y over the box, z over the GLOBAL element layers at this
// rank's planes (a shared plane gets both layers' contributions on both ranks)
static int ensure_box_tab(fk_op* op) {
  if (op->diag_tab != nullptr) return FK_OK;
  const int d = op->d, q = op->q, p = op->p;
  double fb[9] = {}, fg[9] = {};
  for (int i = 0; i < d; ++i)
    for (int a = 0; a < q; ++a) {
      fb[i] += op->w[a] * (op->B[a * d + i] * op->B[a * d + i]);
      fg[i] += op->w[a] * (op->G[a * d + i] * op->G[a * d + i]);
    }
  const int64_t z0p = (int64_t)op->desc.z0_layer * p;
  std::vector<double> h(2 * (op->npx + op->npy + op->npz_local), 0.0);
  auto assemble = [&](double* out, int64_t n, int64_t g0, int64_t nglob, const double* f) {
    for (int64_t l = 0; l < n; ++l) {
      const int64_t g = g0 + l;
      double v = 0.0;
      if (g % p != 0) v = f[g % p];
      else {
        if (g > 0) v += f[p];
        if (g < nglob - 1) v += f[0];
      }
      out[l] = v;
    }
  };
  double* t = h.data();
  assemble(t, op->npx, 0, op->npx, fb);
  assemble(t + op->npx, op->npx, 0, op->npx, fg);
  t += 2 * op->npx;
  assemble(t, op->npy, 0, op->npy, fb);
  assemble(t + op->npy, op->npy, 0, op->npy, fg);
  t += 2 * op->npy;
  assemble(t, op->npz_local, z0p, op->npz_global, fb);
  assemble(t + op->npz_local, op->npz_local, z0p, op->npz_global, fg);
  FK_CUDA(cudaMalloc(&op->diag_tab, sizeof(double) * h.size()));
  FK_CUDA(cudaMemcpyAsync(op->diag_tab, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice,
                          op->stream));
  FK_CUDA(cudaStreamSynchronize(op->stream));
  return FK_OK;
}

static void div_magic32(int d, unsigned& m, int& s) {
  s = 0;
  while ((1ll << s) < d) ++s;
  m = (unsigned)((((1ull << 32) * ((1ull << s) - (unsigned long long)d)) / (unsigned long long)d) + 1);
}

static fk::BoxDiag box_diag(const fk_op* op) {
  fk::BoxDiag b;
  b.tab = op->diag_tab;
  b.npx = (int)op->npx;
  b.npy = (int)op->npy;
  b.npz = (int)op->npz_local;
  b.nc = op->nc;
  const double dj = op->desc.jac_det;
  b.c0 = dj * (op->jinv[0] * op->jinv[0]);
  b.c1 = dj * (op->jinv[1] * op->jinv[1]);
  b.c2 = dj * (op->jinv[2] * op->jinv[2]);
  b.cm = dj;
  b.dirichlet = op->desc.dirichlet ? 1 : 0;
  b.z0p = op->desc.z0_layer * op->p;
  b.npzg = (int)op->npz_global;
  div_magic32(b.npx, b.mx, b.sx);
  div_magic32(b.npy, b.my, b.sy);
  return b;
}

int fk_op_diagonal(fk_op* op, double* diag) {
  if (op == nullptr || diag == nullptr) return fail(FK_EINVAL, "null argument");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  DeviceGuard g(op->device);
  if (op->host_gids.empty()) {
    // structured box: separable closed form, one pass, no atomics and no
    // exchange (the z factor is assembled over the global layers)
    FK_TRY(ensure_box_tab(op));
    fk::diag_box_rn_kernel<<<grid_for(op->ndof, 256, op->num_sms), 256, 0, op->stream>>>(
        diag, box_diag(op), op->ndof);
    FK_CUDA(cudaGetLastError());
    return FK_OK;
  }
  FK_CUDA(cudaMemsetAsync(diag, 0, sizeof(double) * op->ndof, op->stream));
  const fk::KernelEntry* k = fk::find_kernel(op->nc, op->d, op->q, FK_VARIANT_DFMA);
  if (k == nullptr || k->diag == nullptr) return fail(FK_EUNSUPPORTED, "no diagonal kernel");
  if (op->colour) {
    for (int c = 0; c < 8; ++c) {
      const int64_t e0 = op->colour_off[c], ne = op->colour_off[c + 1] - e0;
      if (ne == 0) continue;
      fk::OpView v = view(op);
      v.gids += e0 * op->gs;
      v.pa += e0 * op->ps;
      k->diag(v, diag, ne, (int)std::min<int64_t>(ne, (int64_t)op->num_sms * 16), op->stream);
    }
  } else {
    k->diag(view(op), diag, op->nel, (int)std::min<int64_t>(op->nel, (int64_t)op->num_sms * 16),
            op->stream);
  }
  FK_CUDA(cudaGetLastError());
  if (op->comm) FK_TRY(fk::exchange_interface(op, diag, op->stream));
  if (op->desc.dirichlet && op->n_ess > 0) {
    fk::ess_set_kernel<<<grid_for(op->n_ess, 256, op->num_sms), 256, 0, op->stream>>>(
        diag, op->ess, op->n_ess, 1.0);
    FK_CUDA(cudaGetLastError());
  }
  return FK_OK;
}

int fk_op_set_essential(fk_op* op, double* v, double value) {
  if (op == nullptr || v == nullptr) return fail(FK_EINVAL, "null argument");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  if (!op->desc.dirichlet || op->n_ess == 0) return FK_OK;
  DeviceGuard g(op->device);
  fk::ess_set_kernel<<<grid_for(op->n_ess, 256, op->num_sms), 256, 0, op->stream>>>(v, op->ess,
                                                                                    op->n_ess, value);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}


static int red_blocks(const fk_op* op) { return std::min(op->num_sms * 4, 4096); }

int fk_dot(fk_op* op, const double* a, const double* b, double* host_out) {
  if (op == nullptr || a == nullptr || b == nullptr || host_out == nullptr)
    return fail(FK_EINVAL, "null argument");
  DeviceGuard g(op->device);
  FK_TRY(ensure_reduce_ws(op));
  const int64_t n0 = fk::owned_begin(op);
  fk::dot_kernel<<<red_blocks(op), fk::kRedThreads, 0, op->stream>>>(
      a, b, n0, op->ndof, op->partials, op->counter, op->scal + fk::S_DOT);
  FK_CUDA(cudaGetLastError());
  if (op->comm) FK_TRY(fk::allreduce_scalar(op, op->scal + fk::S_DOT, op->stream));
  FK_CUDA(cudaMemcpyAsync(host_out, op->scal + fk::S_DOT, sizeof(double), cudaMemcpyDeviceToHost,
                          op->stream));
  FK_CUDA(cudaStreamSynchronize(op->stream));
  return FK_OK;
}

// One CG iteration, enqueued on stream s (capturable).  With an EO / MF
// kernel, p.Ap comes out of the apply itself (per-CTA quadratic-form
// partials, summed in fixed order); otherwise a dot pass over p and Ap.
static int cg_iteration(fk_op* op, double* x, cudaStream_t s) {
  const int64_t n = op->ndof, n0 = fk::owned_begin(op);
  double* r = op->work;
  double* p = r + 2 * n;
  double* Ap = p + n;
  double* dinv = Ap + n;
  int* iscal = reinterpret_cast<int*>(op->scal + 16);
  const int rb = red_blocks(op);
  const bool qf = op->kern->launch_qf != nullptr && op->qf_part != nullptr;
  if (qf) {
    FK_CUDA(cudaMemsetAsync(op->qf_part, 0, sizeof(double) * 8 * op->max_blocks, s));
    op->qf_on = true;
    op->qf_seg = 0;
  }
  const int rc = apply_full(op, p, Ap, s);
  op->qf_on = false;
  FK_TRY(rc);
  if (qf)
    fk::qf_sum_kernel<<<1, fk::kRedThreads, 0, s>>>(op->qf_part, (int64_t)op->qf_seg * op->max_blocks,
                                                   op->scal + fk::S_DEN);
  else
    fk::dot_kernel<<<rb, fk::kRedThreads, 0, s>>>(p, Ap, n0, n, op->partials, op->counter,
                                                  op->scal + fk::S_DEN);
  if (op->comm) FK_TRY(fk::allreduce_scalar(op, op->scal + fk::S_DEN, s));
  fk::cg_alpha_kernel<<<1, 1, 0, s>>>(op->scal, iscal);
  fk::cg_residual_kernel<<<rb, fk::kRedThreads, 0, s>>>(r, Ap, dinv, n, n0, op->scal, iscal,
                                                        op->partials, op->counter + 1,
                                                        op->scal + fk::S_BN);
  if (op->comm) FK_TRY(fk::allreduce_scalar(op, op->scal + fk::S_BN, s));
  fk::cg_finish_kernel<<<1, 1, 0, s>>>(op->scal, iscal, op->hist);
  fk::cg_step_kernel<<<grid_for(n, 256, op->num_sms), 256, 0, s>>>(x, p, r, dinv, n, op->scal, iscal);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}

int fk_cg_prepare(fk_op* op, int iters) {
  if (op == nullptr) return fail(FK_EINVAL, "null handle");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  if (iters < 0) return fail(FK_EINVAL, "iters must be >= 0");
  DeviceGuard g(op->device);
  if (op->work == nullptr) FK_CUDA(cudaMalloc(&op->work, sizeof(double) * 5 * op->ndof));
  FK_TRY(ensure_reduce_ws(op));
  if (op->hist_cap < iters + 1) {
    if (op->hist) FK_CUDA(cudaFree(op->hist));
    op->hist = nullptr;
    FK_CUDA(cudaMalloc(&op->hist, sizeof(double) * (iters + 1)));
    op->hist_cap = iters + 1;
  }
  if (op->cg_stream == nullptr) FK_CUDA(cudaStreamCreateWithFlags(&op->cg_stream, cudaStreamNonBlocking));
  if (op->qf_part == nullptr && op->max_blocks > 0)
    FK_CUDA(cudaMalloc(&op->qf_part, sizeof(double) * 8 * op->max_blocks));
  return FK_OK;
}

int fk_cg_solve(fk_op* op, const double* b, double* x, int iters, double rtol, double* hist_host,
                int* iters_done) {
  if (op == nullptr || b == nullptr || x == nullptr) return fail(FK_EINVAL, "null argument");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  if (iters < 0) return fail(FK_EINVAL, "iters must be >= 0");
  DeviceGuard g(op->device);
  const int64_t n = op->ndof;
  FK_TRY(fk_cg_prepare(op, iters));
  cudaStream_t s = op->cg_stream;
  // order after the caller's stream
  FK_CUDA(cudaEventRecord(op->ev0, op->stream));
  FK_CUDA(cudaStreamWaitEvent(s, op->ev0, 0));
  double* r = op->work;
  double* z = r + n;
  double* p = z + n;
  double* dinv = p + 2 * n;
  int* iscal = reinterpret_cast<int*>(op->scal + 16);
  // Jacobi: dinv = 1/diag(A) (ones on essential dofs)
  {
    cudaStream_t saved = op->stream;
    op->stream = s;
    int rc = fk_op_diagonal(op, z);
    op->stream = saved;
    FK_TRY(rc);
  }
  fk::recip_kernel<<<grid_for(n, 256, op->num_sms), 256, 0, s>>>(dinv, z, n);
  const int64_t n0 = fk::owned_begin(op);
  fk::cg_init_kernel<<<red_blocks(op), fk::kRedThreads, 0, s>>>(
      b, x, r, p, dinv, n, n0, op->partials, op->counter + 2, op->scal + fk::S_NOM);
  if (op->comm) FK_TRY(fk::allreduce_scalar(op, op->scal + fk::S_NOM, s));
  fk::cg_start_kernel<<<1, 1, 0, s>>>(op->scal, iscal, op->hist, rtol);
  FK_CUDA(cudaGetLastError());
  if (iters > 0) {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool use_graph = true;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      int rc = cg_iteration(op, x, s);
      cudaError_t ce = cudaStreamEndCapture(s, &graph);
      if (rc != FK_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (ce != cudaSuccess || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
        use_graph = false;
        cudaGetLastError();
      }
    } else {
      use_graph = false;
      cudaGetLastError();
    }
    for (int it = 0; it < iters; ++it) {
      if (use_graph) {
        FK_CUDA(cudaGraphLaunch(exec, s));
      } else {
        FK_TRY(cg_iteration(op, x, s));
      }
    }
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
  int hi[2] = {0, 0};
  FK_CUDA(cudaMemcpyAsync(hi, iscal, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
  FK_CUDA(cudaStreamSynchronize(s));
  const int done_it = hi[fk::I_IT];
  if (hist_host) {
    FK_CUDA(cudaMemcpyAsync(hist_host, op->hist, sizeof(double) * (done_it + 1),
                            cudaMemcpyDeviceToHost, s));
    FK_CUDA(cudaStreamSynchronize(s));
  }
  if (iters_done) *iters_done = done_it;
  // make the caller's stream see the result
  FK_CUDA(cudaEventRecord(op->ev1, s));
  FK_CUDA(cudaStreamWaitEvent(op->stream, op->ev1, 0));
  return FK_OK;
}

int fk_op_time_apply(fk_op* op, const double* x, double* y, int reps, const void* flush,
                     size_t flush_bytes, double* ms_apply, double* ms_kernel) {
  if (op == nullptr || x == nullptr || y == nullptr || reps < 1) return fail(FK_EINVAL, "bad argument");
  if (!op->is_setup) return fail(FK_EINVAL, "fk_op_setup has not been called");
  DeviceGuard g(op->device);
  // all reps enqueued back to back (no host sync in between), so the events
  // see steady-state launches, not the host's launch latency after an idle GPU
  std::vector<cudaEvent_t> ev(4 * (size_t)reps);
  for (auto& e : ev) FK_CUDA(cudaEventCreate(&e));
  int rc = FK_OK;
  for (int r = 0; r < reps && rc == FK_OK; ++r) {
    cudaEvent_t* e = ev.data() + 4 * r;
    if (flush && flush_bytes)
      FK_CUDA(cudaMemsetAsync(const_cast<void*>(flush), r & 0xff, flush_bytes, op->stream));
    FK_CUDA(cudaEventRecord(e[0], op->stream));
    FK_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * op->ndof, op->stream));
    FK_CUDA(cudaEventRecord(e[1], op->stream));
    FK_TRY(launch_all(op, x, y, op->stream));
    FK_CUDA(cudaEventRecord(e[2], op->stream));
    if (op->comm) rc = fk::exchange_interface(op, y, op->stream);
    if (op->desc.dirichlet && op->n_ess > 0)
      fk::ess_copy_kernel<<<grid_for(op->n_ess, 256, op->num_sms), 256, 0, op->stream>>>(
          y, x, op->ess, op->n_ess);
    FK_CUDA(cudaEventRecord(e[3], op->stream));
  }
  // medians over the reps (robust to a stray slow rep, e.g. a clock change)
  std::vector<float> ta(reps), tk(reps);
  if (rc == FK_OK) {
    FK_CUDA(cudaEventSynchronize(ev[4 * (size_t)reps - 1]));
    for (int r = 0; r < reps; ++r) {
      FK_CUDA(cudaEventElapsedTime(&ta[r], ev[4 * r], ev[4 * r + 3]));
      FK_CUDA(cudaEventElapsedTime(&tk[r], ev[4 * r + 1], ev[4 * r + 2]));
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc != FK_OK) return rc;
  std::sort(ta.begin(), ta.end());
  std::sort(tk.begin(), tk.end());
  if (ms_apply) *ms_apply = ta[reps / 2];
  if (ms_kernel) *ms_kernel = tk[reps / 2];
  return FK_OK;
}

}  // extern "C"
