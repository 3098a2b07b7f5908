// fk_internal.h — internal structures of libfk_b200 (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/fk.h"

namespace fk {

struct OpView;  // what a kernel launcher needs
using LaunchFn = void (*)(const OpView&, const double* x, double* y, int blocks, cudaStream_t s);
using DiagFn = void (*)(const OpView&, double* diag, int64_t nel, int blocks, cudaStream_t s);

struct KernelEntry {
  int nc = 0, d = 0, q = 0, variant = 0, cfg = 0;
  int E = 0, T = 0;
  bool persist = true;  // persistent grid (batches strided over CTAs) or one batch per CTA
  bool structured = false;  // ids from the closed-form box restriction (no user gather map)
  LaunchFn launch_qf = nullptr;  // twin with the element quadratic form (OpView::qf), CG only
  const void* func_qf = nullptr;
  size_t smem = 0;
  const void* func = nullptr;
  const void* diag_func = nullptr;  // the assembled-diagonal kernel of this (d, q, nc)
  LaunchFn launch = nullptr;
  DiagFn diag = nullptr;
};

struct OpView {
  const double* B;  // host tables (q*d)
  const double* G;
  const int* gids;
  const double* pa;
  const uint32_t* ebits;  // per-element Dirichlet bits (nullptr: none)
  int nel;
  const double* w;  // host quadrature weights (q), |J| and 1/jac_diag: MF kernels
  double detj;
  double jinv[3];
  // closed-form restriction (GM = 1 kernels): slab sizes and the first element
  // of this launch within the rank's slab
  int nx, ny, p;
  int64_t npx, npy, e0;
  double* qf = nullptr;  // QF-capable kernels: per-CTA quadratic-form partials
};

// Host mirror of GlobalLayout (pa_common.cuh): padded per-element strides.
// PA element stride: even (16-byte bulk-copy granules) and = q^2 (+1) mod 16,
// so the stage-C lines of consecutive elements of a batch (q^2 per element)
// continue the bank sequence instead of colliding (tools/smem_strides.py)
inline int64_t pa_stride(int npa, int q) {
  int64_t n = ((int64_t)npa * q * q * q + 1) / 2 * 2;
  while (((n - q * q) % 16 + 16) % 16 > 1) n += 2;
  return n;
}
// Colour-major element order of the deterministic mode: colour c = cx + 2 cy
// + 4 cz holds the elements with (ex, ey, ez) = (cx, cy, cz) mod 2, each
// colour lexicographic (x fastest).  Slot s of colour c (t = s - off[c]):
// ex = cx + 2 (t % nxc), ey = cy + 2 ((t / nxc) % nyc), ez = cz + 2 (t / (nxc nyc)),
// nxc = (nx + 1 - cx) / 2 etc.
__host__ __device__ inline int64_t colour_count(int c, int nx, int ny, int nz) {
  return (int64_t)((nx + 1 - (c & 1)) / 2) * ((ny + 1 - ((c >> 1) & 1)) / 2) *
         ((nz + 1 - (c >> 2)) / 2);
}
__host__ __device__ inline int64_t colour_element(int64_t s, int nx, int ny, int nz) {
  int c = 0;
  int64_t off = 0;
  for (; c < 7; ++c) {
    const int64_t n = colour_count(c, nx, ny, nz);
    if (s < off + n) break;
    off += n;
  }
  const int64_t t = s - off;
  const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
  const int64_t nxc = (nx + 1 - cx) / 2, nyc = (ny + 1 - cy) / 2;
  const int64_t ex = cx + 2 * (t % nxc), ey = cy + 2 * ((t / nxc) % nyc), ez = cz + 2 * (t / (nxc * nyc));
  return ex + (int64_t)nx * (ey + (int64_t)ny * ez);
}

inline int64_t gid_stride(int d) { return ((int64_t)d * d * d + 3) / 4 * 4; }
inline int64_t bits_stride(int d) { return (((int64_t)d * d * d + 31) / 32 + 3) / 4 * 4; }

// Mirror symmetry of a 1D table pair, B[q-1-a][d-1-i] = B[a][i] and
// G[q-1-a][d-1-i] = -G[a][i] (G may be null), to 128 ulp of the table
// maximum — the rounding of Basis1D.nodal's own tables (fk_api.cu:
// tables_symmetric); the even-odd folded kernels need it.
inline bool mirror_symmetric(const double* B, const double* G, int q, int d) {
  double mb = 0.0, mg = 0.0, eb = 0.0, eg = 0.0;
  for (int a = 0; a < q; ++a)
    for (int i = 0; i < d; ++i) {
      const int j = (q - 1 - a) * d + (d - 1 - i);
      mb = mb > __builtin_fabs(B[a * d + i]) ? mb : __builtin_fabs(B[a * d + i]);
      eb = eb > __builtin_fabs(B[a * d + i] - B[j]) ? eb : __builtin_fabs(B[a * d + i] - B[j]);
      if (G) {
        mg = mg > __builtin_fabs(G[a * d + i]) ? mg : __builtin_fabs(G[a * d + i]);
        eg = eg > __builtin_fabs(G[a * d + i] + G[j]) ? eg : __builtin_fabs(G[a * d + i] + G[j]);
      }
    }
  const double tol = 128.0 * 2.220446049250313e-16;
  return eb <= tol * mb && eg <= tol * mg;
}

const KernelEntry* find_kernel_cfg(int nc, int d, int q, int variant, int cfg);

void register_kernels(std::vector<KernelEntry>& out);  // pa_instances*.cu
const KernelEntry* find_kernel(int nc, int d, int q, int variant);

}  // namespace fk

namespace fk {
constexpr int kMaxRanks = 16;

// Per-rank mailbox of the peer-memory transport (fk_comm.cu), one device
// allocation: control words, then the two halo planes.  Neighbours write into
// it over NVLink (P2P stores through UVA or CUDA-IPC mappings); all flags are
// monotone counters of completed exchanges / reductions, so the protocol
// replays inside CUDA graphs without host involvement.
struct Mailbox {
  unsigned long long recv_flag[2];        // [0] plane from the rank below arrived, [1] from above
  unsigned long long consumed[2];         // [0] the rank below has consumed my plane, [1] above
  unsigned long long red_flag[kMaxRanks]; // reduction contribution of rank j arrived
  unsigned long long seq_x, seq_r;        // completed exchanges / reductions (owner only)
  unsigned int put_done, add_done;        // last-CTA counters of the put / add kernels
  unsigned int pad[2];
  double red_slot[2][kMaxRanks];          // contributions, double-buffered by parity
};
constexpr size_t kMailboxHeader = (sizeof(Mailbox) + 255) / 256 * 256;

struct PeerTable {
  Mailbox* box[kMaxRanks];  // every rank's mailbox as addressable from this rank
};
}  // namespace fk

struct fk_comm {
  int transport = FK_TRANSPORT_NCCL;
  void* nccl = nullptr;  // ncclComm_t
  int rank = 0, nranks = 1, device = 0;
  // peer-memory transport
  fk::Mailbox* box = nullptr;  // own mailbox (device)
  fk::PeerTable peers{};
  int64_t plane_cap = 0;       // doubles per halo plane
  bool ipc_mapped[fk::kMaxRanks] = {};
};

struct fk_op {
  fk_op_desc desc{};
  int p = 0, d = 0, q = 0, nc = 0, npa = 0;
  int64_t npx = 0, npy = 0, npz_local = 0, npz_global = 0;
  int64_t nel = 0, ndof = 0, dof_offset = 0, ndof_global = 0;
  double B[100], G[100], w[10];
  double jinv[3];
  std::vector<int> host_gids;  // optional user map (local ids)
  bool colour = false;         // deterministic mode: colour-major element order
  int64_t colour_off[9] = {};  // element range [colour_off[c], colour_off[c+1]) of colour c
  cudaStream_t stream = nullptr;  // user stream
  cudaStream_t cg_stream = nullptr;
  int device = 0, num_sms = 0;
  int variant = FK_VARIANT_AUTO;
  const fk::KernelEntry* kern = nullptr;
  int blocks = 0;
  bool is_setup = false;
  // device data
  int* gids = nullptr;
  double* pa = nullptr;
  unsigned char* mask = nullptr;
  uint32_t* ebits = nullptr;
  int64_t ps = 0, gs = 0, ms = 0;  // padded strides (doubles, ints, words)
  int cfg = -1;                    // launch-geometry override (FK_CFG)
  int* ess = nullptr;
  int64_t n_ess = 0;
  // host staging for fk_op_apply_host (z-chunk pipeline: H2D / compute / D2H)
  double* stage_x = nullptr;
  double* stage_y = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t chunk_ev[32] = {};
  int max_blocks = 0;  // resident CTAs of the fused kernel on the device
  int block_cap = 0;   // FK_MAX_BLOCKS test hook (0: none)
  // CG / reduction workspace
  double* work = nullptr;  // r, z, p, Ap, dinv (5 * ndof)
  double* scal = nullptr;  // scalars
  double* partials = nullptr;
  unsigned* counter = nullptr;
  double* hist = nullptr;
  int hist_cap = 0;
  // CG: p.Ap as the fused kernel's quadratic form (per-CTA partials of up to 8
  // launches per apply: the colour launches / the overlapped layer ranges)
  double* qf_part = nullptr;
  double* diag_tab = nullptr;  // assembled 1D factors of the closed-form box diagonal
  bool qf_on = false;
  int qf_seg = 0;
  // multi-rank
  fk_comm* comm = nullptr;
  double* halo = nullptr;  // receive buffers (2 planes)
  cudaStream_t comm_stream = nullptr;           // NCCL plane exchange (overlaps interior elements)
  cudaEvent_t ev_bnd = nullptr, ev_xchg = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
};
