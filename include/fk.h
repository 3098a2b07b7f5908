/*
 * fk.h — C-ABI of the B200 partial-assembly (PA) operator library
 * (libfk_b200.so, built from paper_2603_09038_b200/csrc).
 *
 * This is the drop-in boundary for the hot path the reference package
 * feklab composes on the CPU (/root/reference/pkg/src/feklab):
 *
 *   gather (mesh.py:130-131) -> B/G contractions (tensor.py:220-283)
 *   -> pointwise PA data D (operator.py:132-193) -> B^T/G^T contractions
 *   -> scatter_add (mesh.py:133-137)
 *
 * fused into one sm_100a kernel per operator (BP1 mass / BP3 diffusion) and
 * order p = 1..8, plus the Jacobi-PCG solve that calls it and the z-slab
 * interface exchange for multi-GPU runs.  Plain pointers and sizes only; no
 * torch types.  Device pointers are FP64, contiguous, on the handle's device.
 *
 * Errors: every call returns FK_OK (0) or a negative code; the message of the
 * last failing call on this thread is fk_last_error().  A handle is not
 * thread-safe; all work is enqueued on the handle's stream and calls return
 * without synchronising unless stated.
 */
#ifndef FK_B200_H
#define FK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FK_API_VERSION 2

#define FK_OK 0
#define FK_EINVAL (-1)      /* invalid argument / shape ("... do not match ...") */
#define FK_ECUDA (-2)       /* CUDA runtime error */
#define FK_ENCCL (-3)       /* NCCL error */
#define FK_ENOMEM (-4)      /* device allocation failed */
#define FK_EUNSUPPORTED (-5) /* order / quadrature / variant not compiled */

/* Operator kinds (CEED bake-off problems). */
#define FK_KIND_MASS 1      /* BP1: y = G^T B^T W|J| B G x                      */
#define FK_KIND_DIFFUSION 3 /* BP3: y = G^T (B,G)^T W|J| J^-1 J^-T (B,G) G x     */

/* Kernel variants for the element contractions. */
#define FK_VARIANT_AUTO 0   /* per-order choice from the measured sweep */
#define FK_VARIANT_DFMA 1   /* register-blocked FP64 FMA, basis in the constant bank */
#define FK_VARIANT_DMMA 2   /* warp mma.sync.m8n8k4 f64 tiles (DMMA.8x8x4)           */
#define FK_VARIANT_EO 3     /* FP64 FMA with even-odd folding of the symmetric 1D tables
                               (half the multiply-adds; symmetric bases only)         */
#define FK_VARIANT_MF 4     /* matrix-free (the reference's MF strategy, operator.py:280-286):
                               even-odd FMA kernel that recomputes D = w|J|J^-1J^-T of the
                               axis-aligned box in stage C instead of reading PA data */
#define FK_VARIANT_LAST FK_VARIANT_MF

typedef struct fk_op fk_op;
typedef struct fk_comm fk_comm;

typedef struct fk_op_desc {
  int kind;           /* FK_KIND_MASS | FK_KIND_DIFFUSION */
  int p;              /* polynomial order 1..8 (d = p+1 GLL nodes per direction) */
  int q;              /* Gauss points per direction: p+1 or p+2 */
  int nx, ny;         /* elements along x, y (mesh.py:78) */
  int nz_local;       /* element layers owned by this rank (z-slab) */
  int z0_layer;       /* first global element layer owned by this rank */
  int nz_global;      /* global element layers */
  double jac_diag[3]; /* constant Jacobian diagonal h/2 (Mesh.jacobian_diag, mesh.py:56-60) */
  double jac_det;     /* Mesh.jacobian_det (mesh.py:62-64) */
  const double* B;    /* host, q*d row-major: B[a*d+i] = L_i(x_a) (Basis1D.values, tensor.py:77-119) */
  const double* G;    /* host, q*d row-major: Basis1D.gradients */
  const double* w;    /* host, q Gauss weights: Basis1D.quad_weights */
  const int64_t* gather_ids; /* optional host map (nel_local, d^3) of GLOBAL ids as
                                h1_restriction().gather_ids rows (mesh.py:144-166);
                                NULL => built on device from the closed form */
  int dirichlet;      /* 1: homogeneous essential BC on the six box faces
                         (constrained operator, diagonal one) */
  int variant;        /* FK_VARIANT_* */
  int device;         /* CUDA ordinal */
  void* stream;       /* cudaStream_t (NULL: the legacy default stream) */
  fk_comm* comm;      /* NULL for one rank; else the z-slab communicator */
  int deterministic;  /* 1: verification mode — elements in 8-colour order (colour =
                         parities of ex, ey, ez; two elements of one colour share no
                         node), one launch per colour in fixed order, so every dof sums
                         its element contributions in the same order on every run:
                         apply, diagonal and CG bitwise reproducible (the reference's
                         sequential np.add.at is likewise order-fixed, mesh.py:133-137) */
} fk_op_desc;

typedef struct fk_op_info {
  int64_t ndof_local;  /* L-vector length on this rank: npx*npy*(nz_local*p+1) */
  int64_t nel_local;   /* nx*ny*nz_local */
  int64_t dof_offset;  /* global id of local dof 0: z0_layer*p*npx*npy */
  int64_t ndof_global; /* npx*npy*npz */
  int64_t pa_bytes;    /* bytes of stored PA data D on the device */
  int variant;         /* variant actually used by fk_op_apply */
  int elems_per_block; /* launch geometry of the fused kernel */
  int threads_per_block;
  int blocks;          /* persistent grid size */
  int cfg;             /* compiled launch geometry index of that variant (fk_op_set_config) */
} fk_op_info;

int fk_version(void);
const char* fk_last_error(void);

/* Lifecycle.  fk_op_create validates the descriptor and uploads the 1D
 * tables; fk_op_setup builds the device E-restriction (int32) and the PA
 * data D (BP1: w*|J| per point; BP3: 6-component symmetric w*|J|*J^-1 J^-T). */
int fk_op_create(fk_op** out, const fk_op_desc* desc);
int fk_op_setup(fk_op* op);
int fk_op_destroy(fk_op* op);
int fk_op_get_info(const fk_op* op, fk_op_info* info);
int fk_op_set_variant(fk_op* op, int variant);
/* Select one of the compiled launch geometries of a variant (cfg = 0 is the
 * default; FK_EUNSUPPORTED when that cfg does not exist).  Tuning/testing. */
int fk_op_set_config(fk_op* op, int variant, int cfg);

/* Parity hooks: restriction rows as GLOBAL int64 ids (nel_local*d^3) and the
 * PA data (nel_local * ncomp * q^3 doubles, element-major) copied to host. */
int fk_op_restriction(fk_op* op, int64_t* host_out);
int fk_op_pa_data(fk_op* op, double* host_out);

/* y = A x on this rank's L-vector (length ndof_local); with a comm attached
 * the shared interface planes are summed across neighbouring ranks, so y is
 * the assembled P^T A_E P x restricted to this rank. */
int fk_op_apply(fk_op* op, const double* x_dev, double* y_dev);
/* Same with host buffers (pageable or pinned): H2D, apply, D2H, synchronise. */
int fk_op_apply_host(fk_op* op, const double* x_host, double* y_host);
/* Element-local apply without exchange or Dirichlet fix-up (testing). */
int fk_op_apply_local(fk_op* op, const double* x_dev, double* y_dev);

/* Assembled diagonal of A (Jacobi preconditioner); ones on essential dofs. */
int fk_op_diagonal(fk_op* op, double* diag_dev);

/* v[ess] = value on this rank's essential (Dirichlet) dofs (MFEM
 * Vector::SetSubVector(ess_tdof_list, value)); no-op without dirichlet. */
int fk_op_set_essential(fk_op* op, double* v_dev, double value);

/* Jacobi-PCG (MFEM CGSolver semantics, x0 = 0), fixed `iters` iterations
 * unless rtol > 0 stops it (r.z <= rtol^2 r0.z0).  hist_host receives
 * sqrt(r_k . z_k) for k = 0..iters_done (iters+1 doubles).  Synchronises. */
int fk_cg_solve(fk_op* op, const double* b_dev, double* x_dev, int iters, double rtol,
                double* hist_host, int* iters_done);

/* Allocate the CG workspace (5 vectors, reduction scratch, a history of
 * iters+1) so that a following fk_cg_solve with at most `iters` iterations
 * makes no device allocation — ranks sharing one GPU (loopback group) call
 * it on every rank before the collective solve. */
int fk_cg_prepare(fk_op* op, int iters);

/* Device reductions used by multi-rank CG and by tests. */
int fk_dot(fk_op* op, const double* a_dev, const double* b_dev, double* host_out);

/* Multi-GPU: one communicator per rank (z-slab decomposition).
 * Replaces the MPI group exchange of the paper's P / P^T;
 * the reference itself is single-process (P = identity).
 *
 * Two transports:
 *  FK_TRANSPORT_P2P   peer memory over NVLink / NVSwitch: each rank owns a
 *                     mailbox (halo planes + flag words); neighbours store their
 *                     partial interface planes straight into it and release a
 *                     monotone flag; CG scalars are reduced by every rank
 *                     storing its partial into every peer's slot array and
 *                     summing the slots in rank order (bitwise identical on all
 *                     ranks).  Kernel-only, so it is captured in the CG graph.
 *  FK_TRANSPORT_NCCL  grouped ncclSend/ncclRecv + ncclAllReduce.
 * nccl_unique_id points to the 128-byte ncclUniqueId produced by
 * fk_comm_unique_id on rank 0 and broadcast by the caller.
 * Ordering contract: every rank issues the same sequence of exchanges and
 * reductions on a communicator (each operator call is collective), and one
 * communicator's exchanges are issued in ONE stream order per rank (the P2P
 * mailbox counters are per communicator); operators that share a
 * communicator must not run exchanges concurrently on different streams. */
#define FK_TRANSPORT_NCCL 1
#define FK_TRANSPORT_P2P 2
#define FK_MAX_RANKS 16
#define FK_IPC_HANDLE_BYTES 64

int fk_comm_unique_id(void* out128);
int fk_comm_create(fk_comm** out, const void* nccl_unique_id, int rank, int nranks, int device);
/* P2P across processes (one per GPU): allocate this rank's mailbox for halo
 * planes of up to plane_cap doubles and return its CUDA-IPC handle
 * (FK_IPC_HANDLE_BYTES); the caller all-gathers the handles (rank order) and
 * passes them to fk_comm_connect_p2p on every rank. */
int fk_comm_create_p2p(fk_comm** out, int rank, int nranks, int device, int64_t plane_cap,
                       void* ipc_handle_out);
int fk_comm_connect_p2p(fk_comm* comm, const void* all_handles);
/* P2P inside one process: nranks communicators at once (out[0..nranks-1]),
 * rank r on devices[r] (all equal = a loopback group on one GPU; distinct
 * devices get peer access enabled).  Each rank must be driven by its own
 * host thread and stream: the exchange waits on the device for the peers. */
int fk_comm_create_loopback(fk_comm** out, int nranks, const int* devices, int64_t plane_cap);
/* transport, rank, nranks of a communicator */
int fk_comm_query(const fk_comm* comm, int* transport, int* rank, int* nranks);
int fk_comm_destroy(fk_comm* comm);

/* Benchmark hook: time `reps` applies with CUDA events on the handle's
 * stream (after the caller's warm-up); returns mean milliseconds per apply
 * of the whole apply and of the fused kernel alone. */
int fk_op_time_apply(fk_op* op, const double* x_dev, double* y_dev, int reps,
                     const void* flush_dev, size_t flush_bytes,
                     double* ms_apply, double* ms_kernel);


/* ---------------------------------------------------------------------------
 * Acoustic-gravity block operator (feklab/operator.py BlockOperator,
 * strategy FusedPA).  State [u; p]: u = 3 velocity
 * components in the discontinuous space of order_u, element blocks
 * (3, nel, (order_u+1)^3) as State.u (operator.py:63-90); p = pressure dofs
 * of the continuous H1 space of order_p (h1_restriction numbering).
 *   out_u =  cs * B_u^T D^T grad p            (_pressure_to_velocity, :288-301)
 *   out_p = -cs * G^T grad^T D B_u u          (_velocity_to_pressure, :303-319)
 * D = dmat = w|J| J^-1 (9 components per point, :137-144) is read once per
 * element for both blocks.  Compiled spaces: order_u = order_p - 1,
 * num_quad_1d = order_p + 1, order_p = 2..8 (the reference default 4/3/5).
 * Boundary terms (:400-470): absorbing lateral faces (in fk_mix_apply and
 * the RK4 driver), the free-surface lumped mass, the bottom-face load.
 * ------------------------------------------------------------------------- */
typedef struct fk_mix fk_mix;

typedef struct fk_mix_desc {
  int order_p, order_u, num_quad_1d;
  int nx, ny, nz;              /* build_mesh(nx, ny, nz, extents) */
  double jac_diag[3];          /* Mesh.jacobian_diag (mesh.py:56-60) */
  double jac_det;              /* Mesh.jacobian_det */
  const double* Bp;            /* host q x (order_p+1): pressure Basis1D.values */
  const double* Gp;            /* host q x (order_p+1): pressure Basis1D.gradients */
  const double* Bu;            /* host q x (order_u+1): velocity Basis1D.values */
  const double* w;             /* host q: quad_weights */
  const double* rho;           /* host per-element density (nel) or NULL -> rho_scalar */
  const double* bulk;          /* host per-element bulk modulus or NULL -> bulk_scalar */
  double rho_scalar, bulk_scalar;
  double coupling_scale;       /* BlockOperator coupling_scale */
  int matrix_free;             /* 1: strategy FusedMF (dmat recomputed in the kernel,
                                  operator.py:280-286); 0: FusedPA / PA */
  int device;
  void* stream;                /* cudaStream_t */
  int absorbing;               /* 1: impedance term on the lateral (x, y) faces inside apply
                                  (BlockOperator absorbing=True, _apply_absorbing :432-439) */
  double surface_gravity;      /* > 0: free-surface lumped mass on the top face (:268-276);
                                  0: none */
} fk_mix_desc;

typedef struct fk_mix_info {
  int64_t nel, ndof_p, ndof_u; /* ndof_u = 3 * nel * (order_u+1)^3 */
  int64_t pa_bytes;
  int elems_per_block, threads_per_block, blocks;
  int64_t smem_bytes;
} fk_mix_info;

int fk_mix_create(fk_mix** out, const fk_mix_desc* desc);
/* device E-restriction, dmat and the lumped mass diagonals (setup_quad_data) */
int fk_mix_setup(fk_mix* m);
int fk_mix_destroy(fk_mix* m);
int fk_mix_get_info(const fk_mix* m, fk_mix_info* info);
/* BlockOperator.apply: out_u overwritten, out_p overwritten (device pointers) */
int fk_mix_apply(fk_mix* m, const double* u, const double* p, double* out_u, double* out_p);
/* BlockOperator.apply_fused_normal: velocity -> assembled pressure -> velocity */
int fk_mix_fused_normal(fk_mix* m, const double* u, double* out_u);
/* BlockOperator.apply_mass_inverse: u = ru / lump_u, p = rp / lump_p */
int fk_mix_mass_inverse(fk_mix* m, const double* ru, const double* rp, double* u, double* p);
/* `steps` classical RK4 steps of [u,p]' = Minv(-A [u,p]) in place (rk4_step,
 * operator.py:506-531, no forcing); four fused applies per step. */
int fk_mix_rk4(fk_mix* m, double* u, double* p, double dt, int steps);
/* `steps` = 1 forced RK4 step: [u,p]' = Minv(-A [u,p] + f(t)) (rk4_step with
 * forcing, operator.py:506-531).  f0, fh, f1: device [u | p] vectors (3 nel
 * du^3 + ndof_p doubles) of the forcing at t, t + dt/2 and t + dt (NULL: 0). */
int fk_mix_rk4_forced(fk_mix* m, double* u, double* p, double dt, const double* f0,
                      const double* fh, const double* f1);
/* BlockOperator.bottom_face_load (:441-460): load = sum over bottom faces of
 * area * M2d @ vals_f, M2d = kron(m1, m1), m1 = Bp^T W Bp.  vals: device,
 * (nx*ny, (order_p+1)^2) profile values at each bottom face's nodes (first
 * in-plane index fastest, faces x-fastest); load: device ndof_p (overwritten). */
int fk_mix_bottom_load(fk_mix* m, const double* vals, double* load);

/* parity hooks: lumped diagonals (device copies) and restriction rows (host int64) */
int fk_mix_lumped(fk_mix* m, double* lump_u, double* lump_p);
int fk_mix_restriction(fk_mix* m, int64_t* host_out);
/* mean ms per apply (incl. the out_p memset) and of the fused kernel over reps */
int fk_mix_time_apply(fk_mix* m, const double* u, const double* p, double* out_u, double* out_p,
                      int reps, double* ms_apply, double* ms_kernel);

#ifdef __cplusplus
}
#endif

#endif /* FK_B200_H */
