// fk_comm.cu — z-slab communicators and the interface exchange.
//
// The reference is single-process (P = identity); the paper's
// P / P^T is MPI.  Here the box mesh is cut into
// contiguous z-slabs of element layers.  Because global numbering is
// z-slowest (mesh.py:164), each rank's L-vector is one contiguous slice and
// neighbours share exactly one npx*npy plane.  After the element-local apply
// each rank holds a partial sum on its two interface planes; the exchange
// swaps them and adds the neighbour's partial.  IEEE addition is commutative,
// so both copies of a shared plane are bit-identical.
//
// Two transports (include/fk.h):
//
// * P2P (default; NVLink / NVSwitch peer memory).  Every rank owns a Mailbox
//   (fk_internal.h): two halo planes, flag words and reduction slots.  One
//   exchange k = seq_x + 1 on rank r is four stream-ordered kernels:
//     credit  (1 CTA)   wait until each neighbour consumed plane k-1
//     put     (grid)    store my partial bottom/top plane into the
//                       neighbours' halo buffers (remote stores), the last CTA
//                       releases their recv flags = k
//     ...the interior element layers run here (apply_overlapped)...
//     arrive  (1 CTA)   wait until my recv flags reach k
//     add     (grid)    y_plane += halo, the last CTA releases the
//                       neighbours' consumed flags = k and sets seq_x = k
//   A scalar allreduce (CG dots) is one 1-CTA kernel: thread j stores my
//   partial into rank j's slot [k&1][r] and releases its flag; then waits for
//   every rank's flag and sums the slots in rank order — the same bits on all
//   ranks.  Only the 1-CTA kernels spin, so ranks sharing one GPU (the
//   loopback group the tests use) cannot starve each other of SMs.  All state
//   is device-side counters: the sequence replays inside the CG CUDA graph.
//   Mailboxes are mapped across processes with CUDA IPC
//   (fk_comm_create_p2p / fk_comm_connect_p2p) or shared directly inside one
//   process (fk_comm_create_loopback).
//
// * NCCL.  Grouped ncclSend/ncclRecv of the planes on a high-priority comm
//   stream (so its CTAs are dispatched ahead of the persistent interior
//   kernel) and an in-place ncclAllReduce of one double.  NCCL is resolved at
//   run time with dlopen("libnccl.so.2") — the copy torch loaded, or
//   FK_NCCL_LIBRARY — so the library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fk_comm.h"
#include "fk_error.h"
#include "fk_internal.h"

namespace {

struct NcclApi {
  bool loaded = false;
  std::string error;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = nullptr;
  const char* env = std::getenv("FK_NCCL_LIBRARY");
  if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.error = std::string("cannot load NCCL: ") + dlerror();
    return api;
  }
#define FK_SYM(name)                                                              \
  api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name));        \
  if (!api.name) {                                                                \
    api.error = "NCCL symbol nccl" #name " missing";                              \
    return api;                                                                   \
  }
  FK_SYM(GetUniqueId)
  FK_SYM(CommInitRank)
  FK_SYM(CommDestroy)
  FK_SYM(Send)
  FK_SYM(Recv)
  FK_SYM(GroupStart)
  FK_SYM(GroupEnd)
  FK_SYM(AllReduce)
  FK_SYM(GetErrorString)
#undef FK_SYM
  api.loaded = true;
  return api;
}

using fk::Mailbox;
using fk::PeerTable;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double* halo_of(Mailbox* b, int side, int64_t cap) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(b) + fk::kMailboxHeader) + side * cap;
}

// Spin (one thread per awaited flag) until box->flags[side] >= box->seq_x + 1
// (recv) or >= box->seq_x (credit: the neighbour consumed the previous plane).
// One CTA: the only spinning kernels are these and p2p_allreduce_kernel.
__global__ void p2p_wait_kernel(Mailbox* box, int recv, int below, int above) {
  const int t = threadIdx.x;
  if ((t == 0 && below) || (t == 1 && above)) {
    const unsigned long long want = box->seq_x + (recv ? 1ull : 0ull);
    const unsigned long long* f = recv ? &box->recv_flag[t] : &box->consumed[t];
    while (ld_acquire_sys(f) < want) __nanosleep(64);
  }
}

// Store my partial interface planes into the neighbours' halo buffers.
// below: my plane 0 -> rank-1's halo[1] (it receives "from above");
// above: my last plane -> rank+1's halo[0].
__global__ void __launch_bounds__(256) p2p_put_kernel(const double* __restrict__ y, int64_t ndof,
                                                      int64_t P, Mailbox* box, Mailbox* lo,
                                                      Mailbox* hi, int64_t cap) {
  double* dlo = lo ? halo_of(lo, 1, cap) : nullptr;
  double* dhi = hi ? halo_of(hi, 0, cap) : nullptr;
  const double* ytop = y + ndof - P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (dlo) dlo[i] = y[i];
    if (dhi) dhi[i] = ytop[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(&box->put_done, 1u) == gridDim.x - 1) {
      box->put_done = 0u;
      const unsigned long long k = box->seq_x + 1ull;
      __threadfence_system();
      if (lo) st_release_sys(&lo->recv_flag[1], k);
      if (hi) st_release_sys(&hi->recv_flag[0], k);
    }
  }
}

// y_plane += received neighbour partial; the last CTA returns the credits and
// completes exchange k.
__global__ void __launch_bounds__(256) p2p_add_kernel(double* __restrict__ y, int64_t ndof,
                                                      int64_t P, Mailbox* box, Mailbox* lo,
                                                      Mailbox* hi, int64_t cap) {
  const double* hlo = lo ? halo_of(box, 0, cap) : nullptr;
  const double* hhi = hi ? halo_of(box, 1, cap) : nullptr;
  double* ytop = y + ndof - P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (hlo) y[i] += __ldcv(hlo + i);
    if (hhi) ytop[i] += __ldcv(hhi + i);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(&box->add_done, 1u) == gridDim.x - 1) {
      box->add_done = 0u;
      const unsigned long long k = box->seq_x + 1ull;
      __threadfence_system();
      if (lo) st_release_sys(&lo->consumed[1], k);
      if (hi) st_release_sys(&hi->consumed[0], k);
      box->seq_x = k;
    }
  }
}

// *v = sum over ranks (rank order) of every rank's *v.
__global__ void p2p_allreduce_kernel(double* v, PeerTable peers, int rank, int nranks) {
  Mailbox* box = peers.box[rank];
  const int t = threadIdx.x;
  const unsigned long long k = box->seq_r + 1ull;
  const int par = (int)(k & 1ull);
  if (t < nranks) {
    Mailbox* dst = peers.box[t];
    dst->red_slot[par][rank] = *v;
    __threadfence_system();
    st_release_sys(&dst->red_flag[rank], k);
    while (ld_acquire_sys(&box->red_flag[t]) < k) __nanosleep(32);
  }
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
    for (int j = 0; j < nranks; ++j) s += __ldcv(&box->red_slot[par][j]);
    *v = s;
    box->seq_r = k;
  }
}

__global__ void add_plane_kernel(double* __restrict__ y, const double* __restrict__ h, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] += h[i];
}

int put_blocks(const fk_op* op, int64_t P) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((P + 255) / 256, 2 * (int64_t)op->num_sms));
}

}  // namespace

int fk_set_error(int code, const char* msg);  // fk_api.cu

#define NCCL_TRY(call)                                                                     \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess) return fk_set_error(FK_ENCCL, nccl().GetErrorString(r_));       \
  } while (0)

namespace fk {

int64_t owned_begin(const fk_op* op) {
  if (op->comm == nullptr || op->comm->rank == 0) return 0;
  return op->npx * op->npy;
}

bool multi_rank(const fk_op* op) { return op->comm != nullptr && op->comm->nranks > 1; }
bool p2p(const fk_op* op) { return multi_rank(op) && op->comm->transport == FK_TRANSPORT_P2P; }

int preload_comm_kernels() {
  const void* ks[] = {reinterpret_cast<const void*>(&p2p_wait_kernel),
                      reinterpret_cast<const void*>(&p2p_put_kernel),
                      reinterpret_cast<const void*>(&p2p_add_kernel),
                      reinterpret_cast<const void*>(&p2p_allreduce_kernel),
                      reinterpret_cast<const void*>(&add_plane_kernel)};
  for (const void* k : ks) {
    cudaFuncAttributes a;
    FK_CUDA(cudaFuncGetAttributes(&a, k));
  }
  return FK_OK;
}

int comm_setup(fk_op* op) {
  if (!multi_rank(op)) return FK_OK;
  const int64_t P = op->npx * op->npy;
  if (op->comm->transport == FK_TRANSPORT_P2P) {
    if (P > op->comm->plane_cap)
      return fk_fail(FK_EINVAL, "interface plane of %lld dofs does not match the communicator's "
                                "capacity (%lld)", (long long)P, (long long)op->comm->plane_cap);
    return FK_OK;
  }
  if (op->halo == nullptr) {
    if (cudaMalloc(&op->halo, sizeof(double) * 2 * P) != cudaSuccess)
      return fk_set_error(FK_ENOMEM, "halo buffers");
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&op->comm_stream, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&op->ev_bnd, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&op->ev_xchg, cudaEventDisableTiming) != cudaSuccess)
      return fk_set_error(FK_ECUDA, "comm stream/events");
  }
  return FK_OK;
}

// ---- P2P pieces (all on stream s) --------------------------------------------

static int p2p_post(fk_op* op, const double* y, cudaStream_t s) {
  fk_comm* c = op->comm;
  const int64_t P = op->npx * op->npy;
  Mailbox* lo = c->rank > 0 ? c->peers.box[c->rank - 1] : nullptr;
  Mailbox* hi = c->rank < c->nranks - 1 ? c->peers.box[c->rank + 1] : nullptr;
  p2p_wait_kernel<<<1, 32, 0, s>>>(c->box, 0, lo != nullptr, hi != nullptr);
  p2p_put_kernel<<<put_blocks(op, P), 256, 0, s>>>(y, op->ndof, P, c->box, lo, hi, c->plane_cap);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}

static int p2p_finish(fk_op* op, double* y, cudaStream_t s) {
  fk_comm* c = op->comm;
  const int64_t P = op->npx * op->npy;
  Mailbox* lo = c->rank > 0 ? c->peers.box[c->rank - 1] : nullptr;
  Mailbox* hi = c->rank < c->nranks - 1 ? c->peers.box[c->rank + 1] : nullptr;
  p2p_wait_kernel<<<1, 32, 0, s>>>(c->box, 1, lo != nullptr, hi != nullptr);
  p2p_add_kernel<<<put_blocks(op, P), 256, 0, s>>>(y, op->ndof, P, c->box, lo, hi, c->plane_cap);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}

// ---- NCCL pieces -----------------------------------------------------------------

static int nccl_sendrecv(fk_op* op, const double* y, cudaStream_t s) {
  fk_comm* c = op->comm;
  NcclApi& api = nccl();
  ncclComm_t comm = static_cast<ncclComm_t>(c->nccl);
  const int64_t P = op->npx * op->npy;
  NCCL_TRY(api.GroupStart());
  if (c->rank > 0) {
    NCCL_TRY(api.Send(y, P, ncclDouble, c->rank - 1, comm, s));
    NCCL_TRY(api.Recv(op->halo, P, ncclDouble, c->rank - 1, comm, s));
  }
  if (c->rank < c->nranks - 1) {
    NCCL_TRY(api.Send(y + op->ndof - P, P, ncclDouble, c->rank + 1, comm, s));
    NCCL_TRY(api.Recv(op->halo + P, P, ncclDouble, c->rank + 1, comm, s));
  }
  NCCL_TRY(api.GroupEnd());
  return FK_OK;
}

static int nccl_add(fk_op* op, double* y, cudaStream_t s) {
  fk_comm* c = op->comm;
  const int64_t P = op->npx * op->npy;
  const int blocks = put_blocks(op, P);
  if (c->rank > 0) add_plane_kernel<<<blocks, 256, 0, s>>>(y, op->halo, P);
  if (c->rank < c->nranks - 1) add_plane_kernel<<<blocks, 256, 0, s>>>(y + op->ndof - P, op->halo + P, P);
  FK_CUDA(cudaGetLastError());
  return FK_OK;
}

// ---- transport-independent entry points ----------------------------------------

int exchange_post(fk_op* op, double* y, cudaStream_t s) {
  if (!multi_rank(op)) return FK_OK;
  return p2p(op) ? p2p_post(op, y, s) : nccl_sendrecv(op, y, s);
}

int exchange_finish(fk_op* op, double* y, cudaStream_t s) {
  if (!multi_rank(op)) return FK_OK;
  return p2p(op) ? p2p_finish(op, y, s) : nccl_add(op, y, s);
}

int exchange_interface(fk_op* op, double* y, cudaStream_t s) {
  if (!multi_rank(op)) return FK_OK;
  FK_TRY(exchange_post(op, y, s));
  return exchange_finish(op, y, s);
}

int allreduce_scalar(fk_op* op, double* v, cudaStream_t s) {
  if (!multi_rank(op)) return FK_OK;
  fk_comm* c = op->comm;
  if (c->transport == FK_TRANSPORT_P2P) {
    p2p_allreduce_kernel<<<1, 32, 0, s>>>(v, c->peers, c->rank, c->nranks);
    FK_CUDA(cudaGetLastError());
    return FK_OK;
  }
  NCCL_TRY(nccl().AllReduce(v, v, 1, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->nccl), s));
  return FK_OK;
}

}  // namespace fk

namespace {

int alloc_mailbox(fk_comm* c, int64_t plane_cap) {
  FkDeviceGuard g(c->device);
  const size_t bytes = fk::kMailboxHeader + sizeof(double) * 2 * (size_t)std::max<int64_t>(plane_cap, 1);
  void* p = nullptr;
  FK_CUDA(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(p);
    return fk_fail(FK_ECUDA, "mailbox init: %s", cudaGetErrorString(e));
  }
  c->box = static_cast<Mailbox*>(p);
  c->plane_cap = plane_cap;
  c->peers.box[c->rank] = c->box;
  return FK_OK;
}

}  // namespace

extern "C" {

int fk_comm_unique_id(void* out128) {
  if (out128 == nullptr) return fk_set_error(FK_EINVAL, "null argument");
  NcclApi& api = nccl();
  if (!api.loaded) return fk_set_error(FK_ENCCL, api.error.c_str());
  ncclUniqueId id;
  NCCL_TRY(api.GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return FK_OK;
}

int fk_comm_create(fk_comm** out, const void* uid, int rank, int nranks, int device) {
  if (out == nullptr || uid == nullptr) return fk_set_error(FK_EINVAL, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fk_set_error(FK_EINVAL, "bad rank/nranks");
  NcclApi& api = nccl();
  if (!api.loaded) return fk_set_error(FK_ENCCL, api.error.c_str());
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t comm = nullptr;
  ncclResult_t r = api.CommInitRank(&comm, nranks, id, rank);
  cudaSetDevice(prev);
  if (r != ncclSuccess) return fk_set_error(FK_ENCCL, api.GetErrorString(r));
  fk_comm* c = new fk_comm();
  c->transport = FK_TRANSPORT_NCCL;
  c->nccl = comm;
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  *out = c;
  return FK_OK;
}

int fk_comm_create_p2p(fk_comm** out, int rank, int nranks, int device, int64_t plane_cap,
                       void* handle_out) {
  if (out == nullptr || handle_out == nullptr) return fk_set_error(FK_EINVAL, "null argument");
  *out = nullptr;
  if (nranks < 1 || nranks > fk::kMaxRanks || rank < 0 || rank >= nranks)
    return fk_fail(FK_EINVAL, "bad rank %d / nranks %d (1..%d ranks)", rank, nranks, fk::kMaxRanks);
  if (plane_cap < 1) return fk_set_error(FK_EINVAL, "plane capacity must be positive");
  fk_comm* c = new fk_comm();
  c->transport = FK_TRANSPORT_P2P;
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  int rc = alloc_mailbox(c, plane_cap);
  if (rc != FK_OK) {
    delete c;
    return rc;
  }
  FkDeviceGuard g(device);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, c->box);
  if (e != cudaSuccess) {
    cudaFree(c->box);
    delete c;
    return fk_fail(FK_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == FK_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  *out = c;
  return FK_OK;
}

int fk_comm_connect_p2p(fk_comm* c, const void* handles) {
  if (c == nullptr || handles == nullptr) return fk_set_error(FK_EINVAL, "null argument");
  if (c->transport != FK_TRANSPORT_P2P) return fk_set_error(FK_EINVAL, "not a P2P communicator");
  FkDeviceGuard g(c->device);
  const char* hb = static_cast<const char*>(handles);
  for (int j = 0; j < c->nranks; ++j) {
    if (j == c->rank || c->ipc_mapped[j]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + (size_t)j * FK_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fk_fail(FK_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", j, cudaGetErrorString(e));
    c->peers.box[j] = static_cast<Mailbox*>(p);
    c->ipc_mapped[j] = true;
  }
  return FK_OK;
}

int fk_comm_create_loopback(fk_comm** out, int nranks, const int* devices, int64_t plane_cap) {
  if (out == nullptr || devices == nullptr) return fk_set_error(FK_EINVAL, "null argument");
  if (nranks < 1 || nranks > fk::kMaxRanks)
    return fk_fail(FK_EINVAL, "nranks %d outside 1..%d", nranks, fk::kMaxRanks);
  if (plane_cap < 1) return fk_set_error(FK_EINVAL, "plane capacity must be positive");
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  // distinct devices in one process address each other through UVA once peer
  // access is on (NVLink); ranks on one device need nothing
  for (int a = 0; a < nranks; ++a)
    for (int b = 0; b < nranks; ++b) {
      if (devices[a] == devices[b]) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]);
      if (!ok) return fk_fail(FK_EUNSUPPORTED, "device %d cannot access device %d", devices[a], devices[b]);
      FkDeviceGuard g(devices[a]);
      cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fk_fail(FK_ECUDA, "peer access %d->%d: %s", devices[a], devices[b], cudaGetErrorString(e));
      cudaGetLastError();
    }
  fk_comm* made[fk::kMaxRanks] = {};
  for (int r = 0; r < nranks; ++r) {
    made[r] = new fk_comm();
    made[r]->transport = FK_TRANSPORT_P2P;
    made[r]->rank = r;
    made[r]->nranks = nranks;
    made[r]->device = devices[r];
    int rc = alloc_mailbox(made[r], plane_cap);
    if (rc != FK_OK) {
      for (int j = 0; j <= r; ++j) {
        if (made[j]->box) cudaFree(made[j]->box);
        delete made[j];
      }
      return rc;
    }
  }
  for (int r = 0; r < nranks; ++r) {
    for (int j = 0; j < nranks; ++j) made[r]->peers.box[j] = made[j]->box;
    out[r] = made[r];
  }
  return FK_OK;
}

int fk_comm_query(const fk_comm* c, int* transport, int* rank, int* nranks) {
  if (c == nullptr) return fk_set_error(FK_EINVAL, "null communicator");
  if (transport) *transport = c->transport;
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->nranks;
  return FK_OK;
}

// Testing hook (not in include/fk.h's stable surface): the mailbox control
// words {recv[2], consumed[2], seq_x, seq_r, put_done, add_done}, read on a
// private non-blocking stream so it works while exchange kernels wait.
int fk_comm_debug_state(const fk_comm* c, unsigned long long* out8) {
  if (c == nullptr || out8 == nullptr || c->box == nullptr) return fk_set_error(FK_EINVAL, "null argument");
  FkDeviceGuard g(c->device);
  cudaStream_t s;
  FK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  Mailbox h;
  cudaError_t e = cudaMemcpyAsync(&h, c->box, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return fk_fail(FK_ECUDA, "mailbox read: %s", cudaGetErrorString(e));
  out8[0] = h.recv_flag[0];
  out8[1] = h.recv_flag[1];
  out8[2] = h.consumed[0];
  out8[3] = h.consumed[1];
  out8[4] = h.seq_x;
  out8[5] = h.seq_r;
  out8[6] = h.put_done;
  out8[7] = h.add_done;
  return FK_OK;
}

int fk_comm_destroy(fk_comm* c) {
  if (c == nullptr) return FK_OK;
  if (c->nccl && nccl().loaded) nccl().CommDestroy(static_cast<ncclComm_t>(c->nccl));
  if (c->transport == FK_TRANSPORT_P2P) {
    FkDeviceGuard g(c->device);
    for (int j = 0; j < fk::kMaxRanks; ++j)
      if (c->ipc_mapped[j] && c->peers.box[j]) cudaIpcCloseMemHandle(c->peers.box[j]);
    if (c->box) cudaFree(c->box);
  }
  delete c;
  return FK_OK;
}

}  // extern "C"
