// fk_comm.cu — NCCL communicator and the z-slab interface exchange.
//
// The reference is single-process (P = identity); the paper's
// P / P^T is MPI.  Here the box mesh is cut into
// contiguous z-slabs of element layers.  Because global numbering is
// z-slowest (mesh.py:164), each rank's L-vector is one contiguous slice and
// neighbours share exactly one npx*npy plane.  After the element-local apply
// each rank holds a partial sum on its two interface planes; a grouped
// ncclSend/ncclRecv swaps them and an add kernel completes P^T.  IEEE
// addition is commutative, so both copies of a shared plane are bit-identical.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") — the copy torch
// already loaded into the process, or FK_NCCL_LIBRARY — so the single-GPU
// library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fk_comm.h"
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

__global__ void add_plane_kernel(double* __restrict__ y, const double* __restrict__ h, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] += h[i];
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

int comm_setup(fk_op* op) {
  if (op->comm->nranks > 1 && op->halo == nullptr) {
    if (cudaMalloc(&op->halo, sizeof(double) * 2 * op->npx * op->npy) != cudaSuccess)
      return fk_set_error(FK_ENOMEM, "halo buffers");
    if (cudaStreamCreateWithFlags(&op->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&op->ev_bnd, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&op->ev_xchg, cudaEventDisableTiming) != cudaSuccess)
      return fk_set_error(FK_ECUDA, "comm stream/events");
  }
  return FK_OK;
}

int exchange_post(fk_op* op, double* y, cudaStream_t s) {
  fk_comm* c = op->comm;
  if (c == nullptr || c->nranks <= 1) return FK_OK;
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

int exchange_finish(fk_op* op, double* y, cudaStream_t s) {
  fk_comm* c = op->comm;
  if (c == nullptr || c->nranks <= 1) return FK_OK;
  const int64_t P = op->npx * op->npy;
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((P + threads - 1) / threads, 4 * op->num_sms);
  if (c->rank > 0) add_plane_kernel<<<blocks, threads, 0, s>>>(y, op->halo, P);
  if (c->rank < c->nranks - 1) add_plane_kernel<<<blocks, threads, 0, s>>>(y + op->ndof - P, op->halo + P, P);
  if (cudaGetLastError() != cudaSuccess) return fk_set_error(FK_ECUDA, "add_plane_kernel launch");
  return FK_OK;
}

int exchange_interface(fk_op* op, double* y, cudaStream_t s) {
  fk_comm* c = op->comm;
  if (c == nullptr || c->nranks <= 1) return FK_OK;
  NcclApi& api = nccl();
  ncclComm_t comm = static_cast<ncclComm_t>(c->nccl);
  const int64_t P = op->npx * op->npy;
  double* below = op->halo;
  double* above = op->halo + P;
  NCCL_TRY(api.GroupStart());
  if (c->rank > 0) {
    NCCL_TRY(api.Send(y, P, ncclDouble, c->rank - 1, comm, s));
    NCCL_TRY(api.Recv(below, P, ncclDouble, c->rank - 1, comm, s));
  }
  if (c->rank < c->nranks - 1) {
    NCCL_TRY(api.Send(y + op->ndof - P, P, ncclDouble, c->rank + 1, comm, s));
    NCCL_TRY(api.Recv(above, P, ncclDouble, c->rank + 1, comm, s));
  }
  NCCL_TRY(api.GroupEnd());
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((P + threads - 1) / threads, 4 * op->num_sms);
  if (c->rank > 0) add_plane_kernel<<<blocks, threads, 0, s>>>(y, below, P);
  if (c->rank < c->nranks - 1) add_plane_kernel<<<blocks, threads, 0, s>>>(y + op->ndof - P, above, P);
  if (cudaGetLastError() != cudaSuccess) return fk_set_error(FK_ECUDA, "add_plane_kernel launch");
  return FK_OK;
}

int allreduce_scalar(fk_op* op, double* v, cudaStream_t s) {
  fk_comm* c = op->comm;
  if (c == nullptr || c->nranks <= 1) return FK_OK;
  NCCL_TRY(nccl().AllReduce(v, v, 1, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->nccl), s));
  return FK_OK;
}

}  // namespace fk

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
  c->nccl = comm;
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  *out = c;
  return FK_OK;
}

int fk_comm_destroy(fk_comm* c) {
  if (c == nullptr) return FK_OK;
  if (c->nccl && nccl().loaded) nccl().CommDestroy(static_cast<ncclComm_t>(c->nccl));
  delete c;
  return FK_OK;
}

}  // extern "C"
