// fk_comm.h — z-slab multi-GPU plumbing (peer memory or NCCL over NVLink / NVSwitch).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

struct fk_op;

namespace fk {

// First locally OWNED dof: the bottom interface plane of rank r > 0 belongs
// to rank r-1 (the lower rank owns shared planes), so dot products run over
// [owned_begin, ndof_local) and every global dof is counted exactly once.
int64_t owned_begin(const fk_op* op);

bool multi_rank(const fk_op* op);  // a communicator with more than one rank
bool p2p(const fk_op* op);         // ... on the peer-memory transport
int comm_setup(fk_op* op);
// Force-load the exchange / reduction kernels (see preload_kernels, fk_api.cu).
int preload_comm_kernels();
// y_plane += neighbour's partial sum of the same plane, for both interfaces.
int exchange_interface(fk_op* op, double* y, cudaStream_t s);
// Split form for overlap: post both interface planes on stream s (after the
// boundary-layer elements: P2P stores into the neighbours' mailboxes, or the
// grouped NCCL send/recv), then add the received partial sums on stream s2
// (after the interior elements; P2P waits for the neighbours' flags first).
int exchange_post(fk_op* op, double* y, cudaStream_t s);
int exchange_finish(fk_op* op, double* y, cudaStream_t s2);
int allreduce_scalar(fk_op* op, double* dev_scalar, cudaStream_t s);

}  // namespace fk
