// pa_pipe.cuh — the persistent, software-pipelined fused PA kernel skeleton.
//
// One CTA owns batches b = blockIdx.x, blockIdx.x + gridDim.x, ... of E
// elements.  While batch b is contracted, the next batch's inputs stream in
// asynchronously, so no stage waits on HBM latency:
//
//   after stage A(b):  bulk copy (TMA engine) of the next batch's int32 gather
//                      ids (+ Dirichlet bits) into the free smem slot
//   after stage C(b):  bulk copy of the next batch's PA data D (the dominant
//                      byte stream, 48 q^3 B per BP3 element) into smem, and
//                      cp.async (LDGSTS) gathers x[gid] -> X buffer
//   stage E(b):        atomic scatter-add (RED.F64) to y, fire-and-forget
//
// The contraction stages are supplied by Body (pa_dfma.cuh: FP64 FMA lines,
// pa_dmma.cuh: DMMA tiles).  References: gather/scatter feklab/mesh.py:130-137,
// contractions feklab/tensor.py:177-283, PA data feklab/operator.py:132-193.
#pragma once

#include "pa_async.cuh"
#include "pa_common.cuh"

namespace fk {

template <int D, int Q, int NC, int E, int EXTRA>
struct PipeSmem {
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  static constexpr int XS = D * D * L::LS;  // X buffer doubles per element
  // byte offsets (16-byte aligned where bulk copies land)
  static constexpr size_t OFF_BAR = 0;                                    // 3 mbarriers
  static constexpr size_t OFF_DB = 32;                                    // PA data
  static constexpr size_t OFF_GS = OFF_DB + 8ull * E * G::PS;             // 2 gid slots
  static constexpr size_t OFF_MS = OFF_GS + 4ull * 2 * E * G::GS;         // 2 bit slots
  static constexpr size_t OFF_S0 = OFF_MS + 4ull * 2 * E * G::MS;
  static constexpr size_t OFF_S1 = OFF_S0 + 8ull * E * L::P0;
  static constexpr size_t OFF_XB = OFF_S1 + 8ull * E * L::P1;
  static constexpr size_t OFF_EX = (OFF_XB + 8ull * E * XS + 15) / 16 * 16;
  static constexpr size_t BYTES = OFF_EX + 8ull * EXTRA;
};

template <int D, int Q, int NC, class Body, bool PERSIST>
__global__ void __launch_bounds__(Body::T) pa_pipe_kernel(const __grid_constant__ typename Body::Tab tb,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y,
                                                          const int* __restrict__ gids,
                                                          const double* __restrict__ pa,
                                                          const uint32_t* __restrict__ ebits,
                                                          int nel) {
  constexpr int E = Body::E, T = Body::T;
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  using S = PipeSmem<D, Q, NC, E, Body::EXTRA>;
  constexpr int D3 = L::D3, LS = L::LS, XS = S::XS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar_d = reinterpret_cast<uint64_t*>(smem_raw + S::OFF_BAR);
  uint64_t* bar_g = bar_d + 1;  // [2]
  double* db = reinterpret_cast<double*>(smem_raw + S::OFF_DB);
  int* gs = reinterpret_cast<int*>(smem_raw + S::OFF_GS);
  uint32_t* ms = reinterpret_cast<uint32_t*>(smem_raw + S::OFF_MS);
  double* s0 = reinterpret_cast<double*>(smem_raw + S::OFF_S0);
  double* s1 = reinterpret_cast<double*>(smem_raw + S::OFF_S1);
  double* xb = reinterpret_cast<double*>(smem_raw + S::OFF_XB);
  double* ex = reinterpret_cast<double*>(smem_raw + S::OFF_EX);

  const int nbatch = (nel + E - 1) / E;
  if ((int)blockIdx.x >= nbatch) return;
  const bool dirichlet = ebits != nullptr;
  if (threadIdx.x == 0) {
    mbar_init(bar_d, 1);
    mbar_init(bar_g, 1);
    mbar_init(bar_g + 1, 1);
    fence_mbar_init();
  }
  // zero the work regions once: line padding stays finite (the DMMA body reads
  // K padding and relies on zero B-operand rows to annihilate it)
  for (size_t i = threadIdx.x; i < (S::BYTES - S::OFF_S0) / 8; i += T)
    reinterpret_cast<double*>(smem_raw + S::OFF_S0)[i] = 0.0;
  __syncthreads();
  Body::init(tb, ex);
  __syncthreads();

  auto issue_g = [&](int b, int slot) {
    const int e0 = b * E, ne = min(E, nel - e0);
    const uint32_t gb = 4u * ne * G::GS, mb = dirichlet ? 4u * ne * G::MS : 0u;
    mbar_expect_tx(bar_g + slot, gb + mb);
    bulk_g2s(gs + slot * E * G::GS, gids + (size_t)e0 * G::GS, gb, bar_g + slot);
    if (dirichlet) bulk_g2s(ms + slot * E * G::MS, ebits + (size_t)e0 * G::MS, mb, bar_g + slot);
  };
  auto issue_d = [&](int b) {
    const int e0 = b * E, ne = min(E, nel - e0);
    const uint32_t bytes = 8u * ne * G::PS;
    mbar_expect_tx(bar_d, bytes);
    bulk_g2s(db, pa + (size_t)e0 * G::PS, bytes, bar_d);
  };
  auto issue_x = [&](int b, int slot) {
    const int e0 = b * E, ne = min(E, nel - e0);
    const int* g = gs + slot * E * G::GS;
    for (int t = threadIdx.x; t < E * D3; t += T) {
      const int e = t / D3, l = t - e * D3;
      double* dst = xb + e * XS + (l / D) * LS + (l % D);
      if (e < ne) cp_async8(dst, x + g[e * G::GS + l]);
      else *dst = 0.0;
    }
    cp_async_commit();
  };
  auto finish_x = [&](int slot, int ne) {
    cp_async_wait_all();
    if (dirichlet) {
      const uint32_t* m = ms + slot * E * G::MS;
      for (int t = threadIdx.x; t < ne * D3; t += T) {
        const int e = t / D3, l = t - e * D3;
        if ((m[e * G::MS + (l >> 5)] >> (l & 31)) & 1u) xb[e * XS + (l / D) * LS + (l % D)] = 0.0;
      }
    }
  };

  uint32_t ph_d = 0, ph_g0 = 0, ph_g1 = 0;
  // prologue: first batch
  if (threadIdx.x == 0) {
    issue_g(blockIdx.x, 0);
    issue_d(blockIdx.x);
  }
  mbar_wait(bar_g, ph_g0);
  ph_g0 ^= 1;
  issue_x(blockIdx.x, 0);

  auto run_batch = [&](int b, int it, bool has_next) {
    const int slot = it & 1;
    const int e0 = b * E, ne = min(E, nel - e0);
    const int nb = b + gridDim.x;
    finish_x(slot, ne);
    __syncthreads();

    Body::stage_a(tb, it, xb, s1, ne, ex);
    __syncthreads();
    if (has_next && threadIdx.x == 0) {
      fence_proxy_async();
      issue_g(nb, slot ^ 1);
    }
    Body::stage_b(tb, it, s1, s0, ne, ex);
    __syncthreads();
    mbar_wait(bar_d, ph_d);
    ph_d ^= 1;
    Body::stage_c(tb, it, s0, db, s1, ne, ex);
    __syncthreads();
    if (has_next) {
      if (threadIdx.x == 0) {
        fence_proxy_async();
        issue_d(nb);
      }
      if (slot == 0) {
        mbar_wait(bar_g + 1, ph_g1);
        ph_g1 ^= 1;
      } else {
        mbar_wait(bar_g, ph_g0);
        ph_g0 ^= 1;
      }
      issue_x(nb, slot ^ 1);
    }
    Body::stage_d(tb, it, s1, s0, ne, ex);
    __syncthreads();
    Body::stage_e(tb, it, s0, gs + slot * E * G::GS, y, ne, ex);
    __syncthreads();
  };

  if constexpr (PERSIST) {
    int it = 0;
    for (int b = blockIdx.x; b < nbatch; b += gridDim.x, ++it)
      run_batch(b, it, b + (int)gridDim.x < nbatch);
  } else {
    // one batch per CTA: no loop, so the compiler has nothing to hoist the
    // basis-table loads out of (co-resident CTAs overlap load and compute)
    run_batch(blockIdx.x, 0, false);
  }
}

}  // namespace fk
