// pa_pipe.cuh — the persistent, software-pipelined fused PA kernel skeleton.
//
// One CTA owns batches b = blockIdx.x, blockIdx.x + gridDim.x, ... of E
// elements.  While batch b is contracted, the inputs of the next batches
// stream in asynchronously, so no stage waits on HBM latency:
//
//   top of batch b:    x gather of batch b+1 (cp.async / LDGSTS, 8-byte
//                      elements x[gid]) into the other X buffer — a whole
//                      batch of compute hides its latency;
//                      bulk copy (TMA engine, cp.async.bulk) of the int32
//                      gather ids (+ Dirichlet bits) of batch b+2 into the
//                      third gid slot
//   after stage C(b):  bulk copy of batch b+1's PA data D (the dominant
//                      byte stream, 48 q^3 B per BP3 element) into smem
//   stage E(b):        atomic scatter-add (RED.F64) to y, fire-and-forget
//
// The contraction stages are supplied by Body (pa_dfma.cuh: FP64 FMA lines,
// pa_dmma.cuh: DMMA tiles).  References: gather/scatter feklab/mesh.py:130-137,
// contractions feklab/tensor.py:177-283, PA data feklab/operator.py:132-193.
#pragma once

#include <type_traits>

#include "pa_async.cuh"
#include "pa_common.cuh"

namespace fk {

// X buffer addressing: bodies with their own layout (XLAY, pa_dfma_eo.cuh)
// provide xoff(e, l) / gather_map(t, e, l); the others use the line layout
// X[e][j + D k][i] with pitch LS and an element-major gather.
template <class B, class = void>
struct HasXLay : std::false_type {};
template <class B>
struct HasXLay<B, std::void_t<decltype(B::XLAY)>> : std::true_type {};

template <int D, int Q, int NC, class Body, bool XL = HasXLay<Body>::value>
struct XAddr {
  using L = LineLayout<D, Q, NC>;
  static constexpr int XS = D * D * L::LS;
  __device__ __forceinline__ static int off(int e, int l) { return e * XS + (l / D) * L::LS + (l % D); }
  __device__ __forceinline__ static void map(int t, int& e, int& l) {
    e = t / L::D3;
    l = t - e * L::D3;
  }
};
template <int D, int Q, int NC, class Body>
struct XAddr<D, Q, NC, Body, true> {
  static constexpr int XS = Body::XS;
  __device__ __forceinline__ static int off(int e, int l) { return Body::xoff(e, l); }
  __device__ __forceinline__ static void map(int t, int& e, int& l) { Body::gather_map(t, e, l); }
};

// Closed-form element restriction of the structured box (h1_restriction,
// mesh.py:157-164) for the GM = 1 kernels: the id of node (i, j, k) of local
// element e is base(e) + i + npx (j + npy k), base(e) = ex p + npx (ey p +
// npy ez p).  e0 = first element of this launch within the rank's slab.
// mnx/snx, mny/sny: division by nx and ny as (umulhi(n, m) + n) >> s
// (round-up multiplier, exact for n < 2^31; host side struct_ids, pa_inst.cu).
struct StructIds {
  int nx, ny, p, npx, npy;
  long long e0;
  unsigned mnx, mny;
  int snx, sny;
  double* qf;  // non-null: CTA b writes its share of sum_e x_e^T A_e x_e to qf[b]
};

// register PA data of a DR launch (pa_dfma_eo.cuh DfmaEoBody::DRegs)
template <class B, bool DR>
struct DRegsOf {
  struct type {};
};
template <class B>
struct DRegsOf<B, true> {
  using type = typename B::DRegs;
};

// bodies that run stages B, C and D as one register-resident stage
// (pa_eo_bcd.cuh FUSED_BCD): A, stage_bcd, E — three CTA barriers per batch
template <class B, class = void>
struct HasBcd {
  static constexpr bool value = false;
};
template <class B>
struct HasBcd<B, decltype((void)B::FUSED_BCD)> {
  static constexpr bool value = B::FUSED_BCD;
};

// bodies that stream the PA data through a two-slot ring of c-plane pairs
// (pa_eo_ds.cuh D_STREAM)
template <class B, class = void>
struct HasDs {
  static constexpr bool value = false;
};
template <class B>
struct HasDs<B, decltype((void)B::D_STREAM)> {
  static constexpr bool value = B::D_STREAM;
};
// shared-memory bytes of the PA data region: the batch's D (bulk copy), none
// (D from global / matrix-free), or two ring barriers + two pair slots
template <class B, bool NOD, bool DS = HasDs<B>::value>
struct DRegion {
  static constexpr size_t bytes(size_t batch) { return NOD ? 0ull : batch; }
};
template <class B, bool NOD>
struct DRegion<B, NOD, true> {
  static constexpr size_t bytes(size_t) { return 16ull + 16ull * B::SLOT; }
};

// bodies whose stage C can accumulate the element quadratic form (QF_OK)
template <class B, class = void>
struct HasQf {
  static constexpr bool value = false;
};
template <class B>
struct HasQf<B, decltype((void)B::QF_OK)> {
#ifdef FK_NO_QF
  static constexpr bool value = false;  // A/B builds without the quadratic form
#else
  static constexpr bool value = B::QF_OK;
#endif
};

__device__ __forceinline__ int fast_div(int n, unsigned m, int s) {
  return (int)((__umulhi((unsigned)n, m) + (unsigned)n) >> s);
}

template <int D, int Q, int NC, class Body, bool DG = false, int GM = 0, bool SX = false>
struct PipeSmem {
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  static constexpr int E = Body::E, EXTRA = Body::EXTRA;
  static constexpr int XS = XAddr<D, Q, NC, Body>::XS;  // X buffer doubles per element
  static constexpr int NG = 3;              // gather-id slots (batches b, b+1, b+2)
  static constexpr int GSS = GM == 1 ? 1 : G::GS;  // ints per element in a slot (GM 1: base id)
  static constexpr int NX = SX ? 1 : 2;             // X buffers
  // byte offsets (16-byte aligned where bulk copies land)
  static constexpr size_t OFF_BAR = 0;                                 // 4 mbarriers
  static constexpr size_t OFF_DB = 32;                                 // PA data
  static constexpr size_t OFF_GS = OFF_DB + DRegion<Body, DG>::bytes(8ull * E * G::PS);  // NG gid slots
  static constexpr size_t OFF_MS = OFF_GS + (4ull * NG * E * GSS + 15) / 16 * 16;  // NG bit slots
  static constexpr size_t OFF_S0 = OFF_MS + 4ull * NG * E * G::MS;
  static constexpr size_t OFF_S1 = OFF_S0 + 8ull * E * Body::P0;
  static constexpr size_t OFF_XB = OFF_S1 + 8ull * E * Body::P1;      // 2 X buffers
  static constexpr size_t OFF_EX = (OFF_XB + 8ull * NX * E * XS + 15) / 16 * 16;
  static constexpr size_t BYTES = OFF_EX + 8ull * EXTRA;
};

// DG (high orders, where E*48q^3 bytes of smem would cap occupancy): stage C
// reads D straight from global memory; the next batch's D range is pulled
// toward L2 with cp.async.bulk.prefetch.L2 instead of copied into smem.
// MF (matrix-free, even-odd bodies only): no PA data at all — stage C
// recomputes D from the 1D weights and the element Jacobian (Body::stage_c<true>).
// GM = 1 (even-odd bodies): gather ids from the closed form (StructIds) —
// no id array traffic, one int per element per slot.  SX: a single X buffer;
// the next batch's gather is issued after stage A has consumed the current one.
// XP: precomputed per-thread gather slots.  QF: the element quadratic form
// twin (CG).  YS: staged scatter — stage E's outputs through the dead W
// region, RED.F64s in node order.  DR (BP1, with DG): stage C's PA data loaded
// into registers at the start of the batch.  Body traits FUSED_BCD
// (pa_eo_bcd.cuh) and D_STREAM (pa_eo_ds.cuh) select the fused B-C-D stage
// and the c-plane-pair ring of PA data.
template <int D, int Q, int NC, class Body, bool PERSIST, bool DG = false, bool MF = false, int GM = 0,
          bool SX = false, bool XP = false, bool QF = false, bool YS = false, bool DR = false>
__global__ void __launch_bounds__(Body::T) pa_pipe_kernel(const __grid_constant__ typename Body::Tab tb,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y,
                                                          const int* __restrict__ gids,
                                                          const double* __restrict__ pa,
                                                          const uint32_t* __restrict__ ebits,
                                                          int nel, const StructIds sid) {
  constexpr int E = Body::E, T = Body::T;
  using L = LineLayout<D, Q, NC>;
  using G = GlobalLayout<D, Q, NC>;
  using S = PipeSmem<D, Q, NC, Body, DG || MF, GM, SX>;
  constexpr int GSS = S::GSS;
  using XA = XAddr<D, Q, NC, Body>;
  constexpr int D3 = L::D3, XS = S::XS, NG = S::NG;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar_d = reinterpret_cast<uint64_t*>(smem_raw + S::OFF_BAR);
  uint64_t* bar_g = bar_d + 1;  // [NG]
  double* db = reinterpret_cast<double*>(smem_raw + S::OFF_DB);
  int* gs = reinterpret_cast<int*>(smem_raw + S::OFF_GS);
  uint32_t* ms = reinterpret_cast<uint32_t*>(smem_raw + S::OFF_MS);
  double* s0 = reinterpret_cast<double*>(smem_raw + S::OFF_S0);
  double* s1 = reinterpret_cast<double*>(smem_raw + S::OFF_S1);
  double* xb = reinterpret_cast<double*>(smem_raw + S::OFF_XB);
  double* ex = reinterpret_cast<double*>(smem_raw + S::OFF_EX);
  // W (stage C -> D) and R (stage D -> E) regions: in-place bodies put W over T2
  double* sw = Body::IP ? s0 : s1;
  double* sr = Body::IP ? s1 : s0;

  constexpr bool DS = HasDs<Body>::value;
  uint64_t* bar_r = reinterpret_cast<uint64_t*>(smem_raw + S::OFF_DB);   // DS: ring barriers
  double* ring = reinterpret_cast<double*>(smem_raw + S::OFF_DB + 16);  // DS: two pair slots
  const int nbatch = (nel + E - 1) / E;
  if ((int)blockIdx.x >= nbatch) return;
  const bool dirichlet = ebits != nullptr;
  if (threadIdx.x == 0) {
    if constexpr (DS) {
      mbar_init(bar_r, 1);
      mbar_init(bar_r + 1, 1);
    }
    mbar_init(bar_d, 1);
#pragma unroll
    for (int s = 0; s < NG; ++s) mbar_init(bar_g + s, 1);
    fence_mbar_init();
  }
  // zero the work regions once: line padding stays finite (the DMMA body reads
  // K padding and relies on zero B-operand rows to annihilate it)
  for (size_t i = threadIdx.x; i < (S::BYTES - S::OFF_S0) / 8; i += T)
    reinterpret_cast<double*>(smem_raw + S::OFF_S0)[i] = 0.0;
  __syncthreads();
  Body::init(tb, ex);
  __syncthreads();

  // (thread 0) ids of batch b into slot: bulk copy of the id rows (GM 0) or
  // the per-element base ids (GM 1), plus the Dirichlet bits
  auto issue_g = [&](int b, int slot) {
    const int e0 = b * E, ne = min(E, nel - e0);
    if constexpr (GM == 1) {
      (void)ne;
      if (dirichlet) {
        const uint32_t mb = 4u * ne * G::MS;
        mbar_expect_tx(bar_g + slot, mb);
        bulk_g2s(ms + slot * E * G::MS, ebits + (size_t)e0 * G::MS, mb, bar_g + slot);
      }
    } else {
      const uint32_t gb = 4u * ne * G::GS, mb = dirichlet ? 4u * ne * G::MS : 0u;
      mbar_expect_tx(bar_g + slot, gb + mb);
      bulk_g2s(gs + slot * E * G::GS, gids + (size_t)e0 * G::GS, gb, bar_g + slot);
      if (dirichlet) bulk_g2s(ms + slot * E * G::MS, ebits + (size_t)e0 * G::MS, mb, bar_g + slot);
    }
  };
  // GM 1: base ids of batch b's elements into `slot`, one thread per element
  // (all threads call this; visible to the CTA after the next barrier)
  auto fill_base = [&](int b, int slot) {
    if constexpr (GM == 1) {
      const int e0 = b * E, ne = min(E, nel - e0);
      for (int e = threadIdx.x; e < ne; e += T) {
        const int eg = (int)(sid.e0 + e0 + e);  // local element counts are < 2^31
        const int eyz = fast_div(eg, sid.mnx, sid.snx), ez_ = fast_div(eyz, sid.mny, sid.sny);
        const int ex_ = eg - eyz * sid.nx, ey_ = eyz - ez_ * sid.ny;
        gs[slot * E + e] = ex_ * sid.p + sid.npx * (ey_ * sid.p + sid.npy * (ez_ * sid.p));
      }
    }
  };
  // global id of local node l of element e in gid slot `slot`
  auto gid_of = [&](int slot, int e, int l) -> int {
    if constexpr (GM == 1) {
      const int k = l / (D * D), j = (l / D) % D, i = l - D * (j + D * k);
      return gs[slot * E + e] + i + sid.npx * (j + sid.npy * k);
    } else {
      return gs[slot * E * G::GS + e * G::GS + l];
    }
  };
  auto issue_d = [&](int b) {
    if constexpr (MF || DS) return;
    const int e0 = b * E, ne = min(E, nel - e0);
    const uint32_t bytes = 8u * ne * G::PS;
    if constexpr (DG) {
      prefetch_l2(pa + (size_t)e0 * G::PS, bytes);
    } else {
      mbar_expect_tx(bar_d, bytes);
#ifdef FK_PA_NO_L2_HINT
      bulk_g2s(db, pa + (size_t)e0 * G::PS, bytes, bar_d);
#else
      bulk_g2s_hint(db, pa + (size_t)e0 * G::PS, bytes, bar_d, l2_policy_evict_first());
#endif
    }
  };
  // DS (thread 0): the plane windows of pair sp of batch b into ring slot `slot`
  [[maybe_unused]] auto issue_pair = [&](int b, int sp, int slot) {
    if constexpr (DS) {
      const int e0 = b * E, ne = min(E, nel - e0);
      const int c0 = sp, c1 = Q - 1 - sp, nh = c0 != c1 ? 2 : 1;
      uint32_t bytes = 0;
      for (int m = 0; m < Body::NPA; ++m)
        for (int h = 0; h < nh; ++h) bytes += 8u * Body::win_len(m, h ? c1 : c0);
      mbar_expect_tx(bar_r + slot, bytes * (uint32_t)ne);
      const double* pb = pa + (size_t)e0 * G::PS;
      double* dst = ring + slot * Body::SLOT;
      for (int e = 0; e < ne; ++e)
        for (int m = 0; m < Body::NPA; ++m)
          for (int h = 0; h < nh; ++h) {
            const int c = h ? c1 : c0;
            bulk_g2s(dst + Body::slot_at(e, m, h), pb + Body::win_off(e, m, c), 8u * Body::win_len(m, c),
                     bar_r + slot);
          }
    }
  };
  // XP: this thread's gather slots are the same in every batch, so their
  // X-buffer offsets, (element << 16 | node) and id offsets (GM 1: relative
  // to the element's base id, GM 0: into the slot's id rows) are computed once
  // here instead of per batch — the index arithmetic is ~20% of BP1's
  // instructions, but the extra live registers change ptxas' allocation of
  // the basis tables, so it is a per-geometry choice (cfgs 25-31, pa_inst.cu).
  constexpr int NXT = (E * D3 + T - 1) / T;
  constexpr bool XPRE = XP && NXT <= 8;
  int x_off[XPRE ? NXT : 1], x_el[XPRE ? NXT : 1], x_rel[XPRE ? NXT : 1];
  if constexpr (XPRE) {
#pragma unroll
    for (int r = 0; r < NXT; ++r) {
      const int t = threadIdx.x + r * T;
      int e = E, l = 0;
      if (t < E * D3) XA::map(t, e, l);
      x_off[r] = t < E * D3 ? XA::off(e, l) : 0;
      x_el[r] = (e << 16) | l;
      if constexpr (GM == 1) {
        const int k = l / (D * D), j = (l / D) % D, i = l - D * (j + D * k);
        x_rel[r] = i + sid.npx * (j + sid.npy * k);
      } else {
        x_rel[r] = e * G::GS + l;
      }
    }
  }
  auto issue_x = [&](int b, int gslot, double* xdst) {
    const int e0 = b * E, ne = min(E, nel - e0);
    if constexpr (XPRE) {
      const uint32_t xs = smem_u32(xdst);
#pragma unroll
      for (int r = 0; r < NXT; ++r) {
        const int e = x_el[r] >> 16;
        if (e >= E) continue;  // past the batch's E * D^3 slots
        if (e < ne) {
          const int g = GM == 1 ? gs[gslot * E + e] + x_rel[r] : gs[gslot * E * G::GS + x_rel[r]];
          cp_async8_s(xs + 8u * (uint32_t)x_off[r], x + g);
        } else {
          xdst[x_off[r]] = 0.0;
        }
      }
    } else {
      for (int t = threadIdx.x; t < E * D3; t += T) {
        int e, l;
        XA::map(t, e, l);
        double* dst = xdst + XA::off(e, l);
        if (e < ne) cp_async8_s(smem_u32(dst), x + gid_of(gslot, e, l));
        else *dst = 0.0;
      }
    }
    cp_async_commit();
  };
  // staged scatter (YS): y[gid] += yb[X offset] in issue_x's thread -> node map
  auto scatter_y = [&](int gslot, int ne, const double* yb) {
    if constexpr (XPRE) {
#pragma unroll
      for (int r = 0; r < NXT; ++r) {
        const int e = x_el[r] >> 16;
        if (e < ne) {
          const int g = GM == 1 ? gs[gslot * E + e] + x_rel[r] : gs[gslot * E * G::GS + x_rel[r]];
          atomicAdd(y + g, yb[x_off[r]]);
        }
      }
    } else {
      for (int t = threadIdx.x; t < E * D3; t += T) {
        int e, l;
        XA::map(t, e, l);
        if (e < ne) atomicAdd(y + gid_of(gslot, e, l), yb[XA::off(e, l)]);
      }
    }
  };
  auto finish_x = [&](int gslot, int ne, double* xsrc) {
    cp_async_wait_all();
    if (dirichlet) {
      const uint32_t* m = ms + gslot * E * G::MS;
      // same thread -> (e, l) map as issue_x: cp.async.wait_group only covers
      // this thread's own copies
      if constexpr (XPRE) {
#pragma unroll
        for (int r = 0; r < NXT; ++r) {
          const int e = x_el[r] >> 16, l = x_el[r] & 0xffff;
          if (e < ne && ((m[e * G::MS + (l >> 5)] >> (l & 31)) & 1u)) xsrc[x_off[r]] = 0.0;
        }
      } else {
        for (int t = threadIdx.x; t < E * D3; t += T) {
          int e, l;
          XA::map(t, e, l);
          if (e < ne && ((m[e * G::MS + (l >> 5)] >> (l & 31)) & 1u)) xsrc[XA::off(e, l)] = 0.0;
        }
      }
    }
  };
  // mbarrier phase bits of the gid slots (bit s) and of the D barrier
  uint32_t ph_g = 0u, ph_d = 0u;
  auto wait_g = [&](int slot) {
    if (GM == 1 && !dirichlet) return;  // base ids are plain smem stores (ordered by barriers)
    mbar_wait(bar_g + slot, (ph_g >> slot) & 1u);
    ph_g ^= 1u << slot;
  };

  const int stride = PERSIST ? (int)gridDim.x : nbatch;  // single-batch CTAs never see a next
  // prologue: ids of the first two batches, D of the first, x of the first
  if (threadIdx.x == 0) {
    issue_g(blockIdx.x, 0);
    if (blockIdx.x + stride < nbatch) issue_g(blockIdx.x + stride, 1);
    issue_d(blockIdx.x);
    if constexpr (DS) {  // pairs 0 and 1 of the global pair sequence (it * NP + pair)
      for (int g2 = 0; g2 < 2; ++g2) {
        const int bb = (int)blockIdx.x + (g2 / Body::NP) * stride;
        if (bb < nbatch) issue_pair(bb, g2 % Body::NP, g2);
      }
    }
  }
  if constexpr (GM == 1) {  // base ids of the first two batches
    fill_base(blockIdx.x, 0);
    if (blockIdx.x + stride < nbatch) fill_base(blockIdx.x + stride, 1);
    __syncthreads();
  }
  wait_g(0);
  issue_x(blockIdx.x, 0, xb);

  // element quadratic form (QF instances only: CG's p.Ap), per-thread partial
  // in a register; without QF the pointer is a compile-time null and stage C
  // carries no trace of it
  double qacc = 0.0;
  double* const qptr = QF ? &qacc : nullptr;
  auto run_batch = [&](int b, int it) {
    const int gslot = it % NG;
    double* xcur = SX ? xb : xb + (it & 1) * E * XS;
    double* xnext = SX ? xb : xb + ((it + 1) & 1) * E * XS;
    const int e0 = b * E, ne = min(E, nel - e0);
    const int nb = b + stride, nb2 = nb + stride;
    // DR: this batch's PA data into registers now, consumed in stage C
    [[maybe_unused]] typename DRegsOf<Body, DR>::type dreg;
    if constexpr (DR) Body::load_d(pa + (size_t)e0 * G::PS, ne, dreg);
    finish_x(gslot, ne, xcur);
    __syncthreads();
    if (nb < nbatch) {
      if constexpr (!SX) {
        wait_g((it + 1) % NG);
        issue_x(nb, (it + 1) % NG, xnext);
      }
      if (nb2 < nbatch && threadIdx.x == 0) {
        fence_proxy_async();
        issue_g(nb2, (it + 2) % NG);  // slot last read by batch b-1 (done)
      }
      if (nb2 < nbatch) fill_base(nb2, (it + 2) % NG);
    }
    Body::stage_a(tb, it, xcur, s1, ne, ex);
    __syncthreads();
    if constexpr (SX) {  // X(b) consumed: gather X(b+1) into the same buffer
      if (nb < nbatch) {
        wait_g((it + 1) % NG);
        issue_x(nb, (it + 1) % NG, xnext);
      }
    }
    if constexpr (HasBcd<Body>::value) {
      // stages B, C, D in registers (pa_eo_bcd.cuh): T1 -> R in place in region 1
      static_assert(!DG && !MF && !DR && !QF, "fused B-C-D reads the PA data from shared memory");
      mbar_wait(bar_d, ph_d);
      ph_d ^= 1u;
      Body::stage_bcd(tb, s1, db, ne);
      __syncthreads();
      if (nb < nbatch && threadIdx.x == 0) {
        fence_proxy_async();
        issue_d(nb);
      }
    } else {
      Body::stage_b(tb, it, s1, s0, ne, ex);
      __syncthreads();
      if constexpr (QF && HasQf<Body>::value) {
        if constexpr (MF) {
          Body::template stage_c<true>(tb, it, s0, nullptr, sw, ne, ex, qptr);
        } else if constexpr (DG) {
          Body::stage_c(tb, it, s0, pa + (size_t)e0 * G::PS, sw, ne, ex, qptr);
        } else {
          mbar_wait(bar_d, ph_d);
          ph_d ^= 1u;
          Body::stage_c(tb, it, s0, db, sw, ne, ex, qptr);
        }
      } else if constexpr (DS) {
        static_assert(!DG && !MF && !DR, "streamed PA data comes from the ring");
        Body::stage_c_ds(
            tb, it, s0, sw, ne,
            [&](int sp) -> const double* {
              const int gp = it * Body::NP + sp, slot = gp & 1;
              mbar_wait(bar_r + slot, (uint32_t)((gp >> 1) & 1));
              return ring + slot * Body::SLOT;
            },
            [&](int sp) {
              __syncthreads();  // every thread is done with this pair's slot
              if (threadIdx.x == 0) {
                const int gp = it * Body::NP + sp + 2;
                const int bb = b + (gp / Body::NP - it) * stride;
                if (bb < nbatch) {
                  fence_proxy_async();
                  issue_pair(bb, gp % Body::NP, gp & 1);
                }
              }
            });
      } else if constexpr (MF) {
        Body::template stage_c<true>(tb, it, s0, nullptr, sw, ne, ex);
      } else if constexpr (DR) {
        Body::stage_c_dr(tb, it, s0, dreg, sw, ne, ex);
      } else if constexpr (DG) {
        Body::stage_c(tb, it, s0, pa + (size_t)e0 * G::PS, sw, ne, ex);
      } else {
        mbar_wait(bar_d, ph_d);
        ph_d ^= 1u;
        Body::stage_c(tb, it, s0, db, sw, ne, ex);
      }
      __syncthreads();
      if (nb < nbatch && threadIdx.x == 0) {
        fence_proxy_async();
        issue_d(nb);
      }
      Body::stage_d(tb, it, sw, sr, ne, ex);
      __syncthreads();
    }
    if constexpr (YS) {
      // staged scatter: outputs into the dead W region (X layout), then the
      // RED.F64s in the gather's thread -> node order.  The next writer of sw
      // (stage A or B of the next batch) runs after that batch's first barrier.
      static_assert(Body::YS_FITS, "staged scatter needs the X layout to fit in the W region");
      Body::stage_e_stage(tb, it, sr, sw, ne, ex);
      __syncthreads();
      scatter_y(gslot, ne, sw);
    } else if constexpr (GM == 1) {
      Body::stage_e_ids(
          tb, it, sr, [&](int e, int j, int k) { return gs[gslot * E + e] + sid.npx * (j + sid.npy * k); },
          y, ne, ex);
    } else {
      Body::stage_e(tb, it, sr, gs + gslot * E * G::GS, y, ne, ex);
    }
    // no barrier here: every thread passes the barrier after the next batch's
    // finish_x only after its own stage E, and nothing before that barrier
    // touches the regions stage E reads (R, this batch's gid slot)
  };

  if constexpr (PERSIST) {
    int it = 0;
    for (int b = blockIdx.x; b < nbatch; b += gridDim.x, ++it) run_batch(b, it);
  } else {
    // one batch per CTA: no loop, so the compiler has nothing to hoist the
    // basis-table loads out of (co-resident CTAs overlap load and compute)
    run_batch(blockIdx.x, 0);
  }
  if constexpr (QF && HasQf<Body>::value) {
    {  // CTA partial of the quadratic form, fixed reduction order
      __shared__ double qw[(T + 31) / 32];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) qacc += __shfl_down_sync(0xffffffffu, qacc, o);
      if ((threadIdx.x & 31) == 0) qw[threadIdx.x >> 5] = qacc;
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (T + 31) / 32; ++w) s += qw[w];
        sid.qf[blockIdx.x] = s;
      }
    }
  }
}

}  // namespace fk
