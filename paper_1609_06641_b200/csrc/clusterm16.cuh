// clusterm16.cuh — K10: thread-block-cluster / DSMEM kernel for f32 m = 16
// (BASELINE cfg4): ONE HBM pass with NO intermediate in L2.
//
// Selected with CHW_B200_M16=c; NOT the default: measured 0.54 of the HBM peak
// against K6's 0.73 (profiles/r02_ab_cluster_m16.txt).  The exchange moves
// 48 KiB out of and into every CTA per 128 KiB of HBM traffic, and the
// SM-to-SM path sustains ~17-21 B/clk per SM (B300_MICROARCH.md), i.e. it
// saturates at about the HBM roofline itself; 4-CTA clusters also leave 16 of
// the 148 SMs idle.  Kept (and parity-tested) as the measured answer to "can
// the row stay on chip": K6's L2 workspace is the faster exchange medium.
//
// K6 (rowpipe.cuh) sends every row through an L2-resident workspace; a
// no-arithmetic probe of that byte pattern (tools/mix_probe.cu,
// profiles/r02_mix_probe.txt) tops out at 0.70-0.73 of the copy peak for a
// 16-48 MiB workspace, and K6 sits on that ceiling.  K10 keeps the whole row on
// chip instead: a cluster of 4 CTAs owns a row, CTA k holds the contiguous
// quarter (j15, j14) = k (64 KiB) and the cross-quarter exchange goes through
// distributed shared memory.
//
//   1. TMA bulk copy of the quarter into the group's stage S (natural order);
//   2. layout L0 (registers j0, j1, j9..j12): butterflies on those 6 bits;
//      in-place transpose in S (swizzle S1) to layout L1 (registers j2..j6,
//      j13): 6 more bits — all 14 in-quarter bits but j7, j8 are done;
//   3. exchange: the thread's 64 values belong to CTA p = (j1, j0) of the
//      cluster.  They are stored (16-byte vectors, the receiver's swizzle)
//      into a 16 KiB block per destination — the own block straight into the
//      own buffer, the other three into an outgoing area — and one
//      cp.async.bulk per peer moves a block shared::cta -> shared::cluster
//      into slot k of the peer's buffer, completing bytes on the peer's `recv`
//      mbarrier.  A buffer is free once its CTA has passed step 2 (`ready`:
//      one remote mbarrier arrive from every CTA).  (16-byte st.async stores
//      from registers measured 0.49 of the HBM peak: the SM-to-SM path takes
//      ~20 B/clk and the stores queue in the LSU in front of everything else.)
//   4. layout LR (registers j15, j14, j7, j8 + the carried vector bits j2, j3):
//      the last four butterflies, scale, 16-byte dyadic stores — CTA p writes
//      the contiguous output quarter (out bits 15, 14) = (j0, j1), 512 bytes
//      per warp instruction.
//
// Two groups of 256 threads per CTA work on alternate rows of the cluster
// (each with its own 64 KiB buffer, 48 KiB outgoing area and mbarriers), so
// one group's loads, cluster waits and copies overlap the other group's
// arithmetic.  All layouts and
// swizzles are conflict-free in tools/plan_check.py.
#pragma once

#include "rowpipe.cuh"

namespace chwb {

struct ClusterF32M16 {
  static constexpr int M = 16;
  static constexpr int CL = 4;           // CTAs per cluster
  static constexpr int NT = 256;         // threads per group
  static constexpr int TILE = 1 << 14;   // floats per quarter
  // quarter tile, tile bit k = j bit k
  using L0 = Layout<BL<0, 1, 9, 10, 11, 12>, BL<2, 3, 4, 5, 6, 7, 8, 13>>;
  using L1 = Layout<BL<2, 3, 4, 5, 6, 13>, BL<7, 8, 9, 0, 1, 10, 11, 12>>;
  using S1 = Swz<7, 2, 8, 3, 9, 4>;
  using B0 = BL<0, 1, 9, 10, 11, 12>;
  using B1 = BL<2, 3, 4, 5, 6, 13>;
  // exchange tile (the receiver's stage), bits e0..e13 =
  //   j2, j3, j7, j8, j9, j10, j11, j12, j13, j4, j5, j6, j14, j15.
  // Writer: L1's registers in e numbering; tid bits 3, 4 = j0, j1 pick the
  // destination CTA, the other six tid bits are its thread index; e12, e13 =
  // the writer's rank (the slot in the destination's buffer).
  using LW = Layout<BL<0, 1, 9, 10, 11, 8>, BL<2, 3, 4, 5, 6, 7>>;
  using LR = Layout<BL<13, 12, 2, 3, 0, 1>, BL<4, 5, 6, 7, 8, 9, 10, 11>>;
  using SX = Swz<5, 2, 6, 3>;
  using BR = BL<13, 12, 2, 3>;
  // dyadic output position (bit q = j bit 15 - q) of exchange-tile bit e_k
  using MapOut = ListMap<13, 12, 8, 7, 6, 5, 4, 3, 2, 11, 10, 9, 1, 0>;
  static constexpr int E = L0::E;
  static_assert(L0::NT == NT && L1::NT == NT && LR::NT == NT && LW::NT == NT / 4 && L1::E == E && LR::E == E &&
                    LW::E == E,
                "group shape");
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local_smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, "
        "p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_s2dsmem(uint32_t remote_dst, const void* src, uint32_t bytes,
                                             uint32_t remote_bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(remote_dst),
      "r"(smem_u32(src)), "r"(bytes), "r"(remote_bar)
      : "memory");
}

// Registers of layout LW -> one 16 KiB exchange block at `blk` (the block of
// the thread's destination CTA), in the receiver's addressing (swizzle S).
template <class LW, class S, int E>
__device__ __forceinline__ void exchange_store(float* blk, const float (&v)[E], uint32_t tw) {
  constexpr int VB = smem_vec_bits<LW, S, 2>();
  static_assert(VB == 2, "exchange stores are 16-byte vectors");
  constexpr uint32_t tmask = S::image(thr_mask<LW, IdMap>());
  const uint32_t sb = S::apply(thr_off<LW, IdMap>(tw));
  static_for<LW::E>([&](auto R) {
    constexpr int r = decltype(R)::value;
    if constexpr (vec_head<LW, IdMap>(r, VB)) {
      constexpr uint32_t so = S::apply(reg_off<LW, IdMap>(r));
      const uint32_t a = (so & tmask) ? (sb ^ so) : (sb + so);
      float tmp[4];
      static_for<4>([&](auto Q) { tmp[decltype(Q)::value] = v[vec_elem<LW, IdMap>(r, decltype(Q)::value, VB)]; });
      SmemVec<float, 2>::st(blk + a, tmp);
    }
  });
}

template <bool SCALE>
__global__ void __launch_bounds__(2 * ClusterF32M16::NT, 1)
    cluster_m16_kernel(const float* __restrict__ in, float* __restrict__ out, uint32_t rows, float scale) {
  using P = ClusterF32M16;
  constexpr int TILE = P::TILE;
  constexpr int BLK = TILE / P::CL;  // floats per exchange block (16 KiB)
  constexpr uint32_t TB = TILE * 4;
  constexpr int NT = P::NT;
  extern __shared__ __align__(128) float smem_cl[];
  __shared__ __align__(8) uint64_t full[2], ready[2], recv[2];
  const uint32_t tid = threadIdx.x;
  const uint32_t k = cluster_ctarank();  // quarter (j15, j14) this CTA loads
  const uint32_t ncl = gridDim.x / P::CL, cid = blockIdx.x / P::CL;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init_cta(&full[b], 1);
      mbar_init_cta(&ready[b], P::CL);
      mbar_init_cta(&recv[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();  // every CTA's mbarriers exist before any remote arrive
  const uint32_t g = tid / NT, gt = tid % NT;
  float* S = smem_cl + g * TILE;                            // the group's row buffer
  float* T = smem_cl + 2 * TILE + g * (P::CL - 1) * BLK;    // its three outgoing exchange blocks
  const uint32_t barid = 1 + g;
  auto bar = [barid] { named_bar(barid, NT); };
  // rows of this cluster: cid, cid + ncl, ...; group g takes every other one
  const uint32_t nrows = cid < rows ? (rows - 1 - cid) / ncl + 1 : 0;
  uint64_t pol = 0;
  auto issue = [&](uint32_t i) {  // quarter k of the cluster's i-th row -> S (S is free)
    const uint64_t row = cid + (uint64_t)i * ncl;
    mbar_expect_tx_cta(&full[g], TB);
    bulk_g2s(S, in + (row << 16) + ((uint64_t)k << 14), TB, &full[g], pol);
  };
  if (gt == 0) {
    pol = l2_evict_first_policy();
    if (g < nrows) issue(g);
  }
  // destination of this thread's values: CTA p = (j1, j0) = tid bits 4, 3
  const uint32_t p = (gt >> 3) & 3u;
  const uint32_t tw = (gt & 7u) | ((gt >> 5) << 3);
  // own block: straight into slot k of the own buffer; others: outgoing block
  float* blk = (p == k) ? S + k * BLK : T + (p < k ? p : p - 1) * BLK;
  float v[P::E];
  uint32_t it = 0;  // rows this group has processed (mbarrier phase)
  for (uint32_t i = g; i < nrows; i += 2, ++it) {
    const uint32_t ph = it & 1u;
    mbar_wait_cta(&full[g], ph);
    smem_load<P::L0, NoSwz>(S, v, gt);
    butterflies<P::L0, P::B0, false>(v);
    bar();
    smem_store<P::L0, P::S1>(S, v, gt);
    bar();
    smem_load<P::L1, P::S1>(S, v, gt);
    bar();  // every thread has read S: peers may overwrite it
    if (gt == 0) {
      mbar_expect_tx_cta(&recv[g], (P::CL - 1) * BLK * 4);  // 3 x 16 KiB arrive from the peers
#pragma unroll
      for (uint32_t q = 0; q < (uint32_t)P::CL; ++q) mbar_arrive_remote(mapa_u32(smem_u32(&ready[g]), q));
    }
    butterflies<P::L1, P::B1, false>(v);
    // All four buffers of this row are free.  It also means every peer has
    // consumed the blocks this group sent for its previous row (a peer's
    // `ready` arrive follows its read of that row), so T may be overwritten.
    mbar_wait_cluster(&ready[g], ph);
    exchange_store<P::LW, P::SX>(blk, v, tw);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // T: generic writes -> bulk-copy reads
    bar();
    if (gt < (uint32_t)(P::CL - 1)) {  // one thread per peer: 16 KiB block -> slot k of the peer's buffer
      const uint32_t q = gt < k ? gt : gt + 1;
      bulk_s2dsmem(mapa_u32(smem_u32(S + k * BLK), q), T + gt * BLK, BLK * 4, mapa_u32(smem_u32(&recv[g]), q));
    }
    mbar_wait_cluster(&recv[g], ph);  // the peers' three blocks have landed in S
    smem_load<P::LR, P::SX>(S, v, gt);
    bar();  // S is read: refill it with this group's next row
    if (gt == 0 && i + 2 < nrows) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + 2);
    }
    butterflies<P::LR, P::BR, false>(v);
    const uint64_t row = cid + (uint64_t)i * ncl;
    const uint32_t outer = ((k & 1u) << 15) | ((k >> 1) << 14);
    store_global<P::LR, P::MapOut, SCALE, Cache::kStream>(out + (row << 16), v, gt, scale, outer);
  }
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

}  // namespace chwb
