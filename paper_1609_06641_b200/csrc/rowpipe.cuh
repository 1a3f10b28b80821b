// rowpipe.cuh — K6: warp-specialized per-CTA row pipeline for f32 m = 16
// (BASELINE cfg4).
//
// Every persistent CTA (one per SM) owns whole rows (c, c + G, c + 2G, ...)
// and runs BOTH phases of the two-phase transform on them, so no CTA ever
// waits for another:
//   A(i, k): contiguous 16 KiB input tile k of the CTA's i-th row -> butterflies
//            on row bits 0..7 -> the CTA's private workspace row W;
//   B(i, k): column tile k of W -> butterflies on row bits 8..15 -> dyadic output.
// W is ONE row per CTA (256 KiB, 37 MiB over 148 SMs), so it stays in L2: HBM
// sees one read and one write per element, the intermediate only crosses the
// SM<->L2 interface (measured 12.4 TB/s copy, 17.4 TB/s read:
// profiles/r01_l2_probe_kernel.txt).  Consecutive rows alternate between two
// workspace bit layouts (P and its image under the swap of W bits 4..7 <->
// 12..15) so that A(i+1, k) overwrites exactly the region B(i, k) consumed.
//
// Measured alternatives: two workspace rows per CTA spill W to
// HBM (74 MiB, +50-90% DRAM bytes); cp.async prefetch completes in issue order,
// so a row's first W tile waited for freshly issued HBM prefetches; a single
// 4-warp compute group per SM is latency bound.  Hence TMA (per-stage mbarrier
// completion), 8 compute warps in two decoupled groups, and a producer warp per
// stream.
#pragma once

#include "pipelined.cuh"

namespace chwb {

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Drop (without write-back) the 128-byte L2 lines of a dead workspace region.
__device__ __forceinline__ void discard_l2_128(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// HINT bit 0: workspace stores evict_last, input loads evict_first.
// HINT bit 1: before a layout-0 A tile overwrites its contiguous 16 KiB
//             workspace region, discard the region's dead lines (no write-back).
// ORD: 0 dyadic, 1 natural, 2 sequency (chw_order).
template <int HINT_, int ORD = 0>
struct RowPipeF32M16 {
  using F = FusedF32M16b;
  static constexpr int M = 16;
  static constexpr int NT = F::NT;
  static constexpr int TILES = 16;  // A and B tiles per row
  static constexpr int HINT = HINT_;
  static constexpr bool HINT_DISCARD = (HINT & 2) != 0;
  static constexpr Cache CW = (HINT_ & 1) ? Cache::kL2Last : Cache::kL2;
  // layout P (= FusedF32M16b's Pi) and its swapped image P'
  using MapOutA1 = ListMap<2, 3, 0, 1, 15, 12, 13, 14, 8, 9, 10, 11>;
  // B tiles read layout 1 in this tile order (MapInB1: tile bit -> W bit);
  // the TMA tensor map of layout 1 (launch.cuh: rowpipe_tmaps) realises it.
  using MapInB1 = ListMap<0, 1, 2, 3, 8, 9, 10, 11, 4, 5, 6, 7>;
  using ItemA0 = TwoPhase<F::A::L0, F::A::L1, F::A::S, F::A::B0, F::A::B1, -1, IdMap, F::A::MapOut, CW>;
  using ItemA1 = TwoPhase<F::A::L0, F::A::L1, F::A::S, F::A::B0, F::A::B1, -1, IdMap, MapOutA1, CW>;
  // B tile layouts (tile bits as FusedF32M16b::B; butterflies on tile bits
  // 4..11): the second layout holds output bits 0..1 (tile bits 11, 10) in
  // registers, so the dyadic stores are 16-byte vectors in whole 64-byte runs
  // (FusedF32M16b's B stores single floats); conflict-free (tools/plan_check.py).
  using BL0 = Layout<BL<0, 1, 5, 8, 9>, BL<2, 3, 4, 6, 7, 10, 11>>;
  using BL1 = Layout<BL<4, 6, 7, 10, 11>, BL<9, 8, 5, 0, 1, 2, 3>>;
  using BS = Swz<5, 2, 8, 3, 9, 4>;
  // Output orders (f2).  Sequency: inverse Gray code of the dyadic position.
  // Natural: position = j; the B tile's passengers are j0..j3 (workspace
  // addr 0..3 = j2, j3, j0, j1), so every tile still writes whole 64-byte
  // runs (scalar stores; the dyadic order's 16-byte vectors need the tile's
  // butterfly bits low), and its index bits (addr 4..7 = j5, j6, j7, j4)
  // place the tile.
  using MapOutNat = ListMap<2, 3, 0, 1, 8, 9, 10, 11, 12, 13, 14, 15>;
  using OuterOutNat = BL<5, 6, 7, 4>;
  using MapOutB = typename std::conditional<
      ORD == 2, SeqMap<F::B::MapOut, 16>,
      typename std::conditional<ORD == 1, MapOutNat, F::B::MapOut>::type>::type;
  using OuterOutB = typename std::conditional<ORD == 1, OuterOutNat, F::B::OuterOut>::type;
  using ItemB0 = TwoPhase<BL0, BL1, BS, BL<5, 8, 9>, BL<4, 6, 7, 10, 11>, -1, F::B::MapIn, MapOutB,
                          Cache::kStream>;
  static constexpr int TILE = ItemA0::TILE;
  static_assert(TILE == ItemB0::TILE && ItemA0::E == ItemB0::E, "A and B tiles must match");
  // workspace offsets of tile k in layout 0 / 1
  __device__ __forceinline__ static uint32_t a_off(uint32_t k, uint32_t lay) {
    return lay ? deposit<F::B::OuterAddr>(k) : (k << 12);
  }
  __device__ __forceinline__ static uint32_t b_off(uint32_t k, uint32_t lay) {
    return lay ? (k << 12) : deposit<F::B::OuterAddr>(k);
  }
};

__device__ __forceinline__ void mbar_init_cta(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_cta(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
#ifndef CHW_MBAR_HINT
#define CHW_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait_cta(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
#if CHW_MBAR_HINT
    // suspend-time hint (ns): the warp sleeps in hardware until the phase
    // completes instead of re-polling every few hundred cycles
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"((uint32_t)CHW_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
#endif
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tensor3_g2s(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tensor4_g2s(void* dst, const void* tmap, int x, int y, int z, int w, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 128-byte opaque tensor map (CUtensorMap) passed by value as a grid constant.
struct __align__(64) TmapParam {
  unsigned char b[128];
};

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---------------------------------------------------------------------------
// K6f: K6e with two compute groups per stream (16 compute warps per SM).
// Group (s, p) runs the items t = p (mod 2) of stream s; transpose tiles are
// single-buffered (two named barriers per item).  rowstored counts both A
// groups (each arrives after its last tile of the row; neither can reach the
// next row's last tile first, as that needs the row's B tiles, which need
// both arrivals).
// ---------------------------------------------------------------------------
template <class P, int SA, int SB, bool SCALE>
__global__ void __launch_bounds__(4 * P::NT + 64, 1)
    rowpipe_ws4_kernel(const float* __restrict__ in, float* __restrict__ out, float* __restrict__ ws, uint64_t rows,
                       float scale, const __grid_constant__ TmapParam tmap0, const __grid_constant__ TmapParam tmap1) {
  constexpr int TILE = P::TILE;
  constexpr uint32_t TB = TILE * 4;
  constexpr uint64_t n = 1ull << P::M;
  constexpr int NT = P::NT;
  // Each stage must always be consumed by the same group (item parity), else a
  // group running ahead could pass a parity wait on the stage's previous phase.
  static_assert(SA % 2 == 0 && SB % 2 == 0, "ring depths must be even");
  extern __shared__ __align__(128) float smem_w4[];
  float* ringA = smem_w4;
  float* ringB = smem_w4 + SA * TILE;
  float* works = smem_w4 + (SA + SB) * TILE;  // 4 tiles, one per group
  __shared__ __align__(8) uint64_t fullA[SA], emptyA[SA], fullB[SB], emptyB[SB], regionfree[16], rowstored;
  const uint32_t tid = threadIdx.x;
  const uint64_t G = gridDim.x;
  const uint64_t c = blockIdx.x;
  if (c >= rows) return;
  const uint32_t R = (uint32_t)((rows - 1 - c) / G + 1);
  const uint32_t nst = 16u * R;
  float* wsc = ws + c * n;
  if (tid == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init_cta(&fullA[s], 1);
      mbar_init_cta(&emptyA[s], 1);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init_cta(&fullB[s], 1);
      mbar_init_cta(&emptyB[s], 1);
    }
    for (int k = 0; k < 16; ++k) mbar_init_cta(&regionfree[k], 1);
    mbar_init_cta(&rowstored, 2);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t warp = tid >> 5, lane = tid & 31u;
  if (warp >= 16) {
    if (lane != 0) return;
    if (warp == 16) {
      const uint64_t pol_in = (P::HINT & 1) ? l2_evict_first_policy() : l2_evict_normal_policy();
      for (uint32_t t = 0; t < nst; ++t) {
        const int st = t % SA;
        if (t >= (uint32_t)SA) mbar_wait_cta(&emptyA[st], ((t / SA) - 1) & 1u);
        mbar_expect_tx_cta(&fullA[st], TB);
        bulk_g2s(ringA + st * TILE, in + (c + (uint64_t)(t >> 4) * G) * n + ((t & 15u) << 12), TB, &fullA[st],
                 pol_in);
      }
    } else {
      for (uint32_t t = 0; t < nst; ++t) {
        const uint32_t i = t >> 4, kk = t & 15u;
        if (kk == 0) mbar_wait_cta(&rowstored, i & 1u);
        const int st = t % SB;
        if (t >= (uint32_t)SB) mbar_wait_cta(&emptyB[st], ((t / SB) - 1) & 1u);
        mbar_expect_tx_cta(&fullB[st], TB);
        if (i & 1u)
          tensor4_g2s(ringB + st * TILE, &tmap1, 0, 0, 0, (int)(c * 16u + kk), &fullB[st]);
        else
          tensor3_g2s(ringB + st * TILE, &tmap0, 0, (int)kk, (int)(c * 256u), &fullB[st]);
      }
    }
    return;
  }
  const uint32_t grp = warp >> 2;        // 0,1: A stream; 2,3: B stream
  const uint32_t par = grp & 1u;         // item parity of this group
  const uint32_t bar = 1 + grp;          // named barrier id
  const uint32_t gt = tid & (NT - 1);
  float* work = works + grp * TILE;
  float v[P::ItemA0::E];
  if (grp < 2) {
    for (uint32_t t = par; t < nst; t += 2) {
      const int st = t % SA;
      const uint32_t i = t >> 4, kk = t & 15u;
      mbar_wait_cta(&fullA[st], (t / SA) & 1u);
      P::ItemA0::phase0(ringA + st * TILE, work, v, gt);
      named_bar(bar, NT);
      if (gt == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&emptyA[st])) : "memory");
      if (i >= 1) mbar_wait_cta(&regionfree[kk], (i - 1) & 1u);
      float* dst = wsc + P::a_off(kk, i & 1u);
      if (i & 1u)
        P::ItemA1::template phase1<false>(work, dst, v, gt, scale);
      else
        P::ItemA0::template phase1<false>(work, dst, v, gt, scale);
      if (kk >= 14u) {  // this group's last tile of the row
        asm volatile("fence.proxy.async.global;" ::: "memory");
        named_bar(bar, NT);
        if (gt == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&rowstored)) : "memory");
      } else {
        named_bar(bar, NT);  // work tile free for the next phase0
      }
    }
  } else {
    for (uint32_t t = par; t < nst; t += 2) {
      const int st = t % SB;
      const uint32_t i = t >> 4, kk = t & 15u;
      mbar_wait_cta(&fullB[st], (t / SB) & 1u);
      P::ItemB0::phase0(ringB + st * TILE, work, v, gt);
      named_bar(bar, NT);
      if (gt == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&emptyB[st])) : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&regionfree[kk])) : "memory");
      }
      const uint64_t row = c + (uint64_t)i * G;
      P::ItemB0::template phase1<SCALE>(work, out + row * n, v, gt, scale, deposit<typename P::OuterOutB>(kk));
      named_bar(bar, NT);  // work tile free for the next phase0
    }
  }
}

}  // namespace chwb
