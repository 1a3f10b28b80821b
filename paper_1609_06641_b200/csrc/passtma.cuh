// passtma.cuh — K4T: the m = 24 two-pass schedule (K4P, pipelined.cuh) fed by
// the TMA engine.  One persistent CTA per SM, a producer thread and one
// 8-warp compute group.  The 64 KiB tiles are transposed IN PLACE in their
// ring stage (registers hold the whole tile between the read and the
// swizzled write-back), so the 192 KiB of shared memory hold three tiles in
// flight instead of K4P's two stages plus a separate transpose buffer.
//   pass A: contiguous 64 KiB input tile (one bulk copy) -> intermediate;
//   pass B: 8-column x 2048-row tile of the intermediate (one 5-D tensor copy,
//           box order = tile order) -> dyadic output.
#pragma once

#include "rowpipe.cuh"

namespace chwb {

template <class L0_, class L1_, class S_, class B0_, class B1_, int SHFL_, class MapOut_, Cache COUT_>
struct InPlaceItem {
  using L0 = L0_;
  using L1 = L1_;
  using S = S_;
  static constexpr int E = L0::E;
  static constexpr int TILE = 1 << L0::T_BITS;
  static constexpr int NT = L0::NT;
  // stage (natural tile order) -> registers -> butterflies -> stage (swizzled) ->
  // registers in L1 -> butterflies; `bar` orders the group's shared accesses.
  template <class Bar>
  __device__ __forceinline__ static void compute(float* stage, float (&v)[E], uint32_t tid, Bar bar) {
    smem_load<L0, NoSwz>(stage, v, tid);
    butterflies<L0, B0_, false>(v);
    bar();
    smem_store<L0, S>(stage, v, tid);
    bar();
    smem_load<L1, S>(stage, v, tid);
  }
  template <bool SCALE>
  __device__ __forceinline__ static void finish(float* gout, float (&v)[E], uint32_t tid, float scale) {
    butterflies<L1, B1_, false>(v);
    if constexpr (SHFL_ >= 0) shfl_butterfly<L1, SHFL_, false>(v, tid);
    store_global<L1, MapOut_, SCALE, COUT_>(gout, v, tid, scale);
  }
};

struct PassTmaF32M24 {
  using F = FusedF32M24;
  using ItemA = InPlaceItem<F::A::L0, F::A::L1, F::A::S, BL<0, 1, 9, 10, 11, 12>, BL<2, 3, 4, 5, 6, 7>, 8,
                            F::A::MapOut, Cache::kL2>;
  using ItemB = InPlaceItem<F::B::L0, F::B::L1, F::B::S, BL<10, 11, 12, 13>, BL<3, 4, 5, 6, 7, 8>, 9,
                            F::B::MapOut, Cache::kStream>;
  static constexpr int TILE = ItemA::TILE;
  static constexpr int NT = ItemA::NT;
};

// GEO: GeoA24 / GeoB24 (pipelined.cuh).  TENSOR: the source tile is loaded with
// the 5-D tensor map (pass B), else one contiguous bulk copy (pass A).
template <class Item, class Geo, bool TENSOR, int S, bool SCALE>
__global__ void __launch_bounds__(Item::NT + 32, 1)
    pass_tma_kernel(const float* __restrict__ src, float* __restrict__ dst, uint64_t nitems, float scale,
                    const __grid_constant__ TmapParam tmap) {
  constexpr int TILE = Item::TILE;
  constexpr uint32_t TB = TILE * 4;
  constexpr int NT = Item::NT;
  extern __shared__ __align__(128) float smem_pt[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const uint32_t tid = threadIdx.x;
  const uint64_t G = gridDim.x, c = blockIdx.x;
  if (c >= nitems) return;
  const uint64_t nu = (nitems - 1 - c) / G + 1;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init_cta(&full[s], 1);
      mbar_init_cta(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= (uint32_t)NT) {  // producer warp
    if (tid != (uint32_t)NT) return;
    const uint64_t pol = l2_evict_first_policy();
    for (uint64_t u = 0; u < nu; ++u) {
      const int st = (int)(u % S);
      const uint64_t it = c + u * G;
      if (u >= (uint64_t)S) mbar_wait_cta(&empty[st], (uint32_t)((u / S) - 1) & 1u);
      mbar_expect_tx_cta(&full[st], TB);
      float* stage = smem_pt + st * TILE;
      if constexpr (TENSOR) {
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5, %6}], [%7];" ::"r"(smem_u32(stage)),
            "l"(&tmap), "r"(0), "r"((int)(it & 1023u)), "r"(0), "r"(0), "r"((int)(it >> 10)), "r"(smem_u32(&full[st]))
            : "memory");
      } else {
        bulk_g2s(stage, src + Geo::src_off(it), TB, &full[st], pol);
      }
    }
    return;
  }
  auto bar = [] { named_bar(1, NT); };
  float v[Item::E];
  for (uint64_t u = 0; u < nu; ++u) {
    const int st = (int)(u % S);
    float* stage = smem_pt + st * TILE;
    mbar_wait_cta(&full[st], (uint32_t)(u / S) & 1u);
    Item::compute(stage, v, tid, bar);
    bar();  // every thread has read the stage: hand it back to the producer
    if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    Item::template finish<SCALE>(dst + Geo::dst_off(c + u * G), v, tid, scale);
  }
}

}  // namespace chwb
