// pipelined.cuh — building blocks shared by the TMA-fed tile kernels:
// the two-phase tile item (load layout L0 -> butterflies -> shared-memory
// transpose -> layout L1 -> butterflies -> global store), the f32 m = 12 item
// that K1T (k1t.cuh) runs, and the tile geometry of the m = 24 two-pass
// schedule K4T (passtma.cuh).  (The cp.async-pipelined kernels K1P / K5P /
// K4P that first used these items were measured slower than their TMA-fed
// successors and removed in round 2.)
#pragma once

#include "fused.cuh"

namespace chwb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Gather one tile into a swizzled shared stage with 16-byte cp.async, using the
// load layout L (register bits 0..1 must be element bits 0..1: one float4).
template <class L, class MapIn, class S>
__device__ __forceinline__ void issue_tile_copy(float* stage, const float* gsrc, uint32_t tid) {
  static_assert(vec_bits<L, MapIn>(2) == 2, "copy layout needs float4 vectors");
  static_assert(smem_vec_bits<L, S, 2>() == 2, "swizzle splits the float4 vectors");
  constexpr uint32_t tmask = S::image(thr_mask<L, IdMap>());
  const uint32_t tg = thr_off<L, MapIn>(tid);
  const uint32_t ts = S::apply(thr_off<L, IdMap>(tid));
#pragma unroll
  for (int r = 0; r < L::E; ++r) {
    if (!vec_head<L, MapIn>(r, 2)) continue;
    const uint32_t so = S::apply(reg_off<L, IdMap>(r));
    const uint32_t a = (so & tmask) ? (ts ^ so) : (ts + so);
    cp_async16(stage + a, gsrc + (tg + reg_off<L, MapIn>(r)));
  }
}

// A two-phase item type.  The prefetch stage keeps the natural tile order
// (SStage = identity: the load layouts put lanes on element bits 2..4, so the
// 16-byte cp.async writes and LDS.128 reads are conflict-free); the transpose
// buffer uses the plan's swizzle S.
template <class L0_, class L1_, class S_, class B0_, class B1_, int SHFL_, class MapIn_, class MapOut_,
          Cache COUT_, class SStage_ = NoSwz>
struct TwoPhase {
  using L0 = L0_;
  using L1 = L1_;
  using S = S_;
  using SStage = SStage_;
  using MapIn = MapIn_;
  using MapOut = MapOut_;
  static constexpr int E = L0::E;
  static constexpr int TILE = 1 << L0::T_BITS;

  __device__ __forceinline__ static void copy(float* stage, const float* gsrc, uint32_t tid) {
    issue_tile_copy<L0, MapIn, SStage>(stage, gsrc, tid);
  }
  __device__ __forceinline__ static void phase0(const float* stage, float* work, float (&v)[E],
                                                uint32_t tid) {
    smem_load<L0, SStage>(stage, v, tid);
    butterflies<L0, B0_, false>(v);
    smem_store<L0, S>(work, v, tid);
  }
  template <bool SCALE, class TOut>
  __device__ __forceinline__ static void phase1(const float* work, TOut* gout, float (&v)[E], uint32_t tid,
                                                float scale, uint32_t outer = 0) {
    smem_load<L1, S>(work, v, tid);
    butterflies<L1, B1_, false>(v);
    if constexpr (SHFL_ >= 0) shfl_butterfly<L1, SHFL_, false>(v, tid);
    store_global<L1, MapOut, SCALE, COUT_>(gout, v, tid, scale, outer);
  }
};

// f32 m = 12 (cfg2) item with the PlanF32M12 layouts (run by K1T).
struct PipeF32M12 {
  static constexpr int M = 12;
  static constexpr int NT = 64;
  static constexpr int STAGES = 4;      // measured sweep: 4 stages x 2 CTAs/SM best
  static constexpr int MIN_BLOCKS = 2;
  using Item = TwoPhase<PlanF32M12::L0, PlanF32M12::L1, PlanF32M12::S, BL<0, 1, 8, 9, 10, 11>,
                        BL<2, 3, 4, 5, 6, 7>, -1, IdMap, RevMap<12>, Cache::kStream>;
  static constexpr int TILE = Item::TILE;
  static constexpr int SMEM_BYTES = (STAGES + 1) * TILE * 4;
};

// Geometry of the m = 24 two-pass schedule (tiles of FusedF32M24).
struct GeoA24 {
  __device__ __forceinline__ static uint64_t src_off(uint64_t it) { return it << 14; }
  __device__ __forceinline__ static uint64_t dst_off(uint64_t it) { return it << 14; }
};
struct GeoB24 {
  __device__ __forceinline__ static uint64_t src_off(uint64_t it) {
    return ((it >> 10) << 24) | deposit<FusedF32M24::B::OuterAddr>((uint32_t)(it & 1023u));
  }
  __device__ __forceinline__ static uint64_t dst_off(uint64_t it) {
    return ((it >> 10) << 24) | deposit<FusedF32M24::B::OuterOut>((uint32_t)(it & 1023u));
  }
};

}  // namespace chwb
