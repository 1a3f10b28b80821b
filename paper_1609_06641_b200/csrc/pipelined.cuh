// pipelined.cuh — software-pipelined persistent tile kernel (K1P / K5P).
//
// Persistent CTAs walk a list of work items.  Each item is one "two-phase"
// tile (load layout L0 -> butterflies -> shared-memory transpose -> layout L1
// -> butterflies -> global store).  Input tiles are prefetched S items ahead
// with cp.async 16-byte gathers straight into swizzled shared-memory stages
// (no registers, no L1), so every CTA keeps S tiles of HBM traffic in flight
// while it computes — the memory-level parallelism the one-tile-per-CTA K1
// kernel only gets from occupancy.
//
// Per item k (stage s = k % S, work buffer k & 1):
//   cp.async.wait_group(S-1); bar.sync            (item k landed, ring visible)
//   [publish completion of item k-1]              (dataflow schedules only)
//   L0 <- stage s; butterflies; work[k&1] <- L0
//   bar.sync                                      (stage s free, work visible)
//   issue cp.async for item k+S into stage s      (or defer: dependency open)
//   L1 <- work[k&1]; butterflies; global stores
//
// Schedules: StaticSched (independent items, round-robin — K1) and the fused
// two-phase dataflow schedule of fused.cuh (claimed items, per-chunk counters).
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

// A two-phase item type.
template <class L0_, class L1_, class S_, class B0_, class B1_, int SHFL_, class MapIn_, class MapOut_,
          Cache COUT_>
struct TwoPhase {
  using L0 = L0_;
  using L1 = L1_;
  using S = S_;
  using MapIn = MapIn_;
  using MapOut = MapOut_;
  static constexpr int E = L0::E;
  static constexpr int TILE = 1 << L0::T_BITS;

  __device__ __forceinline__ static void copy(float* stage, const float* gsrc, uint32_t tid) {
    issue_tile_copy<L0, MapIn, S>(stage, gsrc, tid);
  }
  __device__ __forceinline__ static void phase0(const float* stage, float* work, float (&v)[E],
                                                uint32_t tid) {
    smem_load<L0, S>(stage, v, tid);
    butterflies<L0, B0_, false>(v);
    smem_store<L0, S>(work, v, tid);
  }
  template <bool SCALE, class TOut>
  __device__ __forceinline__ static void phase1(const float* work, TOut* gout, float (&v)[E], uint32_t tid,
                                                float scale) {
    smem_load<L1, S>(work, v, tid);
    butterflies<L1, B1_, false>(v);
    if constexpr (SHFL_ >= 0) shfl_butterfly<L1, SHFL_, false>(v, tid);
    store_global<L1, MapOut, SCALE, COUT_>(gout, v, tid, scale);
  }
};

// ---------------------------------------------------------------------------
// K1P: f32 m = 12 (cfg2) with the PlanF32M12 layouts, pipelined.
// ---------------------------------------------------------------------------
struct PipeF32M12 {
  static constexpr int M = 12;
  static constexpr int NT = 64;
  static constexpr int STAGES = 2;
  static constexpr int MIN_BLOCKS = 3;
  using Item = TwoPhase<PlanF32M12::L0, PlanF32M12::L1, PlanF32M12::S, BL<0, 1, 8, 9, 10, 11>,
                        BL<2, 3, 4, 5, 6, 7>, -1, IdMap, RevMap<12>, Cache::kStream>;
  static constexpr int TILE = Item::TILE;
  static constexpr int SMEM_BYTES = (STAGES + 2) * TILE * 4;
};

// Static round-robin schedule over independent row tiles.
template <class P, bool SCALE>
__global__ void __launch_bounds__(P::NT, P::MIN_BLOCKS) k1p_kernel(const float* __restrict__ in,
                                                                   float* __restrict__ out,
                                                                   uint64_t ntiles, float scale) {
  using Item = typename P::Item;
  constexpr int S = P::STAGES;
  constexpr int TILE = P::TILE;
  extern __shared__ __align__(128) float smem_f[];
  float* stages = smem_f;
  float* work = smem_f + S * TILE;
  const uint32_t tid = threadIdx.x;
  const uint64_t stride = gridDim.x;
  uint64_t item = blockIdx.x;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const uint64_t it = item + (uint64_t)s * stride;
    if (it < ntiles) Item::copy(stages + s * TILE, in + (it << P::M), tid);
    cp_async_commit();
  }
  float v[Item::E];
  for (uint32_t k = 0; item < ntiles; ++k, item += stride) {
    const int s = k % S;
    cp_async_wait<S - 1>();
    __syncthreads();
    Item::phase0(stages + s * TILE, work + (k & 1) * TILE, v, tid);
    __syncthreads();
    const uint64_t nxt = item + (uint64_t)S * stride;
    if (nxt < ntiles) Item::copy(stages + s * TILE, in + (nxt << P::M), tid);
    cp_async_commit();
    Item::template phase1<SCALE>(work + (k & 1) * TILE, out + (item << P::M), v, tid, scale);
  }
  cp_async_wait<0>();
}

}  // namespace chwb
