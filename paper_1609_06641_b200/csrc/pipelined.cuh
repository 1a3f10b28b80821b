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
// Per item k (stage s = k % S; one work buffer: barrier 1 of item k follows the
// phase-1 reads of item k-1 in every thread):
//   cp.async.wait_group(S-1); bar.sync            (item k landed, ring visible)
//   [publish completion of item k-1]              (dataflow schedules only)
//   L0 <- stage s; butterflies; work <- L0
//   bar.sync                                      (stage s free, work visible)
//   issue cp.async for item k+S into stage s      (or defer: dependency open)
//   L1 <- work; butterflies; global stores
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
  static constexpr int STAGES = 4;      // measured sweep: 4 stages x 2 CTAs/SM best
  static constexpr int MIN_BLOCKS = 2;
  using Item = TwoPhase<PlanF32M12::L0, PlanF32M12::L1, PlanF32M12::S, BL<0, 1, 8, 9, 10, 11>,
                        BL<2, 3, 4, 5, 6, 7>, -1, IdMap, RevMap<12>, Cache::kStream>;
  static constexpr int TILE = Item::TILE;
  static constexpr int SMEM_BYTES = (STAGES + 1) * TILE * 4;
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
    Item::phase0(stages + s * TILE, work, v, tid);
    __syncthreads();
    const uint64_t nxt = item + (uint64_t)S * stride;
    if (nxt < ntiles) Item::copy(stages + s * TILE, in + (nxt << P::M), tid);
    cp_async_commit();
    Item::template phase1<SCALE>(work, out + (item << P::M), v, tid, scale);
  }
  cp_async_wait<0>();
}


// ---------------------------------------------------------------------------
// K5P: the fused two-phase dataflow schedule (fused.cuh) on the pipeline.
// A items (input -> intermediate) always prefetch their input; only their
// stores wait for the slot to be drained.  B items (intermediate -> output)
// prefetch only once their chunk's A tiles are published, else the copy is
// deferred to consume time.  Before any blocking poll a CTA publishes its
// previous item, so every wait points at an earlier, progressing item.
// ---------------------------------------------------------------------------
template <class F>
struct FusedPipe;

template <>
struct FusedPipe<FusedF32M16> {
  using F = FusedF32M16;
  static constexpr int STAGES = 2;
  static constexpr int MIN_BLOCKS = 4;
  using ItemA = TwoPhase<F::A::L0, F::A::L1, F::A::S, BL<0, 1, 6, 7>, BL<2, 3, 4, 5>, -1, IdMap,
                         F::A::MapOut, Cache::kL2>;
  using ItemB = TwoPhase<F::B::L0, F::B::L1, F::B::S, BL<8, 9, 10, 11>, BL<4, 5, 6, 7>, -1, F::B::MapIn,
                         F::B::MapOut, Cache::kStream>;
  static constexpr int TILE = ItemA::TILE;
  static constexpr int SMEM_BYTES = (STAGES + 1) * TILE * 4;
};
template <>
struct FusedPipe<FusedF32M16b> {
  using F = FusedF32M16b;
  static constexpr int STAGES = 2;
  static constexpr int MIN_BLOCKS = 4;
  using ItemA = TwoPhase<F::A::L0, F::A::L1, F::A::S, F::A::B0, F::A::B1, -1, IdMap, F::A::MapOut, Cache::kL2>;
  using ItemB = TwoPhase<F::B::L0, F::B::L1, F::B::S, F::B::B0, F::B::B1, -1, F::B::MapIn, F::B::MapOut,
                         Cache::kStream>;
  static constexpr int TILE = ItemA::TILE;
  static constexpr int SMEM_BYTES = (STAGES + 1) * TILE * 4;
};
template <>
struct FusedPipe<FusedF32M24> {
  using F = FusedF32M24;
  static constexpr int STAGES = 2;
  static constexpr int MIN_BLOCKS = 1;
  using ItemA = TwoPhase<F::A::L0, F::A::L1, F::A::S, BL<0, 1, 9, 10, 11, 12>, BL<2, 3, 4, 5, 6, 7>, 8,
                         IdMap, F::A::MapOut, Cache::kL2>;
  using ItemB = TwoPhase<F::B::L0, F::B::L1, F::B::S, BL<10, 11, 12, 13>, BL<3, 4, 5, 6, 7, 8>, 9,
                         F::B::MapIn, F::B::MapOut, Cache::kStream>;
  static constexpr int TILE = ItemA::TILE;
  static constexpr int SMEM_BYTES = (STAGES + 1) * TILE * 4;
};

struct FusedItem {
  bool valid, is_a;
  uint32_t q, tile;
};

template <class F>
__device__ __forceinline__ FusedItem fused_decode(uint32_t w, const FusedGeom& g) {
  FusedItem it;
  it.valid = decode_work(w, g, it.is_a, it.q, it.tile);
  return it;
}

template <class F, bool SCALE>
__global__ void __launch_bounds__(F::NT, FusedPipe<F>::MIN_BLOCKS)
    fused_p_kernel(const float* __restrict__ in, float* __restrict__ out, float* __restrict__ slots,
                   uint32_t* __restrict__ ctr, FusedGeom g, float scale) {
  using P = FusedPipe<F>;
  using IA = typename P::ItemA;
  using IB = typename P::ItemB;
  static_assert(IA::TILE == IB::TILE && IA::E == IB::E, "A and B tiles must match");
  constexpr int S = P::STAGES;
  constexpr int TILE = P::TILE;
  constexpr uint64_t n = 1ull << F::M;
  extern __shared__ __align__(128) float smem_f[];
  float* stages = smem_f;
  float* work = smem_f + S * TILE;
  __shared__ uint32_t ring[S + 1];
  __shared__ uint32_t issued[S];
  uint32_t* a_done = ctr + 1;
  uint32_t* b_done = ctr + 1 + g.nchunks;
  const uint64_t slot_elems = (uint64_t)g.chunk_rows << F::M;
  const uint32_t tid = threadIdx.x;

  auto src_of = [&](const FusedItem& it) -> const float* {
    const uint32_t rows_q = (it.q == g.nchunks - 1) ? g.rows_last : g.chunk_rows;
    const float* slot = slots + (uint64_t)(it.q % g.nslots) * slot_elems;
    uint32_t row, a, b;
    if (it.is_a) {
      F::a_offsets(it.tile, row, a, b);
      if (row >= rows_q) return nullptr;
      return in + ((uint64_t)it.q * g.chunk_rows + row) * n + a;
    }
    F::b_offsets(it.tile, row, a, b);
    if (row >= rows_q) return nullptr;
    return slot + (uint64_t)row * n + a;
  };
  auto dep_ready = [&](const FusedItem& it) -> bool {  // B items: chunk's A tiles published
    return it.is_a || ld_relaxed_u32(&a_done[it.q]) >= g.nA;
  };
  auto issue = [&](const FusedItem& it, float* stage) {
    const float* src = src_of(it);
    if (!src) return;
    if (it.is_a)
      IA::copy(stage, src, tid);
    else
      IB::copy(stage, src, tid);
  };

  if (tid == 0) {
    for (int i = 0; i <= S; ++i) ring[i] = atomicAdd(ctr, 1u);
    for (int i = 0; i < S; ++i) {
      const FusedItem it = fused_decode<F>(ring[i], g);
      issued[i] = it.valid && dep_ready(it);
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < S; ++s) {
    if (issued[s]) issue(fused_decode<F>(ring[s], g), stages + s * TILE);
    cp_async_commit();
  }
  float v[IA::E];
  FusedItem prev{false, false, 0, 0};
  for (uint32_t k = 0;; ++k) {
    const int s = k % S;
    cp_async_wait<S - 1>();
    __syncthreads();  // barrier 1
    if (tid == 0 && prev.valid) red_release_add(prev.is_a ? &a_done[prev.q] : &b_done[prev.q], 1u);
    const FusedItem it = fused_decode<F>(ring[k % (S + 1)], g);
    if (!it.valid) break;
    float* stage = stages + s * TILE;
    if (!issued[s]) {  // deferred B item: wait for its chunk, then load synchronously
      if (tid == 0) wait_at_least(&a_done[it.q], g.nA);
      __syncthreads();
      issue(it, stage);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
    }
    const uint32_t rows_q = (it.q == g.nchunks - 1) ? g.rows_last : g.chunk_rows;
    uint32_t row, off_a, off_b;
    if (it.is_a)
      F::a_offsets(it.tile, row, off_a, off_b);
    else
      F::b_offsets(it.tile, row, off_a, off_b);
    const bool live = row < rows_q;
    if (live) {
      if (it.is_a)
        IA::phase0(stage, work, v, tid);
      else
        IB::phase0(stage, work, v, tid);
    }
    const FusedItem nx = fused_decode<F>(ring[(k + S) % (S + 1)], g);
    if (tid == 0) {
      issued[s] = nx.valid && dep_ready(nx);
      // A stores into a reused slot wait until the B tiles that drain it are done.
      if (it.is_a && live && it.q >= g.nslots) wait_at_least(&b_done[it.q - g.nslots], g.nB);
    }
    __syncthreads();  // barrier 2
    if (issued[s]) issue(nx, stage);
    cp_async_commit();
    if (tid == 0) ring[k % (S + 1)] = atomicAdd(ctr, 1u);
    if (live) {
      const uint64_t grow = (uint64_t)it.q * g.chunk_rows + row;
      if (it.is_a) {
        float* slot = slots + (uint64_t)(it.q % g.nslots) * slot_elems;
        IA::template phase1<false>(work, slot + (uint64_t)row * n + off_b, v, tid, scale);
      } else {
        IB::template phase1<SCALE>(work, out + grow * n + off_b, v, tid, scale);
      }
    }
    prev = it;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// K4P: one statically scheduled pipelined pass over independent tiles whose
// source/destination offsets come from a geometry functor (phase A or B of a
// two-pass schedule; no cross-CTA dependencies inside a launch).
// ---------------------------------------------------------------------------
template <class Item, class Geo, bool SCALE, int STAGES, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    pass_p_kernel(const float* __restrict__ src, float* __restrict__ dst, uint64_t nitems, float scale) {
  constexpr int TILE = Item::TILE;
  extern __shared__ __align__(128) float smem_pp[];
  float* stages = smem_pp;
  float* work = smem_pp + STAGES * TILE;
  const uint32_t tid = threadIdx.x;
  const uint64_t stride = gridDim.x;
  uint64_t item = blockIdx.x;
#pragma unroll
  for (int s = 0; s < STAGES; ++s) {
    const uint64_t it = item + (uint64_t)s * stride;
    if (it < nitems) Item::copy(stages + s * TILE, src + Geo::src_off(it), tid);
    cp_async_commit();
  }
  float v[Item::E];
  for (uint32_t k = 0; item < nitems; ++k, item += stride) {
    const int s = k % STAGES;
    cp_async_wait<STAGES - 1>();
    __syncthreads();
    Item::phase0(stages + s * TILE, work, v, tid);
    __syncthreads();
    const uint64_t nxt = item + (uint64_t)STAGES * stride;
    if (nxt < nitems) Item::copy(stages + s * TILE, src + Geo::src_off(nxt), tid);
    cp_async_commit();
    Item::template phase1<SCALE>(work, dst + Geo::dst_off(item), v, tid, scale);
  }
  cp_async_wait<0>();
}

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
