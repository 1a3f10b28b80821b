// warpspec.cuh — warp-specialized pipelined tile kernel (K5W).
//
// CTA = NT/32 compute warps + 1 scheduler warp.
//   scheduler warp: walks this CTA's items (static round-robin over the global
//     item order), waits until the stage's previous item is finished
//     (mbarrier done[s]), publishes that item's completion to the other CTAs
//     (red.release.gpu), resolves the new item's dependency (relaxed polls on
//     per-chunk counters), writes the item id into the stage's metadata slot and
//     gathers the input tile into stage s with 16-byte cp.async whose completion
//     arrives on mbarrier full[s].
//   compute warps: wait full[s], run the two-phase tile (stage -> registers ->
//     swizzled transpose buffer -> registers -> global), arrive on done[s].
// Compute warps never touch the schedule; the scheduler never blocks them
// except when a stage's data is not there yet.
//
// Deadlock freedom: dependencies only point at earlier items.  Before the
// scheduler blocks on a dependency it drains and publishes every item its own
// CTA has in flight, so the globally earliest unfinished item can always run
// (all CTAs are co-resident: the grid is sized from the occupancy calculator).
#pragma once

#include "pipelined.cuh"

namespace chwb {

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// Arrive on `bar` once all of this thread's prior cp.async copies have landed.
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Warp-specialized fused spec: same item types as FusedPipe, more stages.
template <class F>
struct FusedWS;
template <>
struct FusedWS<FusedF32M16> {
  using Base = FusedPipe<FusedF32M16>;
  using ItemA = Base::ItemA;
  using ItemB = Base::ItemB;
  static constexpr int STAGES = 3;
  static constexpr int MIN_BLOCKS = 3;
  static constexpr int TILE = Base::TILE;
  static constexpr int SMEM_BYTES = (STAGES + 1) * TILE * 4;
};
template <>
struct FusedWS<FusedF32M16b> {
  using Base = FusedPipe<FusedF32M16b>;
  using ItemA = Base::ItemA;
  using ItemB = Base::ItemB;
  static constexpr int STAGES = 2;
  static constexpr int MIN_BLOCKS = 4;
  static constexpr int TILE = Base::TILE;
  static constexpr int SMEM_BYTES = (STAGES + 1) * TILE * 4;
};
template <>
struct FusedWS<FusedF32M24> {
  using Base = FusedPipe<FusedF32M24>;
  using ItemA = Base::ItemA;
  using ItemB = Base::ItemB;
  static constexpr int STAGES = 2;
  static constexpr int MIN_BLOCKS = 1;
  static constexpr int TILE = Base::TILE;
  static constexpr int SMEM_BYTES = (STAGES + 1) * TILE * 4;
};

template <class F, bool SCALE>
__global__ void __launch_bounds__(F::NT + 32, FusedWS<F>::MIN_BLOCKS)
    fused_ws_kernel(const float* __restrict__ in, float* __restrict__ out, float* __restrict__ slots,
                    uint32_t* __restrict__ ctr, FusedGeom g, float scale) {
  using P = FusedWS<F>;
  using IA = typename P::ItemA;
  using IB = typename P::ItemB;
  constexpr int S = P::STAGES;
  constexpr int TILE = P::TILE;
  constexpr int NT = F::NT;
  constexpr uint64_t n = 1ull << F::M;
  extern __shared__ __align__(128) float smem_f[];
  float* stages = smem_f;
  float* work = smem_f + S * TILE;
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(8) uint64_t done[S];
  __shared__ uint32_t meta[S];
  uint32_t* a_done = ctr + 1;
  uint32_t* b_done = ctr + 1 + g.nchunks;
  const uint64_t slot_elems = (uint64_t)g.chunk_rows << F::M;
  const uint32_t tid = threadIdx.x;
  const uint32_t total = g.nchunks * (g.nA + g.nB);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 33);  // 32 lanes' cp.async completions + lane 0's release arrive
      mbar_init(&done[s], NT);  // every compute thread
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto item_geom = [&](uint32_t w, FusedItem& it, uint32_t& row, uint32_t& oa, uint32_t& ob) -> bool {
    it = fused_decode<F>(w, g);
    if (!it.valid) return false;
    if (it.is_a)
      F::a_offsets(it.tile, row, oa, ob);
    else
      F::b_offsets(it.tile, row, oa, ob);
    const uint32_t rows_q = (it.q == g.nchunks - 1) ? g.rows_last : g.chunk_rows;
    return row < rows_q;
  };

  if (tid >= NT) {
    // ------------------------------ scheduler warp ------------------------------
    const uint32_t lane = tid - NT;
    uint32_t pend_w[S];
    bool pend[S];
#pragma unroll
    for (int s = 0; s < S; ++s) pend[s] = false;
    auto publish = [&](uint32_t w) {
      if (lane == 0) {
        const FusedItem it = fused_decode<F>(w, g);
        red_release_add(it.is_a ? &a_done[it.q] : &b_done[it.q], 1u);
      }
    };
    // Wait for and publish every item still in flight (before blocking on a dependency).
    auto drain = [&](uint32_t i_now) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (pend[s]) {
          // the in-flight item in stage s was issued at local index i with i % S == s
          uint32_t i = i_now - S + ((s - (int)(i_now % S) + S) % S);
          mbar_wait(&done[s], (i / S) & 1u);
          publish(pend_w[s]);
          pend[s] = false;
        }
      }
    };
    uint32_t i = 0;
    for (uint32_t w = blockIdx.x; w < total; w += gridDim.x, ++i) {
      const int s = i % S;
      if (pend[s]) {  // stage reuse: item i-S must be finished
        mbar_wait(&done[s], ((i - S) / S) & 1u);
        publish(pend_w[s]);
        pend[s] = false;
      }
      FusedItem it;
      uint32_t row, oa, ob;
      const bool live = item_geom(w, it, row, oa, ob);
      // Dependencies: B items read the chunk's intermediate (all A tiles of the
      // chunk); A items overwrite a slot the B tiles of chunk q-nslots drain.
      const uint32_t* dep = nullptr;
      uint32_t target = 0;
      if (!it.is_a) {
        dep = &a_done[it.q];
        target = g.nA;
      } else if (it.q >= g.nslots) {
        dep = &b_done[it.q - g.nslots];
        target = g.nB;
      }
      const bool blocked = dep && ld_relaxed_u32(dep) < target;
      // A items prefetch their input even while their slot is still draining
      // (only the stores need the slot); B items cannot read before the chunk
      // is complete.
      auto issue = [&]() {
        if (!live) return;
        const float* src;
        if (it.is_a)
          src = in + ((uint64_t)it.q * g.chunk_rows + row) * n + oa;
        else
          src = slots + (uint64_t)(it.q % g.nslots) * slot_elems + (uint64_t)row * n + oa;
        float* stage = stages + s * TILE;
#pragma unroll 1
        for (uint32_t vt = lane; vt < (uint32_t)NT; vt += 32) {
          if (it.is_a)
            IA::copy(stage, src, vt);
          else
            IB::copy(stage, src, vt);
        }
      };
      if (it.is_a) issue();
      if (blocked) {
        drain(i);
        if (lane == 0) wait_at_least(dep, target);
        __syncwarp();
      }
      if (!it.is_a) issue();
      cp_async_mbar_arrive(&full[s]);  // fires when this lane's copies have landed
      if (lane == 0) {
        meta[s] = w;
        mbar_arrive(&full[s]);  // release: meta (and the dependency) visible to compute warps
      }
      __syncwarp();
      pend[s] = true;
      pend_w[s] = w;
    }
    // Finish: publish what is still in flight, then tell the compute warps to stop.
    drain(i);
    const int s = i % S;
    cp_async_mbar_arrive(&full[s]);
    if (lane == 0) {
      meta[s] = 0xffffffffu;
      mbar_arrive(&full[s]);
    }
    return;
  }

  // ------------------------------- compute warps -------------------------------
  float v[IA::E];
  for (uint32_t i = 0;; ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1u);
    const uint32_t w = meta[s];
    if (w == 0xffffffffu) break;
    FusedItem it;
    uint32_t row, oa, ob;
    const bool live = item_geom(w, it, row, oa, ob);
    const float* stage = stages + s * TILE;
    named_bar_sync(1, NT);  // previous item's reads of `work` are done
    if (live) {
      if (it.is_a)
        IA::phase0(stage, work, v, tid);
      else
        IB::phase0(stage, work, v, tid);
    }
    named_bar_sync(1, NT);  // `work` complete
    if (live) {
      if (it.is_a) {
        float* slot = slots + (uint64_t)(it.q % g.nslots) * slot_elems;
        IA::template phase1<false>(work, slot + (uint64_t)row * n + ob, v, tid, scale);
      } else {
        const uint64_t grow = (uint64_t)it.q * g.chunk_rows + row;
        IB::template phase1<SCALE>(work, out + grow * n + ob, v, tid, scale);
      }
    }
    mbar_arrive(&done[s]);
  }
}

}  // namespace chwb
