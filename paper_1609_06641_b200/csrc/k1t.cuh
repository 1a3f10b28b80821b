// k1t.cuh — K1T: the single-pass tile kernel (K1P's item, pipelined.cuh) fed
// by the TMA engine.  One persistent CTA per SM: a producer thread streams the
// CTA's row tiles (one contiguous bulk copy each) into a ring of S stages with
// per-stage full/empty mbarriers, and NG compute groups of Item::NT threads
// each take every NG-th tile (stage s always belongs to group s mod NG, so
// every parity wait is on the stage's current phase).  Compared with K1P
// (cp.async issued by the compute threads, two CTAs per SM) the loads cost no
// compute-thread instructions and the groups never share a barrier.
#pragma once

#include "rowpipe.cuh"

namespace chwb {

// f32 m = 12 item adapter (K1P's TwoPhase item).
struct ItemF32M12 {
  using T = PipeF32M12::Item;
  using IO = float;
  static constexpr int TILE = T::TILE;
  static constexpr int E = T::E;
  using L0 = T::L0;
  __device__ __forceinline__ static void phase0(const float* stage, float* work, float (&v)[E], uint32_t tid) {
    T::phase0(stage, work, v, tid);
  }
  template <bool SCALE>
  __device__ __forceinline__ static void phase1(const float* work, float* gout, float (&v)[E], uint32_t tid,
                                                float scale) {
    T::template phase1<SCALE>(work, gout, v, tid, scale);
  }
};

// One tile = 2^TB contiguous elements (whole rows).
template <class Item, int TB, int S, int NG, bool SCALE>
__global__ void __launch_bounds__(NG * Item::L0::NT + 32, 1)
    k1t_kernel(const typename Item::IO* __restrict__ in, typename Item::IO* __restrict__ out, uint64_t ntiles,
               float scale) {
  using IO = typename Item::IO;
  static_assert(S % NG == 0, "each stage must belong to one group");
  constexpr int TILE = Item::TILE;
  static_assert(TILE == (1 << TB), "tile size");
  constexpr uint32_t TBYTES = TILE * sizeof(IO);
  constexpr int NT = Item::L0::NT;
  extern __shared__ __align__(128) unsigned char smem_k1t[];
  IO* ring = reinterpret_cast<IO*>(smem_k1t);
  float* works = reinterpret_cast<float*>(smem_k1t + (size_t)S * TBYTES);
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const uint32_t tid = threadIdx.x;
  const uint64_t G = gridDim.x, c = blockIdx.x;
  if (c >= ntiles) return;
  const uint64_t nu = (ntiles - 1 - c) / G + 1;  // tiles of this CTA
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init_cta(&full[s], 1);
      mbar_init_cta(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t warp = tid >> 5;
  if (warp == (uint32_t)(NG * NT / 32)) {  // producer warp
    if ((tid & 31u) != 0) return;
    const uint64_t pol = l2_evict_first_policy();
    for (uint64_t u = 0; u < nu; ++u) {
      const int st = (int)(u % S);
      if (u >= (uint64_t)S) mbar_wait_cta(&empty[st], (uint32_t)((u / S) - 1) & 1u);
      mbar_expect_tx_cta(&full[st], TBYTES);
      bulk_g2s(ring + st * TILE, in + ((c + u * G) << TB), TBYTES, &full[st], pol);
    }
    return;
  }
  const uint32_t g = tid / NT;
  const uint32_t gt = tid % NT;
  float* work = works + g * TILE;
  float v[Item::E];
  for (uint64_t u = g; u < nu; u += NG) {
    const int st = (int)(u % S);
    mbar_wait_cta(&full[st], (uint32_t)(u / S) & 1u);
    Item::phase0(ring + st * TILE, work, v, gt);
    named_bar(1 + g, NT);
    if (gt == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    Item::template phase1<SCALE>(work, out + ((c + u * G) << TB), v, gt, scale);
    named_bar(1 + g, NT);  // work tile free for the next phase0
  }
}


}  // namespace chwb
