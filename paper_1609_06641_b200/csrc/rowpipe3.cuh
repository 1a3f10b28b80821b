// rowpipe3.cuh — K12: the per-CTA row pipeline for f32 m = 16 (BASELINE cfg4)
// with a one-layout first phase.
//
// Same schedule class as K6 (rowpipe.cuh): every persistent CTA owns whole
// rows and sends each through ONE private, L2-resident workspace row between
// its two phases, with alternating workspace layouts so that A(i+1, k)
// overwrites exactly what B(i, k) read; four 128-thread compute groups (two
// per phase, alternating tiles) like K6.  What changes is the split of the 16
// butterfly levels: 6 + 10 instead of 8 + 8, with 64-value threads.
//
//   A(i, ka): the contiguous eighth (j15 j14 j13) = ka of the row (32 KiB) ->
//     ONE register layout (registers j0 j1 j9..j12), 6 levels, NO transpose ->
//     workspace, 512 contiguous bytes per warp store.
//   B(i, kb): the workspace tile (j11 j10 j9) = kb (one 32 KiB bulk copy in
//     layout P, eight 4 KiB copies in layout Q) -> registers t0 t1 t6 t7 t8 t10:
//     4 levels -> in-place transpose -> registers t12 t11 t2..t5: 6 levels,
//     scale, dyadic stores in whole 64-byte runs.
//
// Four shared-memory passes per element instead of K6's six (K6 is bound by
// the LSU pipe, hence by the power-capped SM clock under the bench soak), and
// A reads its stage once, so one stage per A group is enough and each B group
// gets two (a B stage is held for the whole in-place transpose).
//
// Workspace row (2^16 floats), layout P: addr = [j0 j1 | j2..j6 | j7 j8 | j12 |
// j13 j14 j15 | j9 j10 j11]; layout Q swaps the two top triples.  B tile bit
// t_k = address bit k (k < 10), (t10 t11 t12) = (j13 j14 j15).  Layouts and
// swizzle are conflict-free in tools/plan_check.py (tests/test_plans.py).
#pragma once

#include "rowpipe.cuh"

#ifndef CHW_R3_WS
#define CHW_R3_WS 0  // workspace stores: 0 evict_last hint, 1 plain st.cg
#endif

namespace chwb {

struct RowPipe3F32M16 {
  static constexpr int M = 16;
  static constexpr int TILE = 1 << 13;
  static constexpr int NT = 128;
  // A tile bit k = j bit k (k = 0..12)
  using AL = Layout<BL<0, 1, 9, 10, 11, 12>, BL<2, 3, 4, 5, 6, 7, 8>>;
  using AB = BL<0, 1, 9, 10, 11, 12>;
  using AOutP = ListMap<0, 1, 2, 3, 4, 5, 6, 7, 8, 13, 14, 15, 9>;  // + ka << 10
  using AOutQ = ListMap<0, 1, 2, 3, 4, 5, 6, 7, 8, 10, 11, 12, 9>;  // + ka << 13
  // B tile bits t0..t12 = j0 j1 j2 j3 j4 j5 j6 j7 j8 j12 j13 j14 j15
  using BL0 = Layout<BL<0, 1, 6, 7, 8, 10>, BL<2, 3, 4, 5, 9, 11, 12>>;
  using BL1 = Layout<BL<12, 11, 2, 3, 4, 5>, BL<0, 1, 9, 10, 8, 6, 7>>;
  using BS = Swz<9, 2, 10, 3, 8, 4>;
  using BB0 = BL<6, 7, 8, 10>;
  using BB1 = BL<12, 11, 2, 3, 4, 5>;
  // dyadic output position (bit q = j bit 15 - q) of B tile bit t_k; the tile
  // index kb = j9 + 2 j10 + 4 j11 supplies out bits 6, 5, 4
  using BOut = ListMap<15, 14, 13, 12, 11, 10, 9, 8, 7, 3, 2, 1, 0>;
  static constexpr int E = AL::E;
  static_assert(AL::NT == NT && BL0::NT == NT && BL1::NT == NT && E == 64 && BL0::E == E && BL1::E == E,
                "group shape");
};

__device__ __forceinline__ bool mbar_test_cta(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok)
               : "r"(smem_u32(bar)), "r"(parity)
               : "memory");
  return ok != 0;
}

template <bool SCALE>
__global__ void __launch_bounds__(4 * RowPipe3F32M16::NT, 1)
    rowpipe3_m16_kernel(const float* __restrict__ in, float* __restrict__ out, float* __restrict__ ws, uint64_t rows,
                        float scale) {
  using P = RowPipe3F32M16;
  constexpr int TILE = P::TILE;
  constexpr uint32_t TB = TILE * 4;
  constexpr int NT = P::NT;
  extern __shared__ __align__(128) float smem_r3[];
  // [A group 0 stage][A group 1 stage][B group 0: 2 stages][B group 1: 2 stages]
  __shared__ __align__(8) uint64_t fullA[2], fullB[2][2], regionfree[8], rowstored;
  const uint32_t tid = threadIdx.x;
  const uint64_t G = gridDim.x, c = blockIdx.x;
  if (c >= rows) return;
  const uint32_t R = (uint32_t)((rows - 1 - c) / G + 1);  // rows of this CTA: c, c + G, ...
  const uint32_t total = 8u * R;                           // A items (and B items)
  float* wsc = ws + (c << 16);                             // the CTA's workspace row
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init_cta(&fullA[s], 1);
      mbar_init_cta(&fullB[s][0], 1);
      mbar_init_cta(&fullB[s][1], 1);
    }
    for (int k = 0; k < 8; ++k) mbar_init_cta(&regionfree[k], 1);
    mbar_init_cta(&rowstored, 2);  // both A groups, each after its last tile of the row
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t grp = tid / NT, gt = tid % NT;
  const uint32_t g = grp & 1u;  // the group takes the items u = g, g + 2, ...
  const uint32_t barid = 1 + grp;
  auto bar = [barid] { named_bar(barid, NT); };
  float v[P::E];
  if (grp < 2) {  // ---- A groups
    float* stage = smem_r3 + g * TILE;
    uint64_t pol = 0;
    auto issue = [&](uint32_t u) {  // eighth u % 8 of the CTA's (u / 8)-th row -> the group's (free) stage
      mbar_expect_tx_cta(&fullA[g], TB);
      bulk_g2s(stage, in + ((c + (uint64_t)(u >> 3) * G) << 16) + ((uint64_t)(u & 7u) << 13), TB, &fullA[g], pol);
    };
    if (gt == 0) {
      pol = l2_evict_first_policy();
      if (g < total) issue(g);
    }
    for (uint32_t u = g, n = 0; u < total; u += 2, ++n) {
      const uint32_t i = u >> 3, ka = u & 7u;
      mbar_wait_cta(&fullA[g], n & 1u);
      smem_load<P::AL, NoSwz>(stage, v, gt);
      bar();  // every thread has read the stage: refill it
      if (gt == 0 && u + 2 < total) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(u + 2);
      }
      butterflies<P::AL, P::AB, false>(v);
      if (i >= 1) mbar_wait_cta(&regionfree[ka], (i - 1) & 1u);  // B(i-1, ka) has been read
      if (i & 1u)
        store_global<P::AL, P::AOutQ, false, CHW_R3_WS ? Cache::kL2 : Cache::kL2Last>(wsc + (ka << 13), v, gt, 1.0f);
      else
        store_global<P::AL, P::AOutP, false, CHW_R3_WS ? Cache::kL2 : Cache::kL2Last>(wsc + (ka << 10), v, gt, 1.0f);
      if (ka >= 6u) {  // this group's last tile of the row: B reads the row with bulk copies
        asm volatile("fence.proxy.async.global;" ::: "memory");
        bar();
        if (gt == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&rowstored)) : "memory");
      }
    }
  } else {  // ---- B groups
    float* ring = smem_r3 + (2 + 2 * g) * TILE;
    uint64_t pol = 0;
    // Workspace tile u % 8 of the CTA's (u / 8)-th row -> stage ((u - g) / 2) % 2
    // of the group (free).  The group's first tile of a row needs the whole
    // row stored: with wait = false the call returns false instead of blocking.
    auto issue = [&](uint32_t u, bool wait) -> bool {
      const uint32_t i = u >> 3, kb = u & 7u;
      if (kb == g) {
        if (!mbar_test_cta(&rowstored, i & 1u)) {
          if (!wait) return false;
          mbar_wait_cta(&rowstored, i & 1u);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      const uint32_t st = ((u - g) >> 1) & 1u;
      float* stage = ring + st * TILE;
      mbar_expect_tx_cta(&fullB[g][st], TB);
      if (i & 1u) {  // layout Q: eight 4 KiB pieces, one per A tile
#pragma unroll
        for (uint32_t ka = 0; ka < 8u; ++ka)
          bulk_g2s(stage + (ka << 10), wsc + (ka << 13) + (kb << 10), TB / 8, &fullB[g][st], pol);
      } else {
        bulk_g2s(stage, wsc + (kb << 13), TB, &fullB[g][st], pol);
      }
      return true;
    };
    uint32_t next = g;  // thread 0: the group's next tile to issue
    if (gt == 0) pol = l2_evict_normal_policy();
    for (uint32_t u = g, n = 0; u < total; u += 2, ++n) {
      const uint32_t i = u >> 3, kb = u & 7u;
      const uint32_t st = n & 1u;
      float* stage = ring + st * TILE;
      if (gt == 0) {
        if (next == u) {  // not issued yet (it waited for its row): now it must be
          issue(u, true);
          next += 2;
        }
        // the other stage is free (the group's previous tile is done with it)
        if (next == u + 2 && next < total && issue(next, false)) next += 2;
      }
      mbar_wait_cta(&fullB[g][st], (n >> 1) & 1u);
      // B(i, kb)'s workspace bytes are in shared memory: A(i+1, kb) may overwrite them.
      if (gt == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&regionfree[kb])) : "memory");
      smem_load<P::BL0, NoSwz>(stage, v, gt);
      butterflies<P::BL0, P::BB0, false>(v);
      bar();  // every thread has read the stage: transpose in place
      smem_store<P::BL0, P::BS>(stage, v, gt);
      bar();
      smem_load<P::BL1, P::BS>(stage, v, gt);
      bar();  // this stage is free: the group's tile after next goes there
      if (gt == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        while (next <= u + 4 && next < total && issue(next, false)) next += 2;
      }
      butterflies<P::BL1, P::BB1, false>(v);
      const uint32_t outer = ((kb & 1u) << 6) | (((kb >> 1) & 1u) << 5) | ((kb >> 2) << 4);
      store_global<P::BL1, P::BOut, SCALE, Cache::kStream>(out + ((c + (uint64_t)i * G) << 16), v, gt, scale, outer);
    }
  }
}

}  // namespace chwb
