// rowpipe2.cuh — K11: the per-CTA row pipeline for f32 m = 16 (BASELINE cfg4)
// with 128-value threads.
//
// Same schedule class as K6 (rowpipe.cuh): every persistent CTA owns whole
// rows and sends each through ONE private, L2-resident workspace row between
// its two phases, with alternating workspace layouts so that A(i+1, k)
// overwrites exactly what B(i, k) read.  K6 is bound by the LSU pipe (72 % at
// 1.9 GHz: 32-value threads, six shared-memory passes per element, scalar
// second loads) and therefore by the power-capped SM clock under the bench
// soak.  K11 halves the issued instructions and cuts the shared-memory passes
// to four, all 16-byte accesses:
//
//   A(i, ka): the contiguous quarter (j15, j14) = ka of the row -> ONE register
//     layout (registers j0 j1 j9..j13), 7 butterfly levels, no transpose ->
//     workspace, 512 contiguous bytes per warp store.
//   B(i, kb): the workspace tile (j11, j10) = kb (one 64 KiB bulk copy in
//     layout P, four 16 KiB copies in layout Q) -> registers t0 t1 t6 t10..t13:
//     3 levels -> in-place transpose whose 16-byte vector is the register pair
//     (t12, t13) = (j14, j15) common to both layouts -> registers t13 t12 t2..t5
//     t0: 6 levels, scale, dyadic stores in whole 64-byte runs.
//
// Workspace row (2^16 floats), layout P: addr = [j0 j1 | j2..j6 | j9 j12 j13 |
// j7 j8 | j14 j15 | j10 j11]; layout Q swaps the two top pairs.  B tile bit t_k
// = address bit k for k < 12, (t12, t13) = (j14, j15).  All layouts and the
// swizzle are conflict-free in tools/plan_check.py (tests/test_plans.py).
#pragma once

#include "rowpipe.cuh"

#ifndef CHW_R2_EARLYWAIT
#define CHW_R2_EARLYWAIT 0
#endif

namespace chwb {

struct RowPipe2F32M16 {
  static constexpr int M = 16;
  static constexpr int TILE = 1 << 14;
  static constexpr int NT = 128;
  // A tile bit k = j bit k
  using AL = Layout<BL<0, 1, 9, 10, 11, 12, 13>, BL<2, 3, 4, 5, 6, 7, 8>>;
  using AB = BL<0, 1, 9, 10, 11, 12, 13>;
  using AOutP = ListMap<0, 1, 2, 3, 4, 5, 6, 10, 11, 7, 14, 15, 8, 9>;  // tile base ka << 12
  using AOutQ = ListMap<0, 1, 2, 3, 4, 5, 6, 10, 11, 7, 12, 13, 8, 9>;  // tile base ka << 14
  // B tile bits t0..t13 = j0 j1 j2 j3 j4 j5 j6 j9 j12 j13 j7 j8 j14 j15
  using BL0 = Layout<BL<0, 1, 6, 10, 11, 12, 13>, BL<2, 3, 4, 5, 7, 8, 9>>;
  using BL1 = Layout<BL<13, 12, 2, 3, 4, 5, 0>, BL<8, 9, 7, 1, 6, 10, 11>>;
  using BB0 = BL<6, 10, 11>;
  using BB1 = BL<13, 12, 2, 3, 4, 5>;
  // the transpose in the numbering u = t12 t13 t2 t3 t4 t8 t9 t7 t0 t1 t5 t6 t10 t11
  using BL0u = Layout<BL<8, 9, 11, 12, 13, 0, 1>, BL<2, 3, 4, 10, 7, 5, 6>>;
  using BL1u = Layout<BL<1, 0, 2, 3, 4, 10, 8>, BL<5, 6, 7, 9, 11, 12, 13>>;
  using BS = Swz<5, 2, 6, 3, 7, 4>;
  // dyadic output position (bit q = j bit 15 - q) of B tile bit t_k; the tile
  // index kb = j10 + 2 j11 supplies out bits 5 and 4
  using BOut = ListMap<15, 14, 13, 12, 11, 10, 9, 6, 3, 2, 8, 7, 1, 0>;
  static constexpr int E = AL::E;
  static_assert(AL::NT == NT && BL0::NT == NT && BL1::NT == NT && BL0u::NT == NT && BL1u::NT == NT && E == 128,
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
__global__ void __launch_bounds__(2 * RowPipe2F32M16::NT, 1)
    rowpipe2_m16_kernel(const float* __restrict__ in, float* __restrict__ out, float* __restrict__ ws, uint64_t rows,
                        float scale) {
  using P = RowPipe2F32M16;
  constexpr int TILE = P::TILE;
  constexpr uint32_t TB = TILE * 4;
  constexpr int NT = P::NT;
  // One A stage is enough: A reads its stage once (no transpose), so the
  // refill is issued right after the load and flies during the butterflies and
  // the workspace store.  B transposes in place and holds its stage for the
  // whole tile, so it gets two and always has the next tile in flight.
  constexpr int SA = 1, SB = 2;
  extern __shared__ __align__(128) float smem_r2[];
  float* ringA = smem_r2;
  float* ringB = smem_r2 + SA * TILE;
  __shared__ __align__(8) uint64_t fullA[SA], fullB[SB], regionfree[4], rowstored;
  const uint32_t tid = threadIdx.x;
  const uint64_t G = gridDim.x, c = blockIdx.x;
  if (c >= rows) return;
  const uint32_t R = (uint32_t)((rows - 1 - c) / G + 1);  // rows of this CTA: c, c + G, ...
  const uint32_t total = 4u * R;                           // A items (and B items)
  float* wsc = ws + (c << 16);                             // the CTA's workspace row
  if (tid == 0) {
    for (int s = 0; s < SA; ++s) mbar_init_cta(&fullA[s], 1);
    for (int s = 0; s < SB; ++s) mbar_init_cta(&fullB[s], 1);
    for (int k = 0; k < 4; ++k) mbar_init_cta(&regionfree[k], 1);
    mbar_init_cta(&rowstored, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float v[P::E];
  if (tid < (uint32_t)NT) {  // ---- A group
    const uint32_t gt = tid;
    auto bar = [] { named_bar(1, NT); };
    uint64_t pol = 0;
    auto issue = [&](uint32_t u) {  // quarter u % 4 of the CTA's (u / 4)-th row -> stage u % SA (free)
      const int st = (int)(u % SA);
      mbar_expect_tx_cta(&fullA[st], TB);
      bulk_g2s(ringA + st * TILE, in + ((c + (uint64_t)(u >> 2) * G) << 16) + ((uint64_t)(u & 3u) << 14), TB,
               &fullA[st], pol);
    };
    if (gt == 0) {
      pol = l2_evict_first_policy();
      for (uint32_t u = 0; u < (uint32_t)SA && u < total; ++u) issue(u);
    }
    for (uint32_t u = 0; u < total; ++u) {
      const uint32_t i = u >> 2, ka = u & 3u;
      const int st = (int)(u % SA);
      mbar_wait_cta(&fullA[st], (u / SA) & 1u);
      smem_load<P::AL, NoSwz>(ringA + st * TILE, v, gt);
      bar();  // every thread has read the stage: refill it
      if (gt == 0 && u + SA < total) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(u + SA);
      }
#if CHW_R2_EARLYWAIT
      // wait before the butterflies: no barrier between the last level and the
      // stores, so ptxas can spread the 32 stores over the arithmetic
      if (i >= 1) mbar_wait_cta(&regionfree[ka], (i - 1) & 1u);  // B(i-1, ka) has been read
      butterflies<P::AL, P::AB, false>(v);
#else
      butterflies<P::AL, P::AB, false>(v);
      if (i >= 1) mbar_wait_cta(&regionfree[ka], (i - 1) & 1u);  // B(i-1, ka) has been read
#endif
      if (i & 1u)
        store_global<P::AL, P::AOutQ, false, Cache::kL2Last>(wsc + (ka << 14), v, gt, 1.0f);
      else
        store_global<P::AL, P::AOutP, false, Cache::kL2Last>(wsc + (ka << 12), v, gt, 1.0f);
      if (ka == 3u) {  // the row is in the workspace: B reads it with bulk copies
        asm volatile("fence.proxy.async.global;" ::: "memory");
        bar();
        if (gt == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&rowstored)) : "memory");
      }
    }
  } else {  // ---- B group
    const uint32_t gt = tid - NT;
    auto bar = [] { named_bar(2, NT); };
    uint64_t pol = 0;
    // Workspace tile u % 4 of the CTA's (u / 4)-th row -> the (free) B stage.
    // A row's first tile needs the whole row stored: with wait = false the
    // call returns false instead of blocking.
    auto issue = [&](uint32_t u, bool wait) -> bool {
      const uint32_t i = u >> 2, kb = u & 3u;
      if (kb == 0u) {
        if (!mbar_test_cta(&rowstored, i & 1u)) {
          if (!wait) return false;
          mbar_wait_cta(&rowstored, i & 1u);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      const int st = (int)(u % SB);
      float* stage = ringB + st * TILE;
      mbar_expect_tx_cta(&fullB[st], TB);
      if (i & 1u) {  // layout Q: four 16 KiB pieces, one per A tile
#pragma unroll
        for (uint32_t ka = 0; ka < 4u; ++ka)
          bulk_g2s(stage + (ka << 12), wsc + (ka << 14) + (kb << 12), TB / 4, &fullB[st], pol);
      } else {
        bulk_g2s(stage, wsc + (kb << 14), TB, &fullB[st], pol);
      }
      return true;
    };
    uint32_t next = 0;  // thread 0: the next tile to issue (tiles < next are in flight or done)
    if (gt == 0) pol = l2_evict_normal_policy();
    for (uint32_t u = 0; u < total; ++u) {
      const uint32_t i = u >> 2, kb = u & 3u;
      const int st = (int)(u % SB);
      float* stageB = ringB + st * TILE;
      if (gt == 0) {
        if (next == u) {  // not issued yet (it waited for its row): now it must be
          issue(u, true);
          ++next;
        }
        // the other stage is free (tile u - 1 is done with it)
        if (next == u + 1 && next < total && issue(next, false)) ++next;
      }
      mbar_wait_cta(&fullB[st], (u / SB) & 1u);
      // B(i, kb)'s workspace bytes are in shared memory: A(i+1, kb) may overwrite them.
      if (gt == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&regionfree[kb])) : "memory");
      smem_load<P::BL0, NoSwz>(stageB, v, gt);
      butterflies<P::BL0, P::BB0, false>(v);
      bar();  // every thread has read the stage: transpose in place
      smem_store<P::BL0u, P::BS>(stageB, v, gt);
      bar();
      smem_load<P::BL1u, P::BS>(stageB, v, gt);
      bar();  // this stage is free: tile u + 2 goes there (tile u + 1 first, if it is still waiting)
      if (gt == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        while (next <= u + 2 && next < total && issue(next, false)) ++next;
      }
      butterflies<P::BL1, P::BB1, false>(v);
      const uint32_t outer = ((kb & 1u) << 5) | ((kb >> 1) << 4);
      store_global<P::BL1, P::BOut, SCALE, Cache::kStream>(out + ((c + (uint64_t)i * G) << 16), v, gt, scale, outer);
    }
  }
}

}  // namespace chwb
