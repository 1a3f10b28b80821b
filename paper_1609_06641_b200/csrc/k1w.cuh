// k1w.cuh — K1W: warp-per-row single-pass kernel for f32 m = 12 (BASELINE
// cfg2), fed by the TMA engine.
//
// A row (4096 floats, 16 KiB) is one tile of ONE warp: 32 threads x 128
// values.  Two register layouts cover the 12 butterfly levels with two
// register bits to spare (7 + 5), and the spare pair (j10, j11 — butterflied
// in the first layout, carried in the second) is the 16-byte vector of the
// transpose, so all four tile accesses are 16-byte vectors:
//   stage (natural order) --LDS.128--> L0 [regs j0 j1 j7..j11]: 7 levels
//   --STS.128--> the same stage, swizzled, --LDS.128--> L1 [regs j11 j10
//   j2..j6]: 5 levels, scale --STG.128--> dyadic order (out bits 0, 1 = j11,
//   j10; 4 runs of 128 bytes per warp instruction).
// The transpose stays inside the warp (__syncwarp only), so the compute warps
// share nothing but the producer: no named barriers, no work tile, and about
// 8 instructions per element instead of K1T's 14 (64-value threads, scalar
// second load and scalar stores) — the same HBM traffic for less issue and
// less power under the sustained, power-capped bench.
//
// One persistent CTA per SM: NW compute warps + one producer warp; the CTA's
// u-th row goes to warp u % NW through stage u % (2 NW) of the ring (a stage
// always belongs to the same warp, so every parity wait is on its current
// phase).  Layouts and swizzle are conflict-free in tools/plan_check.py.
#pragma once

#include "k1t.cuh"

// Cache-policy experiments (A/B builds): bit 0 = default-policy output stores
// instead of st.global.cs, bit 1 = evict_normal input loads instead of
// evict_first.
#ifndef CHW_K1W_POL
#define CHW_K1W_POL 0
#endif

namespace chwb {

struct WarpRowF32M12 {
  static constexpr int M = 12;
  static constexpr int TILE = 1 << 12;
  static constexpr int NW = 7;        // compute warps per CTA
  static constexpr int S = 2 * NW;    // 16 KiB stages (224 KiB)
  using L0 = Layout<BL<0, 1, 7, 8, 9, 10, 11>, BL<2, 3, 4, 5, 6>>;
  using B0 = BL<0, 1, 7, 8, 9, 10, 11>;
  // the transpose in the numbering u0.. = j10, j11, j2..j9, j0, j1 (tile bit k
  // at shared-memory address bit k): the same registers, vectors on u0, u1
  using L0u = Layout<BL<10, 11, 7, 8, 9, 0, 1>, BL<2, 3, 4, 5, 6>>;
  using L1u = Layout<BL<1, 0, 2, 3, 4, 5, 6>, BL<7, 8, 9, 10, 11>>;
  using Su = Swz<7, 2, 8, 3, 9, 4>;
  using L1 = Layout<BL<11, 10, 2, 3, 4, 5, 6>, BL<7, 8, 9, 0, 1>>;  // L1u in j numbering
  using B1 = BL<2, 3, 4, 5, 6>;
  static constexpr int E = L0::E;
  static_assert(L0::NT == 32 && L1::NT == 32 && L0u::NT == 32 && L1u::NT == 32 && E == 128, "one warp per row");
};

template <bool SCALE>
__global__ void __launch_bounds__((WarpRowF32M12::NW + 1) * 32, 1)
    k1w_kernel(const float* __restrict__ in, float* __restrict__ out, uint64_t rows, float scale) {
  using P = WarpRowF32M12;
  constexpr int TILE = P::TILE;
  constexpr uint32_t TBYTES = TILE * 4;
  constexpr int S = P::S, NW = P::NW;
  extern __shared__ __align__(128) float smem_k1w[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const uint32_t tid = threadIdx.x;
  const uint64_t G = gridDim.x, c = blockIdx.x;
  if (c >= rows) return;
  const uint64_t nu = (rows - 1 - c) / G + 1;  // rows of this CTA
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init_cta(&full[s], 1);
      mbar_init_cta(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t w = tid >> 5, lane = tid & 31u;
  if (w == (uint32_t)NW) {  // producer warp
    if (lane != 0) return;
    const uint64_t pol = (CHW_K1W_POL & 2) ? l2_evict_normal_policy() : l2_evict_first_policy();
    for (uint64_t u = 0; u < nu; ++u) {
      const int st = (int)(u % S);
      if (u >= (uint64_t)S) mbar_wait_cta(&empty[st], (uint32_t)((u / S) - 1) & 1u);
      mbar_expect_tx_cta(&full[st], TBYTES);
      bulk_g2s(smem_k1w + st * TILE, in + ((c + u * G) << 12), TBYTES, &full[st], pol);
    }
    return;
  }
  float v[P::E];
  for (uint64_t u = w; u < nu; u += NW) {
    const int st = (int)(u % S);
    float* stage = smem_k1w + st * TILE;
    mbar_wait_cta(&full[st], (uint32_t)(u / S) & 1u);
    smem_load<P::L0, NoSwz>(stage, v, lane);
    butterflies<P::L0, P::B0, false>(v);
    __syncwarp();  // every lane has read the stage: rewrite it in the transposed addressing
    smem_store<P::L0u, P::Su>(stage, v, lane);
    __syncwarp();
    smem_load<P::L1u, P::Su>(stage, v, lane);
    __syncwarp();  // the stage is read: hand it back to the producer
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    }
    butterflies<P::L1, P::B1, false>(v);
    store_global<P::L1, RevMap<12>, SCALE, (CHW_K1W_POL & 1) ? Cache::kL2 : Cache::kStream>(out + ((c + u * G) << 12), v, lane,
                                                                                             scale);
  }
}

}  // namespace chwb
