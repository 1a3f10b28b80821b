// chw_kernels.cuh — kernels and the (dtype, m) -> schedule dispatch.
//
// K1 (single pass, m <= K1MAX): one CTA per tile of whole rows, the entire
//     cascade in registers + shared memory, one HBM read and one HBM write per
//     element.  Tuned plans for BASELINE cfg2 (f32, m=12) and cfg3 (bf16, m=7);
//     GenericTilePlan elsewhere.
// K4 (multi-pass, m > K1MAX): pass 0 butterflies the low bits of contiguous
//     tiles; each later pass butterflies the next group of bits on tiles made of
//     >= 128-byte contiguous runs; the last pass writes dyadic order.
//     Intermediates live in a workspace (fp32 for f32/bf16, f64 for f64).
#pragma once

#include <cstdint>

#include "plans.cuh"

namespace chwb {

// ---------------------------------------------------------------------------
// Per-dtype regime constants.
// ---------------------------------------------------------------------------
template <class T>
struct Regime;
template <>
struct Regime<double> {
  // EB = 5: 32 doubles per thread, so an m = 10 row (BASELINE cfg1) is one warp
  // and two shared-memory transposes (measured 1.8x faster than EB = 4).
  static constexpr int EB = 5, TMIN = 10, K1MAX = 13, TB0 = 12, TBP = 12, CLMIN = 4;
};
template <>
struct Regime<long long> {
  static constexpr int EB = 4, TMIN = 10, K1MAX = 13, TB0 = 12, TBP = 12, CLMIN = 4;
};
template <>
struct Regime<float> {
  static constexpr int EB = 5, TMIN = 11, K1MAX = 14, TB0 = 13, TBP = 13, CLMIN = 5;
};
template <>
struct Regime<__nv_bfloat16> {
  static constexpr int EB = 5, TMIN = 11, K1MAX = 14, TB0 = 13, TBP = 13, CLMIN = 5;
};

// K1 plan selection: tuned plans where BASELINE names a config, generic otherwise.
template <class T, int M>
struct K1Select {
  using R = Regime<T>;
  static constexpr int TB = M > R::TMIN ? M : R::TMIN;
  using Plan = GenericTilePlan<T, M, TB, R::EB>;
  static constexpr bool kTuned = false;
};
template <>
struct K1Select<float, 12> {
  using Plan = PlanF32M12;
  static constexpr bool kTuned = true;
};
template <>
struct K1Select<__nv_bfloat16, 7> {
  using Plan = PlanBF16M7;
  static constexpr bool kTuned = true;
};

// K4 schedule for M > K1MAX.
template <class T, int M>
struct K4Sched {
  using R = Regime<T>;
  static constexpr int GWMAX = R::TBP - R::CLMIN;
  static constexpr int NPASS = 1 + (M - R::TB0 + GWMAX - 1) / GWMAX;
  template <int p>
  struct Pass {
    static constexpr int G0 = p == 0 ? 0 : R::TB0 + (p - 1) * GWMAX;
    static constexpr int GW = p == 0 ? R::TB0 : ((M - G0) < GWMAX ? (M - G0) : GWMAX);
    static constexpr int CL = p == 0 ? 0 : R::TBP - GW;
    using Plan = MultiPass<T, M, CL, G0, GW, p == 0, p == NPASS - 1, R::EB>;
    static constexpr int TILE_BITS = p == 0 ? R::TB0 : R::TBP;
  };
};

// ---------------------------------------------------------------------------
// Kernels.
// ---------------------------------------------------------------------------
template <class Plan, Scaling SC, bool PRED>
__global__ void __launch_bounds__(Plan::NT) k1_kernel(const typename Plan::IO* __restrict__ in,
                                                      typename Plan::IO* __restrict__ out,
                                                      uint64_t tile0,
                                                      typename IoTraits<typename Plan::IO>::C scale,
                                                      uint32_t limit) {
  using C = typename IoTraits<typename Plan::IO>::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint64_t off = (tile0 + blockIdx.x) << Plan::kTB;
  Plan::template run<PRED, SC>(in + off, out + off, reinterpret_cast<C*>(smem_raw), scale, limit);
}

template <class MP, Scaling SC, bool SCALE_OUT>
__global__ void __launch_bounds__(MP::NT) pass_kernel(const typename MP::TIn* __restrict__ in,
                                                      typename MP::TOut* __restrict__ out,
                                                      typename MP::W scale) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t bin, bout;
  MP::bases(blockIdx.x, bin, bout);
  MP::Pass::template run<false, SC, SCALE_OUT>(in + bin, out + bout,
                                               reinterpret_cast<typename MP::W*>(smem_raw), scale, 0);
}

}  // namespace chwb
