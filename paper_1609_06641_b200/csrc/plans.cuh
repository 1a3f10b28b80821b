// plans.cuh — per-regime tile plans for the CHW kernels.
//
// A plan fixes, for one (dtype, m), the tile shape, the sequence of layouts and
// where the butterflies happen.  The tuned plans below were chosen so that every
// shared-memory access is bank-conflict free, every global load is a coalesced
// 16-byte vector and every global store writes whole 32-byte sectors (see
// tools/plan_check.py for the bank/sector analysis).  The generic plan covers
// every other m with the same engine (correct for all m; tuned for none).
#pragma once

#include <type_traits>

#include "engine.cuh"

namespace chwb {

enum class Scaling : int {
  kPerStage = 0,  // f64 Orthonormal: 1/sqrt2 in every butterfly (bit-exact)
  kDeferred = 1,  // f32/bf16 Orthonormal: one multiply by 2^(-m/2) at the store
  kNone = 2,      // Unnormalized
};

// ---------------------------------------------------------------------------
// Generated bit lists for the generic plans.
// ---------------------------------------------------------------------------
// Load layout registers: element bits [0, V) (one 16-byte vector) plus the top
// EB-V tile bits; the middle bits go to threads, so lanes walk consecutive
// vectors and every warp load is one contiguous 512-byte run.
template <int TB, int EB, int V>
struct L0Regs {
  static constexpr int N = EB;
  CHW_HD static constexpr int at(int k) { return k < V ? k : TB - EB + k; }
};
// Group registers: tile bits [G0, G0+GN) then filler bits taken from the top of
// the tile (descending), skipping the group.
template <int TB, int EB, int G0, int GN>
struct GrpRegs {
  static constexpr int N = EB;
  CHW_HD static constexpr int at(int k) {
    if (k < GN) return G0 + k;
    int need = k - GN;
    for (int b = TB - 1; b >= 0; --b) {
      if (b >= G0 && b < G0 + GN) continue;
      if (need == 0) return b;
      --need;
    }
    return -1;
  }
};
// Thread bits: the tile bits not held by registers, ascending.
template <class Reg, int TB>
struct ThrOf {
  static constexpr int N = TB - Reg::N;
  CHW_HD static constexpr int at(int k) {
    int need = k;
    for (int b = 0; b < TB; ++b) {
      if (find<Reg>(b) >= 0) continue;
      if (need == 0) return b;
      --need;
    }
    return -1;
  }
};
template <int A, int N_>
struct Range {
  static constexpr int N = N_;
  CHW_HD static constexpr int at(int k) { return A + k; }
};

// Bank-spreading swizzle for the generic plans: XOR tile bits [EB, EB+5) into
// word bits [0, 5).
template <int EB>
using GenSwz = Swz<EB, 0, EB + 1, 1, EB + 2, 2, EB + 3, 3, EB + 4, 4>;

template <class C, Scaling S>
struct ScaleTag {
  static constexpr bool kPerStage = (S == Scaling::kPerStage);
  static constexpr bool kDeferred = (S == Scaling::kDeferred);
};

// ---------------------------------------------------------------------------
// Position maps for multi-pass tiles (K4).  A pass tile holds the CL lowest
// element bits (kept contiguous so every global access is a >= 128-byte run)
// plus the GW bits [G0, G0+GW) the pass butterflies.
// ---------------------------------------------------------------------------
template <int CL, int G0>
struct PassMap {
  CHW_HD static constexpr int pos(int k) { return k < CL ? k : G0 + (k - CL); }
};
template <int M, int CL, int G0>
struct RevPassMap {
  CHW_HD static constexpr int pos(int k) {
    const int p = PassMap<CL, G0>::pos(k);
    return p < M ? M - 1 - p : p;
  }
};

__device__ __forceinline__ uint32_t rev_bits(uint32_t x, int m) {
  return m == 0 ? 0u : (__brev(x) >> (32 - m));
}

// ---------------------------------------------------------------------------
// Generic tile pass.  Tile = 2^TB elements; tile-local bit k sits at element
// offset MapIn::pos(k) on input and MapOut::pos(k) on output.  Butterflies act
// on tile bits [B0, B0+BN) in increasing order, EB bits per shared-memory round
// trip, so the f64 path keeps the reference's op order exactly.
// ---------------------------------------------------------------------------
template <class TIn, class TOut, class MapIn, class MapOut, int TB, int EB, int B0, int BN>
struct TilePass {
  using IN = TIn;
  using OUT = TOut;
  using C = typename IoTraits<TIn>::C;
  static_assert(std::is_same<C, typename IoTraits<TOut>::C>::value, "compute type mismatch");
  static constexpr int kTB = TB;
  static constexpr int V = IoTraits<TIn>::VMAX < EB ? IoTraits<TIn>::VMAX : EB;
  using L0 = Layout<L0Regs<TB, EB, V>, ThrOf<L0Regs<TB, EB, V>, TB>>;
  static constexpr int NT = L0::NT;
  static constexpr int SMEM_BYTES = (1 << TB) * (int)sizeof(C);
  static constexpr int P = (BN + EB - 1) / EB;  // shared-memory round trips
  using S = GenSwz<EB>;

  template <int p>
  struct G {
    static constexpr int G0 = B0 + p * EB;
    static constexpr int GN = (B0 + BN - G0) < EB ? (B0 + BN - G0) : EB;
    using Reg = GrpRegs<TB, EB, G0, GN>;
    using L = Layout<Reg, ThrOf<Reg, TB>>;
    using Bits = Range<G0, GN>;
  };

  template <int p, Scaling SC>
  __device__ __forceinline__ static void group_step(C (&v)[1 << EB], C* sm, uint32_t tid) {
    using Prev = typename G<p - 1>::L;
    using Cur = typename G<p>::L;
    __syncthreads();
    smem_store<Prev, S>(sm, v, tid);
    __syncthreads();
    smem_load<Cur, S>(sm, v, tid);
    butterflies<Cur, typename G<p>::Bits, SC == Scaling::kPerStage>(v);
    if constexpr (p + 1 < P) group_step<p + 1, SC>(v, sm, tid);
  }

  // SC_OUT: whether this pass applies the deferred scale (last pass only).
  template <bool PRED, Scaling SC, bool SCALE_OUT>
  __device__ __forceinline__ static void run(const TIn* __restrict__ in, TOut* __restrict__ out,
                                             C* sm, C scale, uint32_t limit) {
    const uint32_t tid = threadIdx.x;
    C v[1 << EB];
    if constexpr (PRED)
      load_global_pred<L0, MapIn>(in, v, tid, limit);
    else
      load_global<L0, MapIn>(in, v, tid);
    if constexpr (P == 0) {
      if constexpr (PRED)
        store_global_pred<L0, MapOut, SCALE_OUT>(out, v, tid, scale, limit);
      else
        store_global<L0, MapOut, SCALE_OUT>(out, v, tid, scale);
    } else {
      using L0G = typename G<0>::L;
      smem_store<L0, S>(sm, v, tid);
      __syncthreads();
      smem_load<L0G, S>(sm, v, tid);
      butterflies<L0G, typename G<0>::Bits, SC == Scaling::kPerStage>(v);
      if constexpr (P > 1) group_step<1, SC>(v, sm, tid);
      using LL = typename G<P - 1>::L;
      if constexpr (PRED)
        store_global_pred<LL, MapOut, SCALE_OUT>(out, v, tid, scale, limit);
      else
        store_global<LL, MapOut, SCALE_OUT>(out, v, tid, scale);
    }
  }
};

// Whole rows per tile (K1 generic): 2^(TB-M) rows of 2^M elements.  MapOut
// RevMap<M> stores dyadic order; IdMap stores natural order (SURVEY §8 f2:
// the order folded into the store addresses, no extra pass).
template <class T, int M, int TB, int EB, class MapOut = RevMap<M>>
struct GenericTilePlan : TilePass<T, T, IdMap, MapOut, TB, EB, 0, M> {
  using Base = TilePass<T, T, IdMap, MapOut, TB, EB, 0, M>;
  using IO = T;
  static constexpr int kM = M;
  template <bool PRED, Scaling SC>
  __device__ __forceinline__ static void run(const T* __restrict__ in, T* __restrict__ out,
                                             typename Base::C* sm, typename Base::C scale,
                                             uint32_t limit) {
    Base::template run<PRED, SC, SC == Scaling::kDeferred>(in, out, sm, scale, limit);
  }
};

// One pass of the multi-pass (K4) schedule for rows of 2^M elements.
//   FIRST: tile = element bits [0, TB) (contiguous), reads the user's input.
//   else : tile = bits [0, CL) + [G0, G0+GW), reads the intermediate.
//   LAST : writes dyadic order (bit-reversed addresses) in the output type.
template <class T, int M, int CL, int G0, int GW, bool FIRST, bool LAST, int EB>
struct MultiPass {
  using W = typename IoTraits<T>::C;  // intermediate precision
  using TIn = typename std::conditional<FIRST, T, W>::type;
  using TOut = typename std::conditional<LAST, T, W>::type;
  static constexpr int kCL = FIRST ? 0 : CL;
  static constexpr int kG0 = FIRST ? 0 : G0;
  static constexpr int TB = FIRST ? GW : CL + GW;
  using MapIn = PassMap<kCL, kG0>;
  using MapOut = typename std::conditional<LAST, RevPassMap<M, kCL, kG0>, PassMap<kCL, kG0>>::type;
  using Pass = TilePass<TIn, TOut, MapIn, MapOut, TB, EB, kCL, GW>;
  static constexpr int NT = Pass::NT;
  static constexpr int SMEM_BYTES = Pass::SMEM_BYTES;
  static constexpr int LO_W = kG0 - kCL;        // outer bits below the group
  static constexpr int HI_W = M - kG0 - GW;     // outer bits above the group
  static_assert(HI_W >= 0 && LO_W >= 0, "bad pass geometry");

  __device__ __forceinline__ static void bases(uint64_t tile, uint64_t& bin, uint64_t& bout) {
    const uint32_t lo = (uint32_t)tile & ((1u << LO_W) - 1u);
    const uint32_t hi = (uint32_t)(tile >> LO_W) & ((1u << HI_W) - 1u);
    const uint64_t row = tile >> (LO_W + HI_W);
    const uint32_t off = (lo << kCL) | (hi << (kG0 + GW));
    bin = (row << M) | off;
    bout = LAST ? ((row << M) | rev_bits(off, M)) : bin;
  }
};

// ---------------------------------------------------------------------------
// Tuned plan, f32 m = 12 (BASELINE cfg2): one 16 KiB row per 64-thread CTA,
// 64 registers per thread, ONE shared-memory round trip.
//   load   : regs {0,1 | 8..11}  thr {2..7}        (float4, 512 B per warp load)
//   phase 0: butterflies on 0,1,8,9,10,11 in registers
//   smem   : STS.128, swizzle 9->2, 10->3, 11->4 (8-lane wavefronts distinct)
//   phase 1: regs {2..7}  lanes {0,1,9,10,11}  warp {8}; LDS.32 conflict-free
//   store  : dyadic address rev12(j); lanes cover output bits {11,10,2,1,0} so
//            each STG.32 writes four full 32-byte sectors.
// ---------------------------------------------------------------------------
struct PlanF32M12 {
  using IO = float;
  using C = float;
  static constexpr int kM = 12;
  static constexpr int kTB = 12;
  using L0 = Layout<BL<0, 1, 8, 9, 10, 11>, BL<2, 3, 4, 5, 6, 7>>;
  using L1 = Layout<BL<2, 3, 4, 5, 6, 7>, BL<0, 1, 9, 10, 11, 8>>;
  using S = Swz<9, 2, 10, 3, 11, 4>;
  static constexpr int NT = L0::NT;
  static constexpr int SMEM_BYTES = (1 << kTB) * 4;

  template <bool PRED, Scaling SC>
  __device__ __forceinline__ static void run(const float* __restrict__ in, float* __restrict__ out,
                                             float* sm, float scale, uint32_t limit) {
    const uint32_t tid = threadIdx.x;
    float v[64];
    load_global<L0, IdMap>(in, v, tid);
    butterflies<L0, BL<0, 1, 8, 9, 10, 11>, false>(v);
    smem_store<L0, S>(sm, v, tid);
    __syncthreads();
    smem_load<L1, S>(sm, v, tid);
    butterflies<L1, BL<2, 3, 4, 5, 6, 7>, false>(v);
    store_global<L1, RevMap<12>, SC == Scaling::kDeferred>(out, v, tid, scale);
  }
};

// ---------------------------------------------------------------------------
// Tuned plan, bf16 m = 7 (BASELINE cfg3): 32 rows of 128 per 256-thread CTA,
// 16 values per thread, fp32 arithmetic, one shared-memory round trip.
//   load   : regs {0,1,2 | 6}  lanes {3,4,5,7,8}  warps {9,10,11}  (8 x bf16 = 16 B)
//   phase 0: butterflies on 0,1,2,6
//   smem   : fp32 STS.128 with swizzle 5->2, 7->3, 8->4
//   phase 1: regs {3,4,5,6}  lanes {0,1,2,7,8}; LDS.32 conflict-free
//   store  : output bits 0..3 = tile bits 6,5,4,3 are registers, so each thread
//            writes 16 consecutive bf16 (two STG.128)
// ---------------------------------------------------------------------------
struct PlanBF16M7 {
  using IO = __nv_bfloat16;
  using C = float;
  static constexpr int kM = 7;
  static constexpr int kTB = 12;
  using L0 = Layout<BL<0, 1, 2, 6>, BL<3, 4, 5, 7, 8, 9, 10, 11>>;
  using L1 = Layout<BL<3, 4, 5, 6>, BL<0, 1, 2, 7, 8, 9, 10, 11>>;
  using S = Swz<5, 2, 7, 3, 8, 4>;
  static constexpr int NT = L0::NT;
  static constexpr int SMEM_BYTES = (1 << kTB) * 4;

  template <bool PRED, Scaling SC>
  __device__ __forceinline__ static void run(const IO* __restrict__ in, IO* __restrict__ out, float* sm,
                                             float scale, uint32_t limit) {
    const uint32_t tid = threadIdx.x;
    float v[16];
    if constexpr (PRED)
      load_global_pred<L0, IdMap>(in, v, tid, limit);
    else
      load_global<L0, IdMap>(in, v, tid);
    butterflies<L0, BL<0, 1, 2, 6>, false>(v);
    smem_store<L0, S>(sm, v, tid);
    __syncthreads();
    smem_load<L1, S>(sm, v, tid);
    butterflies<L1, BL<3, 4, 5>, false>(v);
    if constexpr (PRED)
      store_global_pred<L1, RevMap<7>, SC == Scaling::kDeferred>(out, v, tid, scale, limit);
    else
      store_global<L1, RevMap<7>, SC == Scaling::kDeferred>(out, v, tid, scale);
  }
};

}  // namespace chwb
