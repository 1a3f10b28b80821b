// fused.cuh — K5: two-phase persistent dataflow kernel for long rows.
//
// A row of n = 2^m elements is viewed as [H][L] (L = 2^a low bits, H = 2^b high
// bits).  Phase A transforms the low bits of contiguous tiles and writes an
// intermediate; phase B transforms the high bits of column tiles (c contiguous
// low address bits x all H) and writes dyadic order, i = rev_m(j).  Both phases
// run in ONE persistent launch: CTAs claim work items in a fixed order from a
// global counter (A tiles of row-chunk q, then B tiles of chunk q - lag, ...),
// B tiles of chunk q wait on a per-chunk completion counter for A(q), and A
// tiles reusing an intermediate slot wait for the B tiles that drained it.
// Waits only ever point at earlier-claimed items held by running CTAs, so the
// schedule cannot deadlock whatever the grid size.
//
// The intermediate lives in a small ring of chunk-sized slots: every slot is
// rewritten while its lines are still in L2, so it is served by the 126 MB L2
// instead of HBM (ld/st.global.cg), while the user's input and output stream
// with evict-first hints (ld/st.global.cs).  HBM traffic therefore stays close
// to one read + one write of each element — the single-pass roofline.
//
// The intermediate address of in-row index j is a bit permutation Pi(j) chosen
// so A's final register layout stores coalesced 16-byte vectors and B's loads
// are whole 32/64-byte sectors (tools/plan_check.py verifies the plans).
#pragma once

#include "plans.cuh"

namespace chwb {

template <int... P>
struct ListMap {
  CHW_HD static constexpr int pos(int k) {
    constexpr int a[sizeof...(P) + 1] = {P..., -1};
    return a[k];
  }
};

// Deposit the low bits of x onto the bit positions listed in L (runtime x).
template <class L>
__device__ __forceinline__ uint32_t deposit(uint32_t x) {
  uint32_t o = 0;
#pragma unroll
  for (int k = 0; k < L::N; ++k) o |= ((x >> k) & 1u) << L::at(k);
  return o;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Poll without ld.acquire: an acquire load invalidates L1 (CCTL.IVALL) on every
// probe.  Data published by other CTAs is only ever read with L2-coherent
// ld.global.cg after the CTA barrier that follows this poll, and the producer
// published it with red.release.gpu, so a relaxed poll is sufficient here.
__device__ __forceinline__ void wait_at_least(const uint32_t* p, uint32_t target) {
  if (ld_relaxed_u32(p) >= target) return;
  while (ld_relaxed_u32(p) < target) __nanosleep(32);
}

// ---------------------------------------------------------------------------
// Tile runners shared by all fused specs: two layouts, one shared-memory round
// trip, optional shuffle butterfly on one lane bit in the second layout.
// ---------------------------------------------------------------------------
template <class L0, class L1, class S, class B0, class B1, int SHFL_BIT, class MapIn, class MapOut,
          Cache CI, Cache COUT, bool SCALE, class TIn, class TOut, class C>
__device__ __forceinline__ void run_two_phase(const TIn* __restrict__ in, TOut* __restrict__ out,
                                              C* sm, C scale) {
  const uint32_t tid = threadIdx.x;
  C v[L0::E];
  load_global<L0, MapIn, CI>(in, v, tid);
  butterflies<L0, B0, false>(v);
  smem_store<L0, S>(sm, v, tid);
  __syncthreads();
  smem_load<L1, S>(sm, v, tid);
  butterflies<L1, B1, false>(v);
  if constexpr (SHFL_BIT >= 0) shfl_butterfly<L1, SHFL_BIT, false>(v, tid);
  store_global<L1, MapOut, SCALE, COUT>(out, v, tid, scale);
}

// ---------------------------------------------------------------------------
// m = 16, f32 (BASELINE cfg4): L = H = 256.  64-thread CTAs, 16 KiB tiles.
//   A tile: 16 rows h of 256 l (tile bits k0..7 = j0..7, k8..11 = j8..11).
//   B tile: 16 columns (intermediate address bits 0..3) x 256 h.
//   Pi: j2->0 j3->1 j0->2 j1->3 j6->4 j7->5 j8->6 j4->7 j5->8, rest identity.
// ---------------------------------------------------------------------------
struct FusedF32M16 {
  using T = float;
  using W = float;
  static constexpr int M = 16;
  static constexpr int NT = 64;
  static constexpr int MIN_BLOCKS = 10;  // caps registers at ~96/thread
  static constexpr int SMEM_BYTES = 4096 * 4;
  static constexpr int A_TILES_PER_ROW = 16;
  static constexpr int B_TILES_PER_ROW = 16;
  static constexpr int CHUNK_ROWS = 32;
  static constexpr int LAG = 1;
  static constexpr int NSLOTS = 3;

  struct A {
    using L0 = Layout<BL<0, 1, 6, 7, 10, 11>, BL<2, 3, 4, 5, 8, 9>>;
    using L1 = Layout<BL<2, 3, 4, 5, 10, 11>, BL<0, 1, 6, 7, 8, 9>>;
    using S = Swz<6, 2, 7, 3, 8, 4>;
    using MapOut = ListMap<2, 3, 0, 1, 7, 8, 4, 5, 6, 9, 10, 11>;
  };
  struct B {
    using L0 = Layout<BL<0, 1, 8, 9, 10, 11>, BL<2, 3, 4, 5, 6, 7>>;
    using L1 = Layout<BL<4, 5, 6, 7, 10, 11>, BL<9, 8, 0, 1, 2, 3>>;
    using S = Swz<8, 3, 9, 4>;
    using MapIn = ListMap<0, 1, 2, 3, 6, 9, 10, 11, 12, 13, 14, 15>;
    using MapOut = ListMap<13, 12, 15, 14, 7, 6, 5, 4, 3, 2, 1, 0>;
    using OuterAddr = BL<4, 5, 7, 8>;    // intermediate address bits of the tile index
    using OuterOut = BL<9, 8, 11, 10>;   // = rev16 of Pi^-1 of those bits
  };

  // tile `a` (within the chunk): row-in-chunk and in-row offsets
  __device__ __forceinline__ static void a_offsets(uint32_t a, uint32_t& row, uint32_t& in_off,
                                                   uint32_t& mid_off) {
    row = a >> 4;
    in_off = (a & 15u) << 12;
    mid_off = in_off;  // Pi is the identity on j12..15
  }
  __device__ __forceinline__ static void b_offsets(uint32_t b, uint32_t& row, uint32_t& mid_off,
                                                   uint32_t& out_off) {
    row = b >> 4;
    mid_off = deposit<typename B::OuterAddr>(b & 15u);
    out_off = deposit<typename B::OuterOut>(b & 15u);
  }
  template <bool SCALE>
  __device__ __forceinline__ static void run_a(const T* in, W* mid, W* sm, W scale) {
    run_two_phase<typename A::L0, typename A::L1, typename A::S, BL<0, 1, 6, 7>, BL<2, 3, 4, 5>, -1,
                  IdMap, typename A::MapOut, Cache::kStream, Cache::kL2, false>(in, mid, sm, scale);
  }
  template <bool SCALE>
  __device__ __forceinline__ static void run_b(const W* mid, T* out, W* sm, W scale) {
    run_two_phase<typename B::L0, typename B::L1, typename B::S, BL<8, 9, 10, 11>, BL<4, 5, 6, 7>, -1,
                  typename B::MapIn, typename B::MapOut, Cache::kL2, Cache::kStream, SCALE>(mid, out, sm,
                                                                                              scale);
  }
};

// ---------------------------------------------------------------------------
// m = 16, f32, 32 values per thread (128-thread tiles): twice the warps per SM
// of FusedF32M16 for the latency-bound two-phase schedule.
//   Pi: j2->0 j3->1 j0->2 j1->3 j5->4 j6->5 j7->6 j4->7, rest identity.
// ---------------------------------------------------------------------------
struct FusedF32M16b {
  using T = float;
  using W = float;
  static constexpr int M = 16;
  static constexpr int NT = 128;
  static constexpr int MIN_BLOCKS = 4;
  static constexpr int SMEM_BYTES = 4096 * 4;
  static constexpr int A_TILES_PER_ROW = 16;
  static constexpr int B_TILES_PER_ROW = 16;
  static constexpr int CHUNK_ROWS = 32;
  static constexpr int LAG = 4;     // > the per-CTA prefetch window, in chunk rounds
  static constexpr int NSLOTS = 6;  // 6 x 8 MiB intermediate ring: L2-resident

  struct A {
    using L0 = Layout<BL<0, 1, 5, 6, 7>, BL<2, 3, 4, 8, 9, 10, 11>>;
    using L1 = Layout<BL<2, 3, 4, 10, 11>, BL<0, 1, 5, 6, 7, 8, 9>>;
    using S = Swz<5, 2, 6, 3, 7, 4>;
    using MapOut = ListMap<2, 3, 0, 1, 7, 4, 5, 6, 8, 9, 10, 11>;
    using B0 = BL<0, 1, 5, 6, 7>;
    using B1 = BL<2, 3, 4>;
  };
  struct B {
    using L0 = Layout<BL<0, 1, 9, 10, 11>, BL<2, 3, 4, 5, 6, 7, 8>>;
    using L1 = Layout<BL<4, 5, 6, 7, 8>, BL<11, 10, 9, 0, 1, 2, 3>>;
    using S = Swz<9, 2, 10, 3, 11, 4>;
    using MapIn = ListMap<0, 1, 2, 3, 8, 9, 10, 11, 12, 13, 14, 15>;
    using MapOut = ListMap<13, 12, 15, 14, 7, 6, 5, 4, 3, 2, 1, 0>;
    using OuterAddr = BL<4, 5, 6, 7>;
    using OuterOut = BL<10, 9, 8, 11>;
    using B0 = BL<9, 10, 11>;
    using B1 = BL<4, 5, 6, 7, 8>;
  };

  __device__ __forceinline__ static void a_offsets(uint32_t a, uint32_t& row, uint32_t& in_off,
                                                   uint32_t& mid_off) {
    row = a >> 4;
    in_off = (a & 15u) << 12;
    mid_off = in_off;
  }
  __device__ __forceinline__ static void b_offsets(uint32_t b, uint32_t& row, uint32_t& mid_off,
                                                   uint32_t& out_off) {
    row = b >> 4;
    mid_off = deposit<typename B::OuterAddr>(b & 15u);
    out_off = deposit<typename B::OuterOut>(b & 15u);
  }
  template <bool SCALE>
  __device__ __forceinline__ static void run_a(const T* in, W* mid, W* sm, W scale) {
    run_two_phase<typename A::L0, typename A::L1, typename A::S, typename A::B0, typename A::B1, -1, IdMap,
                  typename A::MapOut, Cache::kStream, Cache::kL2, false>(in, mid, sm, scale);
  }
  template <bool SCALE>
  __device__ __forceinline__ static void run_b(const W* mid, T* out, W* sm, W scale) {
    run_two_phase<typename B::L0, typename B::L1, typename B::S, typename B::B0, typename B::B1, -1,
                  typename B::MapIn, typename B::MapOut, Cache::kL2, Cache::kStream, SCALE>(mid, out, sm,
                                                                                              scale);
  }
};

// ---------------------------------------------------------------------------
// m = 24, f32 (BASELINE cfg5): L = 2^13, H = 2^11.  256-thread CTAs, 64 KiB.
//   A tile: 2 consecutive h-blocks of 8192 contiguous (k0..12 = j0..12, k13 = j13).
//   B tile: 8 columns (intermediate address bits 0..2) x 2048 h.
//   Pi: j8->0 j0->1 j1->2 j9->3 j10->4 j2..7->5..10, rest identity.
// One row per chunk; a single slot (64 MiB) reused row after row so its lines
// are overwritten in L2 instead of written back.
// ---------------------------------------------------------------------------
struct FusedF32M24 {
  using T = float;
  using W = float;
  static constexpr int M = 24;
  static constexpr int NT = 256;
  static constexpr int MIN_BLOCKS = 2;  // caps registers at 128/thread
  static constexpr int SMEM_BYTES = 16384 * 4;
  static constexpr int A_TILES_PER_ROW = 1024;
  static constexpr int B_TILES_PER_ROW = 1024;
  static constexpr int CHUNK_ROWS = 1;
  static constexpr int LAG = 0;
  static constexpr int NSLOTS = 1;

  struct A {
    using L0 = Layout<BL<0, 1, 9, 10, 11, 12>, BL<2, 3, 4, 5, 6, 7, 8, 13>>;
    using L1 = Layout<BL<2, 3, 4, 5, 6, 7>, BL<8, 0, 1, 9, 10, 11, 12, 13>>;
    using S = Swz<8, 2, 9, 3, 10, 4>;
    using MapOut = ListMap<1, 2, 5, 6, 7, 8, 9, 10, 0, 3, 4, 11, 12, 13>;
  };
  struct B {
    using L0 = Layout<BL<0, 1, 10, 11, 12, 13>, BL<2, 3, 4, 5, 6, 7, 8, 9>>;
    using L1 = Layout<BL<3, 4, 5, 6, 7, 8>, BL<13, 12, 11, 10, 9, 0, 1, 2>>;
    using S = Swz<9, 0, 10, 1, 11, 2, 12, 3, 13, 4, 5, 0, 6, 1>;
    using MapIn = ListMap<0, 1, 2, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23>;
    using MapOut = ListMap<15, 23, 22, 10, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0>;
    using OuterAddr = BL<3, 4, 5, 6, 7, 8, 9, 10, 11, 12>;
    using OuterOut = BL<14, 13, 21, 20, 19, 18, 17, 16, 12, 11>;
  };

  __device__ __forceinline__ static void a_offsets(uint32_t a, uint32_t& row, uint32_t& in_off,
                                                   uint32_t& mid_off) {
    row = a >> 10;
    in_off = (a & 1023u) << 14;
    mid_off = in_off;
  }
  __device__ __forceinline__ static void b_offsets(uint32_t b, uint32_t& row, uint32_t& mid_off,
                                                   uint32_t& out_off) {
    row = b >> 10;
    mid_off = deposit<typename B::OuterAddr>(b & 1023u);
    out_off = deposit<typename B::OuterOut>(b & 1023u);
  }
  template <bool SCALE>
  __device__ __forceinline__ static void run_a(const T* in, W* mid, W* sm, W scale) {
    run_two_phase<typename A::L0, typename A::L1, typename A::S, BL<0, 1, 9, 10, 11, 12>,
                  BL<2, 3, 4, 5, 6, 7>, 8, IdMap, typename A::MapOut, Cache::kStream, Cache::kL2, false>(
        in, mid, sm, scale);
  }
  template <bool SCALE>
  __device__ __forceinline__ static void run_b(const W* mid, T* out, W* sm, W scale) {
    run_two_phase<typename B::L0, typename B::L1, typename B::S, BL<10, 11, 12, 13>,
                  BL<3, 4, 5, 6, 7, 8>, 9, typename B::MapIn, typename B::MapOut, Cache::kL2,
                  Cache::kStream, SCALE>(mid, out, sm, scale);
  }
};

}  // namespace chwb
