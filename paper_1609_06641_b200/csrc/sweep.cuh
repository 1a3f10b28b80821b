// sweep.cuh — K9: single-HBM-pass row sweep for f32 m = 24 (BASELINE cfg5).
//
// The transform of one 2^24 row needs every input element before any output
// element exists, so a single HBM pass must hold a whole row's intermediate
// (64 MiB) on chip between its two phases.  K9 keeps it in L2 and runs the
// whole chip on one row at a time, both phases concurrently:
//
//   A(r, a): contiguous 64 KiB input tile a (j bits 14..23 = a) of row r,
//            TMA bulk copy into a 2-stage ring -> butterflies on j bits 0, 1
//            and 4..13 (7 register bits, one in-place smem transpose, 5 more)
//            -> the row workspace W (L2-resident, st .cg);
//   B(r, v): B tile v of W (4 "passenger" j bits 2, 3, 5, 6 kept together for
//            64-byte runs + j bits 14..23), one TMA copy from L2 ->
//            butterflies on j bits 2, 3 and 14..23 (7 register bits, the
//            transpose through a 32 KiB buffer one half at a time, 5 more) ->
//            dyadic output (16-byte stores, 512 contiguous bytes per warp
//            instruction).
// The NATURAL-order plan of the same sweep (K9n, SweepNatF32M24 /
// sweep_nat_m24_kernel) is further down; what bounds both — the SM<->L2 fabric,
// not the SM side — is measured in DESIGN.md §4.1a.
//
// Workspace layouts alternate per row (P for even rows, Q for odd):
//   P: addr[0..3] = passengers, addr[4..13] = v bits, addr[14..23] = a bits;
//   Q: addr[0..3] = passengers, addr[4..13] = a bits, addr[14..23] = v bits.
// With that, A(r+1, t) overwrites exactly the region B(r, t) read (the same
// index t), and CTA c owns A tiles and B tiles {c, c+G, ...}: the WAR
// dependency stays inside the CTA (mbarrier `regionfree[i]`).  The only
// cross-CTA dependency is RAW: B(r, .) needs all 1024 A(r, .) tiles — one
// global counter per row (red.release.gpu by each A tile after an
// async-proxy fence, acquire poll + proxy fence by the B producer).  All CTAs are co-resident
// (cooperative launch, one CTA per SM), so the waits cannot deadlock.
//
// Roles per CTA (256 threads): warps 0-3 A group, warps 4-7 B group; thread
// 0 of each group issues its TMA copies.  Shared memory: 2 A stages (tiles
// transposed in place) + 1 B stage (64 KiB each) + the 32 KiB B transpose
// buffer.
//
// Every layout/swizzle/position map below was checked with tools/plan_check.py
// (tools/swz_search.py): all shared-memory accesses conflict-free, every
// global access whole 32-byte sectors (16 per warp instruction).
#pragma once

#include "passtma.cuh"

// Compile-time switches.  The defaults are the shipped kernel; the others are
// the A/B and diagnostic builds behind profiles/r02_ab_sweep_*.txt
// (tools/build_ab.sh).  Measured slower and removed from the source in round
// 2: A tiles leaving through a TMA store (0.502 vs 0.535), B tiles loaded
// straight from L2 into registers (0.464), L2 discard of consumed layout-Q
// regions (0.522), butterflying the passengers j2, j3 in A instead of B
// (0.526 vs 0.546), and K9b — 64-value threads, 16 warps, three layouts (0.49).
#ifndef CHW_SWEEP_OPAQUE
#define CHW_SWEEP_OPAQUE 1  // opaque thread index: keeps swizzled addresses out of live registers (no spills)
#endif
// Debug builds (-DCHW_SWEEP_TRACE=1, tools/sweep_trace.py) record %globaltimer
// stamps per tile for CTAs 0 and 1: [cta][group][item][event].
#ifndef CHW_SWEEP_TRACE
#define CHW_SWEEP_TRACE 0
#endif
// Diagnostic builds only (wrong results): 1 = the A group alone (no waits on B),
// 2 = the B group alone (no waits on A), 3 = both warp groups run B tiles —
// each group's stand-alone tile rate (profiles/r02_ab_sweep_only.txt).
#ifndef CHW_SWEEP_ONLY
#define CHW_SWEEP_ONLY 0
#endif
// Which tile (A: input tile a = j14..23; B: workspace tile v) the CTA's i-th
// item c + i G names: a fixed bit permutation of that number, the same for A
// and B (so A(r+1, .) still overwrites exactly what B(r, .) read).  0: identity
// (CTAs c, c+1 share every 128-byte workspace line); 1: the low item bits are
// the tile bits that sit lowest in the OUTPUT position (out bits 10..16), so
// the 148 CTAs write neighbouring 4 KiB runs at any moment; 2: bit 0 kept, bits
// 1..4 -> out bits 10..13.  Measured 0.527 / 0.516 / 0.521
// (profiles/r02_ab_sweep_tperm.txt).
#ifndef CHW_SWEEP_TPERM
#define CHW_SWEEP_TPERM 0
#endif
// Workspace cache hints: bit 0 = A's workspace stores carry an L2 evict_last
// policy, bit 1 = B's workspace loads carry evict_first (the data is dead once
// read).  Measured 0.506 / 0.526 / 0.515 vs 0.526 (profiles/r02_ab_sweep_wshint.txt).
#ifndef CHW_SWEEP_WSHINT
#define CHW_SWEEP_WSHINT 0
#endif

namespace chwb {

struct SweepF32M24 {
  static constexpr int M = 24;
  static constexpr int TILE = 1 << 14;
  static constexpr int NT = 128;             // threads per compute group
  static constexpr uint32_t NTILES = 1024;   // A tiles (and B tiles) per row
  // ---- A tiles: tile bit k = j bit k (k = 0..13), natural order in the stage.
  using AL0 = Layout<BL<0, 1, 5, 6, 7, 8, 9>, BL<2, 3, 4, 10, 11, 12, 13>>;
  using AL1 = Layout<BL<2, 3, 4, 10, 11, 12, 13>, BL<5, 6, 0, 1, 7, 8, 9>>;
  using AS = Swz<5, 2, 6, 3, 7, 4>;
  using AB0 = BL<0, 1, 5, 6, 7, 8, 9>;
  // passengers j2, j3 are butterflied by B (register bits t0, t1 of BL0)
  using AB1 = BL<4, 10, 11, 12, 13>;
  // workspace position of tile bit k: passengers j2,j3,j5,j6 -> addr 0..3;
  // v bits (j0,j1,j7,j8,j9,j4,j10..13) -> addr 4..13 (P) or 14..23 (Q).
  using AOutP = ListMap<4, 5, 0, 1, 9, 2, 3, 6, 7, 8, 10, 11, 12, 13>;         // tile base a << 14
  using AOutQ = ListMap<14, 15, 0, 1, 19, 2, 3, 16, 17, 18, 20, 21, 22, 23>;   // tile base a << 4
  // ---- B tiles: tile bits t0..t3 = passengers (addr 0..3), t4..t13 = j14..23.
  using BL0 = Layout<BL<0, 1, 7, 8, 9, 10, 11>, BL<2, 3, 4, 5, 6, 12, 13>>;
  using BL1 = Layout<BL<13, 12, 4, 5, 6, 0, 1>, BL<11, 10, 9, 8, 7, 2, 3>>;
  using BS = Swz<9, 2, 10, 3, 11, 4>;
  using BB0 = BL<0, 1, 7, 8, 9, 10, 11>;
  using BB1 = BL<4, 5, 6, 12, 13>;
  // B tile positions in a layout-P workspace (tile base v << 4); layout Q: IdMap (base v << 14).
  using BInP = ListMap<0, 1, 2, 3, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23>;
  // The B transpose goes through a 32 KiB buffer in two halves (t0 = 0, 1):
  // the same layouts with tile bit t0 removed (tile bits renumbered t1 -> 0,
  // ..., t13 -> 12); 8-byte vectors on t1; conflict-free (tools/swz_search.py).
  using BH0 = Layout<BL<0, 6, 7, 8, 9, 10>, BL<1, 2, 3, 4, 5, 11, 12>>;
  using BH1 = Layout<BL<12, 11, 3, 4, 5, 0>, BL<10, 9, 8, 7, 6, 1, 2>>;
  using BHS = Swz<7, 1, 8, 2, 9, 3, 10, 4>;
  static constexpr int BL0_T0 = 0;  // register bit of t0 in BL0
  using BHB1 = BL<3, 4, 5, 11, 12>;                                      // BB1 in half numbering
  using BOutH = ListMap<20, 18, 17, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0>;       // BOut without t0 (out bit 21)
  // dyadic output position (bit q = j bit 23 - q) of tile bit t, and of the
  // B tile index bits (v0..v9 = j0,j1,j7,j8,j9,j4,j10,j11,j12,j13).
  using BOut = ListMap<21, 20, 18, 17, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0>;
  using BOuter = BL<23, 22, 16, 15, 14, 19, 13, 12, 11, 10>;
  static constexpr int E = AL0::E;
  static constexpr bool kNatural = false;
  static_assert(AL0::NT == NT && BL0::NT == NT && BL0::E == E, "group shape");
};

// The same sweep with NATURAL output order (chw_order 1, orderings.hpp:45-78)
// folded in.  The output position of row bit j is j itself, so the B tile's
// passengers must be j0..j3 (whole 64-byte runs in the output): workspace addr
// 0..3 = j0..j3, v bits = j4..j13 in order.  A butterflies j0, j1 (first
// layout, they are its 16-byte vector) and j4..j13; j0, j1 ride along in its
// second layout, so both sides of A's transpose are 16-byte accesses.  B
// butterflies j2, j3 and j14..j23: its first layout holds t0..t3 in registers,
// which is conflict-free only if the stage is written under TMA's 64-byte
// swizzle (BStage); no register bit is shared between B's two layouts, so the
// transpose is in place in the stage (no half buffer) and the stores are
// scalar, two whole 64-byte runs per warp instruction.
struct SweepNatF32M24 {
  static constexpr int M = 24;
  static constexpr int TILE = 1 << 14;
  static constexpr int NT = 128;
  static constexpr uint32_t NTILES = 1024;
  using AL0 = Layout<BL<0, 1, 5, 6, 7, 8, 9>, BL<2, 3, 4, 10, 11, 12, 13>>;
  using AL1 = Layout<BL<0, 1, 4, 10, 11, 12, 13>, BL<2, 3, 5, 6, 7, 8, 9>>;
  using AS = Swz<5, 4>;
  using AB0 = BL<0, 1, 5, 6, 7, 8, 9>;
  using AB1 = BL<4, 10, 11, 12, 13>;
  using AOutP = IdMap;                                                          // tile base a << 14
  using AOutQ = ListMap<0, 1, 2, 3, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23>;   // tile base a << 4
  // B tile bits t0..t3 = j0..j3 (addr 0..3), t4..t13 = j14..j23
  using BL0 = Layout<BL<0, 1, 2, 3, 7, 8, 9>, BL<4, 5, 6, 10, 11, 12, 13>>;
  using BL1 = Layout<BL<4, 5, 6, 10, 11, 12, 13>, BL<0, 1, 2, 3, 7, 8, 9>>;
  using BStage = Swz<5, 2, 6, 3>;        // CU_TENSOR_MAP_SWIZZLE_64B in float-index bits
  using BS = Swz<5, 2, 6, 3, 7, 4>;
  using BB0 = BL<2, 3, 7, 8, 9>;
  using BB1 = BL<4, 5, 6, 10, 11, 12, 13>;
  using BInP = ListMap<0, 1, 2, 3, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23>;
  using BOut = ListMap<0, 1, 2, 3, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23>;    // natural position; tile index v -> v << 4
  static constexpr int E = AL0::E;
  static constexpr bool kNatural = true;
  static_assert(AL0::NT == NT && AL1::NT == NT && BL0::NT == NT && BL1::NT == NT && BL0::E == E, "group shape");
};

// B-side tensor map (layout P rows): the workspace as [4][256][1024][16]
// floats (addr 22..23, 14..21, 4..13, 0..3), box {16, 1, 256, 4} = one B tile
// in tile-bit order (t0..3 = addr 0..3, t4..13 = addr 14..23).  Layout Q rows
// read a contiguous 64 KiB region with one bulk copy.
__device__ __forceinline__ void tensor4_g2s_hint(void* dst, const void* tmap, int x, int y, int z, int w,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
      "{%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// Register index of layout L from the half-layout index rh: insert bit HV at
// register bit SLOT (the half layouts list L's register bits minus that one,
// in the same order).
CHW_HD constexpr int ins_bit(int rh, int slot, int hv) {
  return (rh & ((1 << slot) - 1)) | (hv << slot) | ((rh >> slot) << (slot + 1));
}
// Store / load the half (tile bit 0 == HV) of a 128-value tile through a
// half-size shared buffer addressed in the half layout Lh under swizzle S.
template <class Lh, class S, int SLOT, int HV, int E>
__device__ __forceinline__ void smem_store_half(float* sm, const float (&v)[E], uint32_t tid) {
  constexpr int VB = smem_vec_bits<Lh, S, 2>();
  constexpr uint32_t tmask = S::image(thr_mask<Lh, IdMap>());
  const uint32_t sb = S::apply(thr_off<Lh, IdMap>(tid));
  static_for<Lh::E>([&](auto R) {
    constexpr int rh = decltype(R)::value;
    if constexpr (vec_head<Lh, IdMap>(rh, VB)) {
      constexpr uint32_t so = S::apply(reg_off<Lh, IdMap>(rh));
      const uint32_t a = (so & tmask) ? (sb ^ so) : (sb + so);
      float tmp[1 << VB];
      static_for<(1 << VB)>([&](auto Q) {
        tmp[decltype(Q)::value] = v[ins_bit(vec_elem<Lh, IdMap>(rh, decltype(Q)::value, VB), SLOT, HV)];
      });
      SmemVec<float, VB>::st(sm + a, tmp);
    }
  });
}
template <class Lh, class S, int E2>
__device__ __forceinline__ void smem_load_half(const float* sm, float (&w)[E2], uint32_t tid) {
  constexpr int VB = smem_vec_bits<Lh, S, 2>();
  constexpr uint32_t tmask = S::image(thr_mask<Lh, IdMap>());
  const uint32_t sb = S::apply(thr_off<Lh, IdMap>(tid));
  static_for<Lh::E>([&](auto R) {
    constexpr int rh = decltype(R)::value;
    if constexpr (vec_head<Lh, IdMap>(rh, VB)) {
      constexpr uint32_t so = S::apply(reg_off<Lh, IdMap>(rh));
      const uint32_t a = (so & tmask) ? (sb ^ so) : (sb + so);
      float tmp[1 << VB];
      SmemVec<float, VB>::ld(sm + a, tmp);
      static_for<(1 << VB)>([&](auto Q) { w[vec_elem<Lh, IdMap>(rh, decltype(Q)::value, VB)] = tmp[decltype(Q)::value]; });
    }
  });
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Roles (256 threads = 8 warps, so each thread may use up to 255 registers:
// a 9th warp would put 3 warps on one SM sub-partition and cap registers at
// 168, which spills the 128-value tiles): warps 0-3 A group, warps 4-7 B
// group.  The TMA copies are issued by thread 0 of each group the moment a
// stage becomes free: A stages hold input tiles (HBM), the B stage holds
// workspace tiles (L2).  B(r, .) is issued only once all 1024 A(r, .) tiles
// are counted (acquire + async-proxy fence); B(r, i)'s bytes landing in
// shared memory free its workspace region, so the B group signals
// `regionfree[i]` as soon as the stage is full and A(r+1, i) may overwrite it.
#if CHW_SWEEP_TRACE
__device__ unsigned long long* g_sweep_trace = nullptr;
__device__ __forceinline__ void trace_stamp(uint32_t cta, uint32_t grp, uint32_t item, uint32_t ev) {
  if (g_sweep_trace && cta < 2 && item < 512) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_sweep_trace[((cta * 2 + grp) * 512 + item) * 8 + ev] = t;
  }
}
#define SWEEP_STAMP(grp, ev) \
  if (gt == 0) trace_stamp(c, grp, u, ev)
#else
#define SWEEP_STAMP(grp, ev) \
  do {                       \
  } while (0)
#endif

__device__ __forceinline__ uint32_t tile_of(uint32_t item) {
#if CHW_SWEEP_TPERM == 1
  return deposit<BL<9, 8, 7, 6, 4, 3, 2, 5, 1, 0>>(item);
#elif CHW_SWEEP_TPERM == 2
  return deposit<BL<0, 9, 8, 7, 6, 4, 3, 2, 5, 1>>(item);
#else
  return item;
#endif
}

template <bool SCALE, bool SEQ = false>
__global__ void __launch_bounds__(2 * SweepF32M24::NT, 1)
    sweep_m24_kernel(const float* __restrict__ in, float* __restrict__ out, float* __restrict__ ws,
                     uint32_t* __restrict__ cnt, uint32_t rows, float scale, const __grid_constant__ TmapParam tmapP) {
  using P = SweepF32M24;
  constexpr int TILE = P::TILE;
  constexpr uint32_t TB = TILE * 4;
  constexpr int NT = P::NT;
  constexpr int SA = 2;
  constexpr int MAXT = 8;  // tiles per CTA per row (ceil(1024 / 148) = 7)
  extern __shared__ __align__(128) float smem_sw[];
  float* ringA = smem_sw;
  float* stageB = smem_sw + SA * TILE;
  float* bufB = stageB + TILE;  // TILE / 2 floats: the B transpose buffer
  __shared__ __align__(8) uint64_t fullA[SA], fullB, regionfree[MAXT];
  const uint32_t tid = threadIdx.x;
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const uint32_t nt = (P::NTILES - c + G - 1) / G;  // tiles this CTA owns: c, c+G, ...
  if (nt == 0 || nt > MAXT) return;
  if (tid == 0) {
    for (int s = 0; s < SA; ++s) mbar_init_cta(&fullA[s], 1);
    mbar_init_cta(&fullB, 1);
    for (int k = 0; k < MAXT; ++k) mbar_init_cta(&regionfree[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t total = rows * nt;  // A items (and B items) of this CTA
  float v[P::E];
  if (tid < (uint32_t)NT && CHW_SWEEP_ONLY != 3) {  // ---- A group
    if (CHW_SWEEP_ONLY == 2) return;
    const uint32_t gt = tid;
    auto bar = [] { named_bar(1, NT); };
    uint64_t pol = 0;
    auto issue = [&](uint32_t u) {  // input tile u -> stage u % SA (the stage is free)
      const uint32_t r = u / nt, i = u - r * nt;
      const int st = (int)(u % SA);
      mbar_expect_tx_cta(&fullA[st], TB);
      const uint64_t a = (uint64_t)tile_of(c + i * G);
      bulk_g2s(ringA + st * TILE, in + ((uint64_t)r << 24) + (a << 14), TB, &fullA[st], pol);
    };
    if (gt == 0) {
      pol = l2_evict_first_policy();
      for (uint32_t u = 0; u < (uint32_t)SA && u < total; ++u) issue(u);
    }
    for (uint32_t u = 0, r = 0, i = 0; u < total; ++u, i = (i + 1 == nt) ? 0 : i + 1, r += (i == 0)) {
      const int st = (int)(u % SA);
      float* stage = ringA + st * TILE;
      // Opaque copy of the thread index: keeps the per-register swizzled
      // shared-memory addresses inside the loop (hoisted, they need ~20 live
      // registers and spill).
      uint32_t gtv = gt;
#if CHW_SWEEP_OPAQUE
      asm volatile("mov.b32 %0, %1;" : "=r"(gtv) : "r"(gt));
#endif
      SWEEP_STAMP(0, 0);
      mbar_wait_cta(&fullA[st], (u / SA) & 1u);
      SWEEP_STAMP(0, 1);
      smem_load<P::AL0, NoSwz>(stage, v, gtv);
      butterflies<P::AL0, P::AB0, false>(v);
      bar();
      smem_store<P::AL0, P::AS>(stage, v, gtv);
      bar();
      smem_load<P::AL1, P::AS>(stage, v, gtv);
      bar();  // every thread has read the stage: refill it
      if (gt == 0 && u + SA < total) {
        // order the group's generic-proxy reads of the stage before the TMA write
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(u + SA);
      }
      butterflies<P::AL1, P::AB1, false>(v);
      SWEEP_STAMP(0, 2);
      if (CHW_SWEEP_ONLY != 1 && r >= 1) mbar_wait_cta(&regionfree[i], (r - 1) & 1u);  // B(r-1, a) has been read
      SWEEP_STAMP(0, 3);
      const uint32_t a = tile_of(c + i * G);
      if (r & 1u)
        store_global<P::AL1, P::AOutQ, false, (CHW_SWEEP_WSHINT & 1) ? Cache::kL2Last : Cache::kL2>(
            ws + ((uint64_t)a << 4), v, gtv, 1.0f);
      else
        store_global<P::AL1, P::AOutP, false, (CHW_SWEEP_WSHINT & 1) ? Cache::kL2Last : Cache::kL2>(
            ws + ((uint64_t)a << 14), v, gtv, 1.0f);
      if (i + 1 == nt) {  // this CTA's last A tile of row r: publish all nt of them
        asm volatile("fence.proxy.async.global;" ::: "memory");  // other CTAs read them with TMA
        bar();
        if (gt == 0) red_release_add(&cnt[r], nt);
      }
      SWEEP_STAMP(0, 4);
    }
  } else {  // ---- B group
    if (CHW_SWEEP_ONLY == 1) return;
    // CHW_SWEEP_ONLY == 3 (diagnostic): both warp groups run the B path on
    // alternate tiles, each with its own stage, buffer, mbarrier and barrier id.
    const uint32_t bg = (CHW_SWEEP_ONLY == 3) ? tid / NT : 0u;
    const uint32_t ustep = (CHW_SWEEP_ONLY == 3) ? 2u : 1u;
    const uint32_t gt = (CHW_SWEEP_ONLY == 3) ? tid % NT : tid - NT;
    if (CHW_SWEEP_ONLY == 3) {
      stageB = smem_sw + bg * (TILE + TILE / 2);
      bufB = stageB + TILE;
    }
    uint64_t* fullBp = (CHW_SWEEP_ONLY == 3) ? &fullA[bg] : &fullB;
    const uint32_t barid = 2 + bg;
    auto bar = [barid] { named_bar(barid, NT); };
    uint64_t pol = 0;
    // Issue workspace tile u into the (free) B stage.  The first tile of a row
    // needs every A tile of that row: with wait = false the call returns
    // false instead of spinning, and the caller retries before it next waits.
    auto issue = [&](uint32_t u, bool wait) -> bool {
      const uint32_t r = u / nt, i = u - r * nt;
      if (CHW_SWEEP_ONLY < 2 && i == 0) {
        if (ld_relaxed_u32(&cnt[r]) < P::NTILES) {
          if (!wait) return false;
          while (ld_relaxed_u32(&cnt[r]) < P::NTILES) __nanosleep(64);
        }
        (void)ld_acquire_gpu_u32(&cnt[r]);  // synchronizes with every A tile's release
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      mbar_expect_tx_cta(fullBp, TB);
      const uint32_t t = tile_of(c + i * G);
      if (r & 1u)
        bulk_g2s(stageB, ws + ((uint64_t)t << 14), TB, fullBp, pol);
      else
        tensor4_g2s_hint(stageB, &tmapP, 0, (int)t, 0, 0, fullBp, pol);
      return true;
    };
    bool pending = false;  // thread 0: tile u not issued yet
    if (gt == 0) {
      pol = (CHW_SWEEP_WSHINT & 2) ? l2_evict_first_policy() : l2_evict_normal_policy();
      pending = total > bg;
    }
    for (uint32_t u = bg, r = 0, i = bg; u < total; u += ustep) {
      r = u / nt;
      i = u - r * nt;
      SWEEP_STAMP(1, 0);
      if (pending) pending = !issue(u, true);
      SWEEP_STAMP(1, 1);
      uint32_t gtv = gt;  // opaque thread index (see the A loop)
#if CHW_SWEEP_OPAQUE
      asm volatile("mov.b32 %0, %1;" : "=r"(gtv) : "r"(gt));
#endif
      mbar_wait_cta(fullBp, (u / ustep) & 1u);
      SWEEP_STAMP(1, 2);
      // B(r, t)'s workspace bytes are in shared memory: A(r+1, t) may overwrite them.
      if (gt == 0 && CHW_SWEEP_ONLY != 3) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&regionfree[i])) : "memory");
      smem_load<P::BL0, NoSwz>(stageB, v, gtv);
      bar();  // the stage is read: load the next B tile while this one is computed
      if (gt == 0 && u + ustep < total) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        pending = !issue(u + ustep, false);
      }
      SWEEP_STAMP(1, 4);
      butterflies<P::BL0, P::BB0, false>(v);
      SWEEP_STAMP(1, 5);
      // L0 -> L1 through the 32 KiB buffer one t0-half at a time; B1 (which
      // never touches t0) and the stores run per half, so only 64 extra
      // registers are live.
      const uint32_t t = tile_of(c + i * G);
      float* orow = out + ((uint64_t)r << 24);
      const uint32_t outer = deposit<P::BOuter>(t);
      using MapO = typename std::conditional<SEQ, SeqMap<P::BOutH, 24>, P::BOutH>::type;
      float w[P::E / 2];
      smem_store_half<P::BH0, P::BHS, P::BL0_T0, 0>(bufB, v, gtv);
      bar();
      smem_load_half<P::BH1, P::BHS>(bufB, w, gtv);
      bar();
      smem_store_half<P::BH0, P::BHS, P::BL0_T0, 1>(bufB, v, gtv);
      butterflies<P::BH1, P::BHB1, false>(w);
      store_global<P::BH1, MapO, SCALE, Cache::kStream>(orow, w, gtv, scale, outer);
      SWEEP_STAMP(1, 6);
      bar();
      smem_load_half<P::BH1, P::BHS>(bufB, w, gtv);
      butterflies<P::BH1, P::BHB1, false>(w);
      store_global<P::BH1, MapO, SCALE, Cache::kStream>(orow, w, gtv, scale, outer | (1u << 21));
      SWEEP_STAMP(1, 3);
    }
  }
}

// ---------------------------------------------------------------------------
// K9n: the K9 sweep with NATURAL output order folded in (plan SweepNatF32M24).
// Same roles, mbarriers and row protocol as sweep_m24_kernel; the B group
// transposes in place in its stage (shared memory: two A stages + one B
// stage), loads both workspace layouts through swizzling tensor maps and
// stores scalars in whole 64-byte runs.
// ---------------------------------------------------------------------------
template <bool SCALE>
__global__ void __launch_bounds__(2 * SweepNatF32M24::NT, 1)
    sweep_nat_m24_kernel(const float* __restrict__ in, float* __restrict__ out, float* __restrict__ ws,
                         uint32_t* __restrict__ cnt, uint32_t rows, float scale,
                         const __grid_constant__ TmapParam tmapP, const __grid_constant__ TmapParam tmapQ) {
  using P = SweepNatF32M24;
  constexpr int TILE = P::TILE;
  constexpr uint32_t TB = TILE * 4;
  constexpr int NT = P::NT;
  constexpr int SA = 2;
  constexpr int MAXT = 8;
  extern __shared__ __align__(1024) float smem_sn[];
  float* ringA = smem_sn;
  float* stageB = smem_sn + SA * TILE;
  __shared__ __align__(8) uint64_t fullA[SA], fullB, regionfree[MAXT];
  const uint32_t tid = threadIdx.x;
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const uint32_t nt = (P::NTILES - c + G - 1) / G;  // tiles this CTA owns: c, c+G, ...
  if (nt == 0 || nt > MAXT) return;
  if (tid == 0) {
    for (int s = 0; s < SA; ++s) mbar_init_cta(&fullA[s], 1);
    mbar_init_cta(&fullB, 1);
    for (int k = 0; k < MAXT; ++k) mbar_init_cta(&regionfree[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t total = rows * nt;
  float v[P::E];
  if (tid < (uint32_t)NT) {  // ---- A group
    const uint32_t gt = tid;
    auto bar = [] { named_bar(1, NT); };
    uint64_t pol = 0;
    auto issue = [&](uint32_t u) {
      const uint32_t r = u / nt, i = u - r * nt;
      const int st = (int)(u % SA);
      mbar_expect_tx_cta(&fullA[st], TB);
      const uint64_t a = c + (uint64_t)i * G;
      bulk_g2s(ringA + st * TILE, in + ((uint64_t)r << 24) + (a << 14), TB, &fullA[st], pol);
    };
    if (gt == 0) {
      pol = l2_evict_first_policy();
      for (uint32_t u = 0; u < (uint32_t)SA && u < total; ++u) issue(u);
    }
    for (uint32_t u = 0, r = 0, i = 0; u < total; ++u, i = (i + 1 == nt) ? 0 : i + 1, r += (i == 0)) {
      const int st = (int)(u % SA);
      float* stage = ringA + st * TILE;
      uint32_t gtv = gt;  // opaque thread index (see sweep_m24_kernel)
      asm volatile("mov.b32 %0, %1;" : "=r"(gtv) : "r"(gt));
      mbar_wait_cta(&fullA[st], (u / SA) & 1u);
      smem_load<P::AL0, NoSwz>(stage, v, gtv);
      butterflies<P::AL0, P::AB0, false>(v);
      bar();
      smem_store<P::AL0, P::AS>(stage, v, gtv);
      bar();
      smem_load<P::AL1, P::AS>(stage, v, gtv);
      bar();  // every thread has read the stage: refill it
      if (gt == 0 && u + SA < total) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(u + SA);
      }
      butterflies<P::AL1, P::AB1, false>(v);
      if (r >= 1) mbar_wait_cta(&regionfree[i], (r - 1) & 1u);  // B(r-1, a) has been read
      const uint32_t a = c + i * G;
      if (r & 1u)
        store_global<P::AL1, P::AOutQ, false, Cache::kL2>(ws + ((uint64_t)a << 4), v, gtv, 1.0f);
      else
        store_global<P::AL1, P::AOutP, false, Cache::kL2>(ws + ((uint64_t)a << 14), v, gtv, 1.0f);
      if (i + 1 == nt) {  // this CTA's last A tile of row r: publish all nt of them
        asm volatile("fence.proxy.async.global;" ::: "memory");
        bar();
        if (gt == 0) red_release_add(&cnt[r], nt);
      }
    }
  } else {  // ---- B group
    const uint32_t gt = tid - NT;
    auto bar = [] { named_bar(2, NT); };
    uint64_t pol = 0;
    auto issue = [&](uint32_t u, bool wait) -> bool {
      const uint32_t r = u / nt, i = u - r * nt;
      if (i == 0) {
        if (ld_relaxed_u32(&cnt[r]) < P::NTILES) {
          if (!wait) return false;
          while (ld_relaxed_u32(&cnt[r]) < P::NTILES) __nanosleep(64);
        }
        (void)ld_acquire_gpu_u32(&cnt[r]);  // synchronizes with every A tile's release
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      mbar_expect_tx_cta(&fullB, TB);
      const uint32_t t = c + i * G;
      // both layouts through 64-byte-swizzling tensor maps (Q: the contiguous region as [4][256][16])
      if (r & 1u)
        tensor3_g2s(stageB, &tmapQ, 0, 0, (int)(4u * t), &fullB);
      else
        tensor4_g2s_hint(stageB, &tmapP, 0, (int)t, 0, 0, &fullB, pol);
      return true;
    };
    bool pending = false;
    if (gt == 0) {
      pol = l2_evict_normal_policy();
      pending = total > 0;
    }
    for (uint32_t u = 0, r = 0, i = 0; u < total; ++u, i = (i + 1 == nt) ? 0 : i + 1, r += (i == 0)) {
      if (pending) pending = !issue(u, true);
      uint32_t gtv = gt;
      asm volatile("mov.b32 %0, %1;" : "=r"(gtv) : "r"(gt));
      mbar_wait_cta(&fullB, u & 1u);
      // B(r, t)'s workspace bytes are in shared memory: A(r+1, t) may overwrite them.
      if (gt == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&regionfree[i])) : "memory");
      smem_load<P::BL0, P::BStage>(stageB, v, gtv);
      butterflies<P::BL0, P::BB0, false>(v);
      bar();  // every thread has read the stage (TMA's swizzle): rewrite it
      smem_store<P::BL0, P::BS>(stageB, v, gtv);
      bar();
      smem_load<P::BL1, P::BS>(stageB, v, gtv);
      bar();  // the stage is free: load the next B tile
      if (gt == 0 && u + 1 < total) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        pending = !issue(u + 1, false);
      }
      butterflies<P::BL1, P::BB1, false>(v);
      const uint32_t t = c + i * G;  // v bits = j4..j13 in order: natural position t << 4
      store_global<P::BL1, P::BOut, SCALE, Cache::kStream>(out + ((uint64_t)r << 24), v, gtv, scale, t << 4);
    }
  }
}

}  // namespace chwb
