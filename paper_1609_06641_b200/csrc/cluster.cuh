// cluster.cuh — K3: single-pass CHW for rows larger than one CTA's shared
// memory, using a thread-block cluster and distributed shared memory (DSMEM).
//
// f32, m = 16 (BASELINE cfg4): a 256 KiB row is spread over a 4-CTA cluster,
// 64 KiB per CTA (row element j, CTA rank r = j >> 14).  Per row:
//   1. each CTA loads its contiguous quarter (16-byte vectors) and butterflies
//      the 14 local bits: 6 in registers, one smem transpose, 6 in registers,
//      2 by warp shuffles;
//   2. cluster barrier; every thread writes its values with 16-byte DSMEM
//      stores into the CTA that owns their OUTPUT quarter — dyadic output
//      quarter q = (j0 << 1) | j1, which depends only on the two lowest bits,
//      so the destination is uniform per warp — at local index u = j >> 2;
//   3. cluster barrier; each CTA butterflies the two cross-CTA bits (u12, u13)
//      in registers and stores its contiguous 64 KiB output quarter.
// HBM sees exactly one read and one write per element; the exchange moves 3/4
// of the row SM-to-SM through DSMEM, not through L2 (DESIGN.md §4.1 explains
// why that matters: SM<->L2 bandwidth is only ~1.2x HBM on this part).
// All shared-memory accesses are bank-conflict free (tools/plan_check.py).
#pragma once

#include <cooperative_groups.h>

#include "plans.cuh"

namespace chwb {

__device__ __forceinline__ uint32_t cl_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Shared::cluster address of `local_addr` in CTA `rank` of this cluster.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
// 16-byte DSMEM store that completes 16 transaction bytes on the destination
// CTA's mbarrier (the destination waits on its own barrier; no cluster-wide
// release fence is needed).
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
      "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ void mbar_init_cl(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cl_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
                   cl_smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(cl_smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}

struct ClusterF32M16 {
  static constexpr int M = 16;
  static constexpr int CLUSTER = 4;
  static constexpr int NT = 256;
  static constexpr int LOCAL = 1 << 14;  // elements per CTA
  static constexpr int SMEM_BYTES = LOCAL * 4;
  // phase 1 (local bits j0..j13)
  using L0 = Layout<BL<0, 1, 10, 11, 12, 13>, BL<2, 3, 4, 5, 6, 7, 8, 9>>;
  using L1 = Layout<BL<2, 3, 4, 5, 6, 7>, BL<8, 9, 10, 11, 12, 13, 0, 1>>;
  using S1 = Swz<8, 0, 9, 1, 10, 2, 11, 3, 12, 4, 5, 0, 6, 1>;
  // phase 2 (u = j >> 2 | source rank << 12; butterflies on u12, u13)
  using L2 = Layout<BL<12, 13, 0, 1, 2, 3>, BL<11, 10, 9, 8, 7, 4, 5, 6>>;
  using S2 = Swz<6, 2, 7, 3, 8, 4, 9, 2, 10, 3, 11, 4>;
  struct Rev14 {
    CHW_HD static constexpr int pos(int k) { return 13 - k; }
  };
};

// XCH selects the exchange protocol (measured):
//   0: generic DSMEM stores, full cluster barrier before and after
//   1: generic DSMEM stores, relaxed barrier before, full barrier after
//   2: st.async into the destination's mbarrier, relaxed barrier before
template <bool SCALE, int XCH>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(256, 2)
    cluster_m16_kernel(const float* __restrict__ in, float* __restrict__ out, uint64_t rows, float scale) {
  using K = ClusterF32M16;
  namespace cg = cooperative_groups;
  extern __shared__ __align__(128) float buf[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t r = cl.block_rank();
  const uint64_t cid = blockIdx.x / K::CLUSTER;
  const uint64_t ncl = gridDim.x / K::CLUSTER;
  const uint32_t tid = threadIdx.x;
  const uint32_t w = tid >> 5;
  const uint32_t lane = tid & 31u;
  // In layout L1 the warp index bits are (j13, j0, j1): destination rank
  // (j0 << 1) | j1 is uniform per warp.
  const uint32_t rp = (((w >> 1) & 1u) << 1) | ((w >> 2) & 1u);
  __shared__ __align__(8) uint64_t xbar;  // exchange barrier: 64 KiB of st.async per row
  if (tid == 0) {
    mbar_init_cl(&xbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();  // barriers initialised cluster-wide before any remote complete_tx
  float* gbuf = cl.map_shared_rank(buf, rp);
  const uint32_t rbuf = mapa_u32(cl_smem_u32(buf), rp);
  const uint32_t rbar = mapa_u32(cl_smem_u32(&xbar), rp);
  const uint32_t xbase = K::S2::apply((lane << 6) | ((w & 1u) << 11) | (r << 12));
  float v[64];
  uint32_t parity = 0;
  for (uint64_t row = cid; row < rows; row += ncl, parity ^= 1u) {
    const float* src = in + (row << K::M) + (uint64_t)r * K::LOCAL;
    load_global<K::L0, IdMap, Cache::kStream>(src, v, tid);
    butterflies<K::L0, BL<0, 1, 10, 11, 12, 13>, false>(v);
    __syncthreads();  // this CTA's reads of buf for the previous row are done
    smem_store<K::L0, K::S1>(buf, v, tid);
    __syncthreads();
    smem_load<K::L1, K::S1>(buf, v, tid);
    butterflies<K::L1, BL<2, 3, 4, 5, 6, 7>, false>(v);
    shfl_butterfly<K::L1, 8, false>(v, tid);
    shfl_butterfly<K::L1, 9, false>(v, tid);
    if constexpr (XCH == 2) {
      if (tid == 0) mbar_arrive_expect_tx(&xbar, K::LOCAL * 4);
    }
    // Every CTA has finished reading its buf (the butterflies above consumed
    // all loaded values) before any peer writes into it.
    if constexpr (XCH == 0)
      cl.sync();
    else
      cluster_sync_relaxed();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const uint32_t a = xbase ^ (uint32_t)(q << 2);
      const float4 x = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      if constexpr (XCH == 2)
        st_async_v4(rbuf + a * 4u, x, rbar);
      else
        *reinterpret_cast<float4*>(gbuf + a) = x;
    }
    if constexpr (XCH == 2)
      mbar_wait_cluster(&xbar, parity);  // all 64 KiB of this CTA's quarter have landed
    else
      cl.sync();  // release/acquire: the exchange is visible
    smem_load<K::L2, K::S2>(buf, v, tid);
    butterflies<K::L2, BL<12, 13>, false>(v);
    store_global<K::L2, K::Rev14, SCALE, Cache::kStream>(out + (row << K::M) + (uint64_t)r * K::LOCAL, v, tid,
                                                         scale);
  }
  cl.sync();  // no CTA exits while a peer may still write into its shared memory
}



}  // namespace chwb
