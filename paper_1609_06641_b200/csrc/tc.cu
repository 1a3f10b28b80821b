// tc.cu — K7TC: the optional tensor-core block path of north_star item (3)
// for the short-row bf16 config (cfg3: rows of n = 2^7, bf16 in/out, fp32
// accumulation).
//
// A row's dyadic WHT is one dense product y = s * x * H^T with the 128 x 128
// +-1 matrix H[i][j] = (-1)^popcount(rev_7(i) & j) (the
// reference builds the same matrix densely in oracle.hpp:50-69,
// hadamard_dyadic_dense).  A batch is then a plain TN GEMM
//   D[rows x 128] = X[rows x 128] . H^T      (K = 128, both operands K-major)
// which tcgen05 runs at M = 128 rows per instruction group:
//   * one persistent CTA per SM walks 128-row tiles of X;
//   * warp 0 lane 0: TMA producer (two 64 x 128 SWIZZLE_128B boxes per tile
//     into a 4-stage ring; H is loaded once per CTA the same way);
//   * warp 1: allocates 256 TMEM columns (two 128 x 128 fp32 accumulators);
//     its lane 0 issues the 8 tcgen05.mma (kind::f16, 128 x 128 x 16) per
//     tile and commits them to the stage's `empty` and the accumulator's
//     `full` mbarriers;
//   * warps 2-5 (TMEM lane quarters 2, 3, 0, 1): epilogue — tcgen05.ld the
//     thread's row (128 fp32 columns), scale once, round to bf16 once, stage
//     the row in shared memory in the output tensor map's SWIZZLE_128B layout
//     (two staging buffers), and one thread TMA-stores the 128 x 128 bf16 tile.
// The products are exact (+-1 weights), the sums fp32 in the tensor core, so
// the result matches the fp32 shuffle path's error budget (one bf16 rounding).
// Output orders are the rows of H: dyadic here (natural / sequency would be a
// row permutation of H, not built).  Default for bf16 m = 7 dyadic (it beats
// the K1 shuffle kernel by 2.6 % in a cold ncu launch and ties it in the
// sustained bench, at higher clocks); CHW_B200_TC=0 selects K1.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "launch.cuh"

namespace chwb {
namespace {

constexpr int kTcRows = 128;                 // rows per tile (UMMA M)
constexpr int kTcN = 128;                    // row length (UMMA N = K = 128)
constexpr int kTcStages = 4;
constexpr uint32_t kTileBytes = kTcRows * kTcN * 2;  // 32 KiB of bf16
constexpr uint32_t kHalfBytes = kTileBytes / 2;      // one 64-column SWIZZLE_128B box

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(su32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load2(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store2(const void* tmap, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
               "r"(su32(src)), "r"(x), "r"(y)
               : "memory");
}
// K-major SWIZZLE_128B UMMA shared-memory descriptor (canonical
// ((8,m),(T,2)):((8T,SBO),(1,T)): SBO = 1024 B between 8-row groups, LBO = 1
// (unused for swizzled K-major), version 1 (Blackwell), layout type 2).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Instruction descriptor: D f32, A/B bf16, both K-major, N = 128, M = 128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                            ((uint32_t)(kTcRows >> 4) << 24);

template <bool SCALE>
__global__ void __launch_bounds__(192, 1)
    tc_bf16_m7_kernel(const __grid_constant__ TmapParam tmx, const __grid_constant__ TmapParam tmh,
                      const __grid_constant__ TmapParam tmy, uint32_t ntiles, float scale) {
  extern __shared__ __align__(1024) unsigned char smem_tc[];
  // 1024-byte aligned base (SWIZZLE_128B atoms)
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_tc) + 1023) &
                                                         ~(uintptr_t)1023);
  unsigned char* ring = base;                                // kTcStages x 32 KiB
  unsigned char* hmat = ring + kTcStages * kTileBytes;       // 32 KiB
  unsigned char* ostages = hmat + kTileBytes;                // 2 x 32 KiB output staging
  __shared__ __align__(8) uint64_t full[kTcStages], empty[kTcStages], hfull, tfull[2], tempty[2], ofree[2];
  __shared__ uint32_t tmem_base_s;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const uint32_t nmine = c < ntiles ? (ntiles - 1 - c) / G + 1 : 0;
  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    mb_init(&hfull, 1);
    for (int a = 0; a < 2; ++a) {
      mb_init(&tfull[a], 1);
      mb_init(&tempty[a], 4);  // one arrival per epilogue warp
    }
    mb_init(&ofree[0], 1);
    mb_init(&ofree[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 256 columns = two 128 x 128 fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tmem_base_s))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {  // ---- TMA producer
    if (lane == 0) {
      mb_expect_tx(&hfull, kTileBytes);
      tma_load2(hmat, &tmh, 0, 0, &hfull);
      tma_load2(hmat + kHalfBytes, &tmh, 64, 0, &hfull);
      for (uint32_t u = 0; u < nmine; ++u) {
        const int s = (int)(u % kTcStages);
        if (u >= (uint32_t)kTcStages) mb_wait(&empty[s], ((u / kTcStages) - 1) & 1u);
        const int row0 = (int)((c + u * G) * kTcRows);
        unsigned char* st = ring + s * kTileBytes;
        mb_expect_tx(&full[s], kTileBytes);
        tma_load2(st, &tmx, 0, row0, &full[s]);
        tma_load2(st + kHalfBytes, &tmx, 64, row0, &full[s]);
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer
    if (lane == 0) {
      mb_wait(&hfull, 0);
      const uint32_t hb = su32(hmat);
      for (uint32_t u = 0; u < nmine; ++u) {
        const int s = (int)(u % kTcStages);
        const uint32_t acc = u & 1u;
        mb_wait(&full[s], (u / kTcStages) & 1u);
        if (u >= 2) mb_wait(&tempty[acc], ((u / 2) - 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ab = su32(ring + s * kTileBytes);
        const uint32_t d = tmem + acc * kTcN;
#pragma unroll
        for (int k = 0; k < kTcN / 16; ++k) {
          const uint32_t off = (uint32_t)(k >> 2) * kHalfBytes + (uint32_t)(k & 3) * 32u;
          const uint64_t da = umma_desc_sw128(ab + off);
          const uint64_t db = umma_desc_sw128(hb + off);
          const uint32_t accum = k > 0 ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
              "l"(da), "l"(db), "r"(kIdesc), "r"(accum)
              : "memory");
        }
        // stage free once these MMAs have read it; accumulator ready for the epilogue
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         su32(&empty[s]))
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         su32(&tfull[acc]))
                     : "memory");
      }
    }
  } else {  // ---- epilogue warps 2..5: TMEM lane quarter q = warp % 4
    const uint32_t q = warp & 3u;
    const uint32_t row = q * 32u + lane;  // tile row = TMEM lane
    for (uint32_t u = 0; u < nmine; ++u) {
      const uint32_t acc = u & 1u;
      mb_wait(&tfull[acc], (u / 2) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[kTcN];
#pragma unroll
      for (int cblk = 0; cblk < kTcN / 32; ++cblk) {
        const uint32_t ta = tmem + ((q * 32u) << 16) + acc * kTcN + (uint32_t)cblk * 32u;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(r[cblk * 32 + 0]), "=r"(r[cblk * 32 + 1]), "=r"(r[cblk * 32 + 2]), "=r"(r[cblk * 32 + 3]),
              "=r"(r[cblk * 32 + 4]), "=r"(r[cblk * 32 + 5]), "=r"(r[cblk * 32 + 6]), "=r"(r[cblk * 32 + 7]),
              "=r"(r[cblk * 32 + 8]), "=r"(r[cblk * 32 + 9]), "=r"(r[cblk * 32 + 10]), "=r"(r[cblk * 32 + 11]),
              "=r"(r[cblk * 32 + 12]), "=r"(r[cblk * 32 + 13]), "=r"(r[cblk * 32 + 14]), "=r"(r[cblk * 32 + 15]),
              "=r"(r[cblk * 32 + 16]), "=r"(r[cblk * 32 + 17]), "=r"(r[cblk * 32 + 18]), "=r"(r[cblk * 32 + 19]),
              "=r"(r[cblk * 32 + 20]), "=r"(r[cblk * 32 + 21]), "=r"(r[cblk * 32 + 22]), "=r"(r[cblk * 32 + 23]),
              "=r"(r[cblk * 32 + 24]), "=r"(r[cblk * 32 + 25]), "=r"(r[cblk * 32 + 26]), "=r"(r[cblk * 32 + 27]),
              "=r"(r[cblk * 32 + 28]), "=r"(r[cblk * 32 + 29]), "=r"(r[cblk * 32 + 30]), "=r"(r[cblk * 32 + 31])
            : "r"(ta)
            : "memory");
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mb_arrive(&tempty[acc]);  // accumulator may be overwritten
      // Output staging buffer u % 2 must have been read by tile u-2's TMA store.
      unsigned char* ostage = ostages + (u & 1u) * kTileBytes;
      if (u >= 2) mb_wait(&ofree[u & 1u], ((u / 2) - 1) & 1u);
      // Row `row` -> output staging in SWIZZLE_128B layout: half h holds
      // columns 64h..64h+63 as 128-byte rows, 16-byte chunk j of row r at
      // chunk j ^ (r & 7).
#pragma unroll
      for (int ch = 0; ch < kTcN / 8; ++ch) {  // 16 chunks of 8 bf16
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float a = __uint_as_float(r[ch * 8 + 2 * e]);
          float b = __uint_as_float(r[ch * 8 + 2 * e + 1]);
          if (SCALE) {
            a *= scale;
            b *= scale;
          }
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
          w[e] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        const uint32_t h = (uint32_t)ch >> 3, j = (uint32_t)ch & 7u;
        unsigned char* dst = ostage + h * kHalfBytes + row * 128u + ((j ^ (row & 7u)) << 4);
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == 2 && lane == 0) {
        const int row0 = (int)((c + u * G) * kTcRows);
        tma_store2(&tmy, ostage, 0, row0);
        tma_store2(&tmy, ostage + kHalfBytes, 64, row0);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (u >= 1) {  // tile u-1's store has read its staging buffer
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          mb_arrive(&ofree[(u - 1) & 1u]);
        }
      }
    }
    if (warp == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

// H[i][j] = (-1)^popcount(rev_7(i) & j) as bf16 (+-1 exactly).
__global__ void tc_build_h_kernel(__nv_bfloat16* h) {
  const uint32_t i = blockIdx.x, j = threadIdx.x;
  const uint32_t ri = __brev(i) >> (32 - 7);
  h[i * kTcN + j] = __float2bfloat16_rn((__popc(ri & j) & 1) ? -1.0f : 1.0f);
}

chw_status tc_tmap(void* ptr, uint64_t rows, bool store, TmapParam* t) {
  TmapEncodeFn fn = nullptr;
  if (chw_status s = tmap_encoder(&fn)) return s;
  const cuuint64_t dims[2] = {(cuuint64_t)kTcN, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)kTcN * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)kTcRows};
  const cuuint32_t e[2] = {1, 1};
  (void)store;
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(t), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHW_ERR_CUDA, "chw_forward: cuTensorMapEncodeTiled (tensor-core path) failed");
  return CHW_OK;
}

// Per-device H matrix (built once).
__nv_bfloat16* g_h[64] = {};
std::mutex g_h_mu;

chw_status tc_h(int dev, cudaStream_t st, __nv_bfloat16** out) {
  std::lock_guard<std::mutex> lk(g_h_mu);
  if (!g_h[dev]) {
    void* p = nullptr;
    CHW_CUDA(cudaMalloc(&p, kTcN * kTcN * 2));
    tc_build_h_kernel<<<kTcN, kTcN, 0, st>>>(static_cast<__nv_bfloat16*>(p));
    if (chw_status s = check_launch("tc_build_h_kernel")) return s;
    CHW_CUDA(cudaStreamSynchronize(st));
    g_h[dev] = static_cast<__nv_bfloat16*>(p);
  }
  *out = g_h[dev];
  return CHW_OK;
}

template <bool SCALE>
chw_status launch_tc_t(const __nv_bfloat16* in, __nv_bfloat16* out, int64_t batch, float scale, cudaStream_t st) {
  constexpr auto k = tc_bf16_m7_kernel<SCALE>;
  constexpr int smem = (kTcStages + 3) * (int)kTileBytes + 1024;
  if (((uintptr_t)in | (uintptr_t)out) & 15u)
    return fail(CHW_ERR_ARGUMENT, "chw_forward: buffers must be 16-byte aligned");
  if (chw_status s = prep_kernel<k>(smem)) return s;
  int dev = 0, sms = 0;
  if (chw_status s = current_device(&dev)) return s;
  CHW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  __nv_bfloat16* h = nullptr;
  if (chw_status s = tc_h(dev, st, &h)) return s;
  TmapParam tx, th, ty;
  if (chw_status s = tc_tmap(const_cast<__nv_bfloat16*>(in), (uint64_t)batch, false, &tx)) return s;
  if (chw_status s = tc_tmap(h, kTcN, false, &th)) return s;
  if (chw_status s = tc_tmap(out, (uint64_t)batch, true, &ty)) return s;
  const uint64_t ntiles = ((uint64_t)batch + kTcRows - 1) / kTcRows;
  if (ntiles > 0xffffffffull) return fail(CHW_ERR_UNSUPPORTED, "chw_forward: batch too large");
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sms);
  k<<<grid, 192, smem, st>>>(tx, th, ty, (uint32_t)ntiles, scale);
  return check_launch("tc_bf16_m7_kernel");
}

}  // namespace

// bf16 m = 7 (cfg3) dyadic runs through the tensor-core path by default;
// CHW_B200_TC=0 selects the K1 shuffle kernel.  A/B (profiles/r02_ab_tc.txt,
// r02_ncu_cfg3_{k1,tc}.json): sustained bench 0.842 / 0.841 vs 0.844 / 0.844
// of HBM peak (both HBM-bound; the TC path at 1912-1965 MHz vs 1725 MHz under
// sw_power_cap), single cold launch 85.0 us vs 87.2 us, issue slots 18 % vs
// 60 %, tensor pipe 22 %, DRAM bytes equal (algorithmic).
bool tc_bf16_m7_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CHW_B200_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

chw_status launch_tc_bf16_m7(bool scale_mode, const __nv_bfloat16* in, __nv_bfloat16* out, int64_t batch,
                             float scale, cudaStream_t st) {
  return scale_mode ? launch_tc_t<true>(in, out, batch, scale, st) : launch_tc_t<false>(in, out, batch, scale, st);
}

}  // namespace chwb
