// launch.cuh — host-side launch templates shared by the per-dtype
// instantiation units (inst_*.cu).  Kernels for one dtype and one regime are
// compiled in their own translation unit so the build parallelises.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstdint>
#include <string>
#include <type_traits>

#include "../../include/chw_b200.h"
#include "chw_kernels.cuh"
#include "fused.cuh"
#include "pipelined.cuh"
#include "rowpipe.cuh"
#include "clusterm16.cuh"
#include "k1t.cuh"
#include "passtma.cuh"

namespace chwb {

constexpr int kMaxM = 30;  // 2^30 elements per row (8 GiB of f64)

// Defined in chw_b200.cu.
chw_status fail(chw_status s, const std::string& msg);
chw_status cuda_fail(cudaError_t e, const char* where);
chw_status current_device(int* dev);
void count_launch();

#define CHW_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

inline chw_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, what);
  count_launch();
  return CHW_OK;
}

// ---------------------------------------------------------------------------
// Persisting-L2 window for an L2-resident intermediate (the multi-phase
// schedules' workspace).  B200 sets aside up to
// cudaDevAttrMaxPersistingL2CacheSize (79 MiB measured) of the 126 MB L2 for
// "persisting" lines, which normal (streaming) lines cannot evict.  The
// launches that touch the workspace carry an access-policy window over it
// (hitProp Persisting, missProp Streaming) so the intermediate's lines stay
// in L2 while the input and output stream past, and are overwritten there
// instead of being written back.  OFF by default (CHW_B200_L2PERSIST=1 turns
// it on for A/B runs): measured, a carve-out with a 1 GiB window (K4T, 16-row
// chunks, hitRatio 0.08) cut cfg5 from 0.43 to 0.16 of HBM peak AND the same
// process's plain 1 GiB copy from 6.2 to 2.9 TB/s; a 1-row window (K4T,
// chunk 1) ran 272 vs 299 Gelem/s without it; K6 (cfg4, 37 MiB window)
// gained ~1.5 %.  DESIGN.md §4.3.
// ---------------------------------------------------------------------------
inline int l2_persist_mode() {
  static const int v = [] {
    const char* e = std::getenv("CHW_B200_L2PERSIST");
    return (e && e[0] >= '0' && e[0] <= '9') ? e[0] - '0' : 0;
  }();
  return v;
}
// Raise the device's persisting carve-out to at least `bytes` (capped at the
// device maximum) once; returns the carve-out in effect (0 = unavailable).
inline size_t ensure_persist_carveout(size_t bytes) {
  static std::atomic<size_t> have[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return 0;
  }
  size_t cur = have[dev].load(std::memory_order_acquire);
  if (cur >= bytes) return cur;
  int maxp = 0;
  if (cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess || maxp <= 0) {
    cudaGetLastError();
    return 0;
  }
  const size_t want = std::min<size_t>(bytes, (size_t)maxp);
  size_t now = 0;
  if (cudaDeviceGetLimit(&now, cudaLimitPersistingL2CacheSize) == cudaSuccess && now >= want) {
    have[dev].store(now, std::memory_order_release);
    return now;
  }
  if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  have[dev].store(want, std::memory_order_release);
  return want;
}
// Launch attribute list: an access-policy window over [base, base+bytes)
// when persistence is on and available, else none.
struct PersistWindow {
  cudaLaunchAttribute attr[1];
  unsigned n = 0;
  PersistWindow(const void* base, size_t bytes) {
    if (!l2_persist_mode() || !base || bytes == 0) return;
    const size_t carve = ensure_persist_carveout(bytes);
    if (carve == 0) return;
    int dev = 0, maxw = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess || maxw <= 0) {
      cudaGetLastError();
      return;
    }
    const size_t win = std::min<size_t>(bytes, (size_t)maxw);
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr[0].val.accessPolicyWindow.num_bytes = win;
    attr[0].val.accessPolicyWindow.hitRatio = std::min(1.0f, (float)((double)carve / (double)win));
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    n = 1;
  }
};
template <class... KArgs, class... Args>
chw_status launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     const PersistWindow& w, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = const_cast<cudaLaunchAttribute*>(w.attr);
  cfg.numAttrs = w.n;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernelEx");
  return CHW_OK;
}

template <auto Kern>
chw_status prep_kernel(int smem) {
  // One-time (per kernel, per device) opt-in above 48 KiB of dynamic shared memory.
  // (Static __shared__ counts against the 48 KiB default too, so opt in for
  // anything near it.)
  static std::atomic<uint64_t> done_mask{0};
  if (smem <= 32 * 1024) return CHW_OK;
  int dev = 0;
  if (chw_status s = current_device(&dev)) return s;
  const uint64_t bit = 1ull << dev;
  if (done_mask.load(std::memory_order_acquire) & bit) return CHW_OK;
  CHW_CUDA(cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  done_mask.fetch_or(bit, std::memory_order_acq_rel);
  return CHW_OK;
}

// K1T (k1t.cuh): TMA-fed single-pass kernel for f32 m = 12 (cfg2, default):
// 8-stage ring, 2 compute groups.  Same-box A/B: 95.3-95.9 %
// of HBM peak vs 90.7-91.2 % for the cp.async K1P it replaced (removed, with
// the other measured ring/group variants, in round 2).  K1W, a warp-per-row
// variant with all-vector accesses (8 instead of 14 instructions per element),
// measured the same throughput at higher SM clocks and was removed too
// (profiles/r02_ab_k1w.txt).
template <class Item, int TB, int S, int NG, bool SCALE>
chw_status launch_k1t_x(const typename Item::IO* in, typename Item::IO* out, int64_t tiles, float scale,
                        cudaStream_t st) {
  constexpr auto k = k1t_kernel<Item, TB, S, NG, SCALE>;
  constexpr int smem = S * Item::TILE * (int)sizeof(typename Item::IO) + NG * Item::TILE * 4;
  if (((uintptr_t)in | (uintptr_t)out) & 15u)
    return fail(CHW_ERR_ARGUMENT, "chw_forward: buffers must be 16-byte aligned");
  if (chw_status s = prep_kernel<k>(smem)) return s;
  int dev = 0, sms = 0;
  if (chw_status s = current_device(&dev)) return s;
  CHW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)sms);
  k<<<grid, NG * Item::L0::NT + 32, smem, st>>>(in, out, (uint64_t)tiles, scale);
  return check_launch("k1t_kernel");
}
template <bool SCALE>
chw_status launch_k1t(const float* in, float* out, int64_t batch, float scale, cudaStream_t st) {
  return launch_k1t_x<ItemF32M12, 12, 8, 2, SCALE>(in, out, batch, scale, st);
}

// Natural-order single pass (f2): the generic K1 plan with identity store map.
template <class T, int M, Scaling SC, class MapOut = IdMap>
chw_status launch_k1_nat(const T* in, T* out, int64_t batch, typename IoTraits<T>::C scale, cudaStream_t st) {
  using R = Regime<T>;
  constexpr int TB = M > R::TMIN ? M : R::TMIN;
  using Plan = GenericTilePlan<T, M, TB, R::EB, MapOut>;
  constexpr int ROWS_PER_TILE = 1 << (TB - M);
  const uint64_t full = (uint64_t)batch / ROWS_PER_TILE;
  const uint64_t tail_rows = (uint64_t)batch % ROWS_PER_TILE;
  if (full > 0) {
    constexpr auto k = k1_kernel<Plan, SC, false>;
    if (chw_status s = prep_kernel<k>(Plan::SMEM_BYTES)) return s;
    for (uint64_t t0 = 0; t0 < full; t0 += 0x7fffffffull) {
      const unsigned g = (unsigned)std::min<uint64_t>(full - t0, 0x7fffffffull);
      k<<<g, Plan::NT, Plan::SMEM_BYTES, st>>>(in, out, t0, scale, 0);
      if (chw_status s = check_launch("k1_kernel(natural)")) return s;
    }
  }
  if constexpr (TB > M) {
    if (tail_rows > 0) {
      constexpr auto k = k1_kernel<Plan, SC, true>;
      if (chw_status s = prep_kernel<k>(Plan::SMEM_BYTES)) return s;
      k<<<1, Plan::NT, Plan::SMEM_BYTES, st>>>(in, out, full, scale, (uint32_t)(tail_rows << M));
      if (chw_status s = check_launch("k1_kernel(natural tail)")) return s;
    }
  }
  return CHW_OK;
}
// Output order of the single-pass plan's store map: NATURAL = identity
// (fwht_natural), SEQUENCY = inverse Gray code of the dyadic position
// (apply_permutation(dyadic_to_sequency)) — both folded into the stores.
template <class T, Scaling SC, int M, int MHI>
chw_status dispatch_range_nat(int m, bool seq, const T* in, T* out, int64_t batch, typename IoTraits<T>::C scale,
                              cudaStream_t st) {
  if constexpr (M > MHI) {
    return fail(CHW_ERR_UNSUPPORTED, "chw_forward: unsupported length");
  } else {
    if (m == M) {
      if (seq) return launch_k1_nat<T, M, SC, SeqMap<RevMap<M>, M>>(in, out, batch, scale, st);
      return launch_k1_nat<T, M, SC>(in, out, batch, scale, st);
    }
    return dispatch_range_nat<T, SC, M + 1, MHI>(m, seq, in, out, batch, scale, st);
  }
}

template <class Plan, class T, int M, Scaling SC>
chw_status launch_k1_plan(const T* in, T* out, int64_t batch, typename IoTraits<T>::C scale, cudaStream_t st);

// Optional tensor-core block path for bf16 m = 7 (tc.cu; CHW_B200_TC=1).
bool tc_bf16_m7_enabled();
chw_status launch_tc_bf16_m7(bool scale_mode, const __nv_bfloat16* in, __nv_bfloat16* out, int64_t batch,
                             float scale, cudaStream_t st);

// Output-order variants of a plan are produced by swapping the output map.
template <class T, int M, Scaling SC>
chw_status launch_k1(const T* in, T* out, int64_t batch, typename IoTraits<T>::C scale,
                     cudaStream_t st) {
  if constexpr (std::is_same<T, float>::value && M == 12)
    return launch_k1t<SC == Scaling::kDeferred>(in, out, batch, scale, st);
  if constexpr (std::is_same<T, __nv_bfloat16>::value && M == 7)
    if (tc_bf16_m7_enabled()) return launch_tc_bf16_m7(SC == Scaling::kDeferred, in, out, batch, scale, st);
  // (f64 m = 10, cfg1: EB 3/4/5 x 1/2/4 rows per CTA measured within noise
  // of each other, 0.14-0.18 of HBM peak: a single 16 MiB wave is launch- and
  // latency-bound; profiles/r02_ab_cfg1.txt)
  return launch_k1_plan<typename K1Select<T, M>::Plan, T, M, SC>(in, out, batch, scale, st);
}

template <class Plan, class T, int M, Scaling SC>
chw_status launch_k1_plan(const T* in, T* out, int64_t batch, typename IoTraits<T>::C scale, cudaStream_t st) {
  constexpr int TB = Plan::kTB;
  constexpr int ROWS_PER_TILE = 1 << (TB - M);
  const uint64_t full = (uint64_t)batch / ROWS_PER_TILE;
  const uint64_t tail_rows = (uint64_t)batch % ROWS_PER_TILE;
  if (full > 0) {
    constexpr auto k = k1_kernel<Plan, SC, false>;
    if (chw_status s = prep_kernel<k>(Plan::SMEM_BYTES)) return s;
    for (uint64_t t0 = 0; t0 < full; t0 += 0x7fffffffull) {
      const unsigned g = (unsigned)std::min<uint64_t>(full - t0, 0x7fffffffull);
      k<<<g, Plan::NT, Plan::SMEM_BYTES, st>>>(in, out, t0, scale, 0);
      if (chw_status s = check_launch("k1_kernel")) return s;
    }
  }
  if (tail_rows > 0) {
    if constexpr (TB > M) {
      constexpr auto k = k1_kernel<Plan, SC, true>;
      if (chw_status s = prep_kernel<k>(Plan::SMEM_BYTES)) return s;
      k<<<1, Plan::NT, Plan::SMEM_BYTES, st>>>(in, out, full, scale,
                                               (uint32_t)(tail_rows << M));
      if (chw_status s = check_launch("k1_kernel(tail)")) return s;
    }
  }
  return CHW_OK;
}

template <class T, int M, Scaling SC, int p>
chw_status launch_k4_pass(const void* in, void* out, int64_t batch,
                          typename IoTraits<T>::C scale, cudaStream_t st) {
  using Sched = K4Sched<T, M>;
  using PassT = typename Sched::template Pass<p>;
  using MP = typename PassT::Plan;
  constexpr bool LAST = (p == Sched::NPASS - 1);
  constexpr auto k = pass_kernel<MP, SC, LAST && SC == Scaling::kDeferred>;
  if (chw_status s = prep_kernel<k>(MP::SMEM_BYTES)) return s;
  const uint64_t tiles = (uint64_t)batch << (M - PassT::TILE_BITS);
  if (tiles > 0x7fffffffull) return fail(CHW_ERR_UNSUPPORTED, "chw_forward: batch too large");
  k<<<(unsigned)tiles, MP::NT, MP::SMEM_BYTES, st>>>(
      static_cast<const typename MP::TIn*>(in), static_cast<typename MP::TOut*>(out), scale);
  return check_launch("pass_kernel");
}

template <class T, int M, Scaling SC, int p>
chw_status launch_k4_from(const T* in, T* out, void* ws, int64_t batch,
                          typename IoTraits<T>::C scale, cudaStream_t st) {
  using Sched = K4Sched<T, M>;
  constexpr int NP = Sched::NPASS;
  const void* src = (p == 0) ? static_cast<const void*>(in) : static_cast<const void*>(ws);
  void* dst = (p == NP - 1) ? static_cast<void*>(out) : ws;
  if (chw_status s = launch_k4_pass<T, M, SC, p>(src, dst, batch, scale, st)) return s;
  if constexpr (p + 1 < NP) return launch_k4_from<T, M, SC, p + 1>(in, out, ws, batch, scale, st);
  return CHW_OK;
}

// f32 m = 16 (cfg4): K6f, the per-CTA row pipeline (rowpipe.cuh).  The
// measured alternatives (K3 cluster/DSMEM 47 %, K5 fused dataflow 38-41 %,
// K6e one group per stream 55-60 %) were removed in round 2.

// K6 workspace: one row per CTA (one CTA per SM).
inline size_t rowpipe_workspace(int64_t batch) {
  if (batch <= 0) return 0;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(batch, (int64_t)sms);
  return (size_t)grid * ((size_t)1 << RowPipeF32M16<0>::M) * sizeof(float);
}

// Tensor maps over a K6 workspace of `ctas` rows (tile order in smem):
//   layout 0 column tile: [ctas*256][16][16] floats (W bits 8..15 + CTA, 4..7, 0..3), box {16, 1, 256};
//   layout 1 region tile: [ctas*16][W bits 4..7][W bits 8..11][W bits 0..3], box {16, 16, 16, 1}.
using TmapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline chw_status tmap_encoder(TmapEncodeFn* out) {
  static TmapEncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CHW_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      return fail(CHW_ERR_CUDA, "chw_forward: cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<TmapEncodeFn>(p);
  }
  *out = fn;
  return CHW_OK;
}
inline chw_status rowpipe_tmaps(void* ws, int ctas, TmapParam* t0, TmapParam* t1) {
  static_assert(sizeof(CUtensorMap) == sizeof(TmapParam), "tensor map size");
  TmapEncodeFn fn = nullptr;
  if (chw_status s = tmap_encoder(&fn)) return s;
  const cuuint64_t d0[3] = {16, 16, (cuuint64_t)ctas * 256};
  const cuuint64_t s0[2] = {64, 1024};
  const cuuint32_t b0[3] = {16, 1, 256};
  const cuuint32_t e[4] = {1, 1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(t0), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ws, d0, s0, b0, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHW_ERR_CUDA, "chw_forward: cuTensorMapEncodeTiled (layout 0) failed");
  const cuuint64_t d1[4] = {16, 16, 16, (cuuint64_t)ctas * 16};
  const cuuint64_t s1[3] = {1024, 64, 16384};
  const cuuint32_t b1[4] = {16, 16, 16, 1};
  r = fn(reinterpret_cast<CUtensorMap*>(t1), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ws, d1, s1, b1, e,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHW_ERR_CUDA, "chw_forward: cuTensorMapEncodeTiled (layout 1) failed");
  return CHW_OK;
}

template <bool SCALE, int SA, int SB, int HINT, int ORD = 0>
chw_status launch_rowpipe_ws4_m16_x(const float* in, float* out, void* ws, int64_t batch, float scale,
                                    cudaStream_t st) {
  using P = RowPipeF32M16<HINT, ORD>;
  constexpr auto k = rowpipe_ws4_kernel<P, SA, SB, SCALE>;
  if (((uintptr_t)in | (uintptr_t)out | (uintptr_t)ws) & 15u)
    return fail(CHW_ERR_ARGUMENT, "chw_forward: buffers and workspace must be 16-byte aligned");
  constexpr int smem = (SA + SB + 4) * P::TILE * 4;
  if (chw_status s = prep_kernel<k>(smem)) return s;
  int dev = 0, sms = 0;
  if (chw_status s = current_device(&dev)) return s;
  CHW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = (int)std::min<int64_t>(batch, (int64_t)sms);
  TmapParam t0, t1;
  if (chw_status s = rowpipe_tmaps(ws, grid, &t0, &t1)) return s;
  const PersistWindow win(ws, (size_t)grid << 18);  // one 256 KiB workspace row per CTA
  if (chw_status s = launch_ex(k, grid, 4 * P::NT + 64, smem, st, win, in, out, static_cast<float*>(ws),
                               (uint64_t)batch, scale, t0, t1))
    return s;
  return check_launch("rowpipe_ws4_kernel");
}

// K6f default: rings of 4 A stages and 6 B stages, two compute groups per
// stream, evict-first input / evict-last workspace hints.
template <bool SCALE>
chw_status launch_rowpipe_m16(const float* in, float* out, void* ws, int64_t batch, float scale,
                              cudaStream_t st) {
  return launch_rowpipe_ws4_m16_x<SCALE, 4, 6, 1>(in, out, ws, batch, scale, st);
}

// f32 m = 16 schedule: 'c' K10 cluster/DSMEM kernel (clusterm16.cuh), 'r' K6
// row pipeline (default).  K11, the row pipeline with 128-value threads (half
// the instructions, four shared-memory passes), measured +3 % under the soak
// and -13 % cold against K6 and was removed; so was K12, the same idea with
// four groups of 64-value threads and a 6 + 10 level split (+3.4 % soaked,
// -3..-10 % cold) (profiles/r02_ab_k11.txt).
inline char m16_mode() {
  static const char mode = [] {
    const char* e = std::getenv("CHW_B200_M16");
    return (e && e[0] == 'c') ? 'c' : 'r';
  }();
  return mode;
}
// K10: clusters of 4 CTAs, one row per cluster at a time, no workspace.
template <bool SCALE>
chw_status launch_cluster_m16(const float* in, float* out, int64_t batch, float scale, cudaStream_t st) {
  using P = ClusterF32M16;
  constexpr auto k = cluster_m16_kernel<SCALE>;
  if (((uintptr_t)in | (uintptr_t)out) & 15u)
    return fail(CHW_ERR_ARGUMENT, "chw_forward: buffers and workspace must be 16-byte aligned");
  if (batch > 0x7fffffffLL) return fail(CHW_ERR_UNSUPPORTED, "chw_forward: batch too large for the m = 16 cluster kernel");
  constexpr int smem = (2 * P::TILE + 2 * (P::CL - 1) * (P::TILE / P::CL)) * 4;  // 2 buffers + 2 x 3 blocks
  if (chw_status s = prep_kernel<k>(smem)) return s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P::CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(2 * P::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent grid: as many clusters as can be resident (or one per row)
  static std::atomic<int> max_clusters{0};
  int ncl = max_clusters.load();
  if (ncl <= 0) {
    cfg.gridDim = dim3(P::CL * 64);
    CHW_CUDA(cudaOccupancyMaxActiveClusters(&ncl, k, &cfg));
    if (ncl <= 0) return fail(CHW_ERR_RESOURCE, "chw_forward: no room for a 4-CTA cluster (m = 16)");
    max_clusters.store(ncl);
  }
  ncl = (int)std::min<int64_t>(ncl, batch);
  cfg.gridDim = dim3((unsigned)(P::CL * ncl));
  CHW_CUDA(cudaLaunchKernelEx(&cfg, k, in, out, (uint32_t)batch, scale));
  return check_launch("cluster_m16_kernel");
}

// m = 24 (cfg5).  K4T: two statically scheduled passes through an HBM
// intermediate in 16-row chunks (both passes TMA-fed).
constexpr int64_t kM24Chunk = 16;  // rows per chunk: 1 GiB intermediate
// K4T rows per chunk (CHW_B200_M24_CHUNK=1..16; default 16).
inline int64_t m24_chunk_rows() {
  static const int64_t v = [] {
    const char* e = std::getenv("CHW_B200_M24_CHUNK");
    const long x = e ? std::strtol(e, nullptr, 10) : 0;
    return (int64_t)((x >= 1 && x <= kM24Chunk) ? x : kM24Chunk);
  }();
  return v;
}
// f32 m = 24 schedule: 's' K9 row sweep (default), 't' K4T two-pass.  (K4P
// and the K5 dataflow kernels were measured slower and removed in round 2.)
inline char m24_mode() {
  static const char mode = [] {
    const char* e = std::getenv("CHW_B200_M24");
    return (e && e[0] == 't') ? 't' : 's';
  }();
  return mode;
}
// K9 workspace: one row (64 MiB, L2-resident) + one completion counter per row.
inline size_t sweep_m24_workspace(int64_t batch) {
  return ((size_t)64 << 20) + (((size_t)std::max<int64_t>(batch, 0) * 4 + 255) & ~(size_t)255);
}
// K9 launcher (sweep.cu, its own translation unit); order: 0 dyadic, 1 natural
// (K9n), 2 sequency — all folded into the sweep's stores.
chw_status launch_sweep_m24(bool scale_mode, const float* in, float* out, void* ws, int64_t batch, float scale,
                            cudaStream_t st, int order = 0);
// Natural (order 1) / sequency (order 2) folded into the f32 m = 16 (K6,
// inst_f32_m16.cu) store map.
chw_status launch_rowpipe_m16_ordered(int order, bool scale_mode, const float* in, float* out, void* ws,
                                      int64_t batch, float scale, cudaStream_t st);

// K4T (passtma.cuh): the K4P two-pass schedule fed by TMA, in-place tile
// transposes (3 tiles in flight per SM).  Same-box A/B: 42.8-42.9 % vs K4P
// 37.9-38.0 % of HBM peak (profiles/r01_ab_k4t.txt).
inline chw_status m24_mid_tmap(float* mid, int64_t rows, TmapParam* t) {
  TmapEncodeFn fn = nullptr;
  if (chw_status s = tmap_encoder(&fn)) return s;
  const cuuint64_t dims[5] = {8, 1024, 256, 8, (cuuint64_t)rows};
  const cuuint64_t strides[4] = {32, 32768, 8388608, 67108864};
  const cuuint32_t box[5] = {8, 1, 256, 8, 1};
  const cuuint32_t e[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(t), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, mid, dims, strides, box, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHW_ERR_CUDA, "chw_forward: cuTensorMapEncodeTiled (m = 24) failed");
  return CHW_OK;
}
template <bool SCALE>
chw_status launch_two_pass_tma_m24(const float* in, float* out, void* ws, int64_t batch, float scale,
                                   cudaStream_t st) {
  using P = PassTmaF32M24;
  constexpr int S = 3;
  constexpr int smem = S * P::TILE * 4;
  constexpr auto ka = pass_tma_kernel<P::ItemA, GeoA24, false, S, false>;
  constexpr auto kb = pass_tma_kernel<P::ItemB, GeoB24, true, S, SCALE>;
  if (((uintptr_t)in | (uintptr_t)out | (uintptr_t)ws) & 15u)
    return fail(CHW_ERR_ARGUMENT, "chw_forward: buffers and workspace must be 16-byte aligned");
  if (chw_status s = prep_kernel<ka>(smem)) return s;
  if (chw_status s = prep_kernel<kb>(smem)) return s;
  int dev = 0, sms = 0;
  if (chw_status s = current_device(&dev)) return s;
  CHW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float* mid = static_cast<float*>(ws);
  TmapParam none{};
  const int64_t chunk = m24_chunk_rows();
  const PersistWindow win(mid, (size_t)std::min<int64_t>(chunk, batch) << 26);
  for (int64_t r0 = 0; r0 < batch; r0 += chunk) {
    const int64_t rows = std::min<int64_t>(chunk, batch - r0);
    const uint64_t items = (uint64_t)rows * 1024;
    const unsigned grid = (unsigned)std::min<uint64_t>(items, (uint64_t)sms);
    if (chw_status s = launch_ex(ka, grid, P::NT + 32, smem, st, win, in + ((uint64_t)r0 << 24), mid, items, scale,
                                 none))
      return s;
    if (chw_status s = check_launch("pass_tma_kernel(A)")) return s;
    TmapParam tm;
    if (chw_status s = m24_mid_tmap(mid, rows, &tm)) return s;
    if (chw_status s = launch_ex(kb, grid, P::NT + 32, smem, st, win, (const float*)mid,
                                 out + ((uint64_t)r0 << 24), items, scale, tm))
      return s;
    if (chw_status s = check_launch("pass_tma_kernel(B)")) return s;
  }
  return CHW_OK;
}


template <class T, int MLO = Regime<T>::K1MAX + 1>
size_t k4_workspace_m(int m, int64_t batch, size_t inter) {
  if constexpr (MLO > kMaxM) {
    return 0;
  } else {
    if (m != MLO) return k4_workspace_m<T, MLO + 1>(m, batch, inter);
    if (batch <= 0) return 0;
    if constexpr (std::is_same<T, float>::value && MLO == 16) return rowpipe_workspace(batch);
    if constexpr (std::is_same<T, float>::value && MLO == 24) {
      if (m24_mode() == 's') return sweep_m24_workspace(batch);  // K9: one L2-resident row
      // K4T: 16-row intermediate (never less than the sweep needs: the fused
      // natural / sequency orders run on the sweep in either mode)
      return std::max((size_t)std::min<int64_t>(batch, kM24Chunk) << 26, sweep_m24_workspace(batch));
    }
    return (size_t)batch * ((size_t)1 << m) * inter;
  }
}

template <class T, int M, Scaling SC>
chw_status launch_m(const T* in, T* out, void* ws, int64_t batch, typename IoTraits<T>::C scale,
                    cudaStream_t st) {
  if constexpr (M <= Regime<T>::K1MAX) {
    return launch_k1<T, M, SC>(in, out, batch, scale, st);
  } else if constexpr (std::is_same<T, float>::value && M == 16) {
    if (m16_mode() == 'c') return launch_cluster_m16<SC == Scaling::kDeferred>(in, out, batch, scale, st);
    return launch_rowpipe_m16<SC == Scaling::kDeferred>(in, out, ws, batch, scale, st);
  } else if constexpr (std::is_same<T, float>::value && M == 24) {
    if (m24_mode() == 's') return launch_sweep_m24(SC == Scaling::kDeferred, in, out, ws, batch, scale, st);
    return launch_two_pass_tma_m24<SC == Scaling::kDeferred>(in, out, ws, batch, scale, st);
  } else {
    return launch_k4_from<T, M, SC, 0>(in, out, ws, batch, scale, st);
  }
}

template <class T, Scaling SC, int M, int MHI>
chw_status dispatch_range(int m, const T* in, T* out, void* ws, int64_t batch,
                          typename IoTraits<T>::C scale, cudaStream_t st) {
  if constexpr (M > MHI) {
    return fail(CHW_ERR_UNSUPPORTED, "chw_forward: unsupported length");
  } else {
    if (m == M) return launch_m<T, M, SC>(in, out, ws, batch, scale, st);
    return dispatch_range<T, SC, M + 1, MHI>(m, in, out, ws, batch, scale, st);
  }
}

template <class T, int M = 0>
const char* plan_name_m(int m) {
  if constexpr (M > kMaxM) {
    return "unsupported";
  } else {
    if (m != M) return plan_name_m<T, M + 1>(m);
    if constexpr (M <= Regime<T>::K1MAX) {
      if constexpr (std::is_same<T, float>::value && M == 12) return "k1t-tma";
      if constexpr (std::is_same<T, __nv_bfloat16>::value && M == 7)
        if (tc_bf16_m7_enabled()) return "k7tc-tcgen05";
      return K1Select<T, M>::kTuned ? "k1-tuned" : "k1-generic";
    } else if constexpr (std::is_same<T, float>::value && M == 16) {
      return m16_mode() == 'c' ? "k10-cluster-dsmem" : "k6-rowpipe";
    } else if constexpr (std::is_same<T, float>::value && M == 24) {
      return m24_mode() == 's' ? "k9-row-sweep" : "k4t-two-pass-tma";
    } else {
      static const std::string s = "k4-multipass:" + std::to_string(K4Sched<T, M>::NPASS);
      return s.c_str();
    }
  }
}



// Entry points per dtype, instantiated in inst_<dtype>_<regime>.cu:
//   forward_k1<T>: m in [0, K1MAX];  forward_k4<T>: m in (K1MAX, kMaxM].
template <class T>
chw_status forward_k1(int m, bool scaled_mode, const T* in, T* out, int64_t batch,
                      typename IoTraits<T>::C scale, cudaStream_t st);
template <class T>
chw_status forward_k1_natural(int m, bool scaled_mode, bool seq, const T* in, T* out, int64_t batch,
                              typename IoTraits<T>::C scale, cudaStream_t st);
template <class T>
chw_status forward_k4(int m, bool scaled_mode, const T* in, T* out, void* ws, int64_t batch,
                      typename IoTraits<T>::C scale, cudaStream_t st);
template <class T>
const char* plan_name(int m);
template <class T>
size_t k4_workspace(int m, int64_t batch);

// scaled_mode: Orthonormal.  f64 scales per butterfly (bit-exact with the
// reference); f32/bf16 defer to one multiply; int64 is never scaled.
template <class T>
struct ModeScaling {
  static constexpr Scaling kOrtho = std::is_same<T, double>::value ? Scaling::kPerStage
                                                                   : Scaling::kDeferred;
};

#define CHW_INSTANTIATE_K1(T)                                                                 \
  template <>                                                                                  \
  chw_status forward_k1<T>(int m, bool scaled_mode, const T* in, T* out, int64_t batch,         \
                           typename IoTraits<T>::C scale, cudaStream_t st) {                    \
    if constexpr (!std::is_same<T, long long>::value) {                                         \
      if (scaled_mode)                                                                          \
        return dispatch_range<T, ModeScaling<T>::kOrtho, 0, Regime<T>::K1MAX>(                  \
            m, in, out, nullptr, batch, scale, st);                                             \
    }                                                                                           \
    return dispatch_range<T, Scaling::kNone, 0, Regime<T>::K1MAX>(m, in, out, nullptr, batch,    \
                                                                   scale, st);                   \
  }                                                                                             \
  template <>                                                                                  \
  chw_status forward_k1_natural<T>(int m, bool scaled_mode, bool seq, const T* in, T* out, int64_t batch, \
                                   typename IoTraits<T>::C scale, cudaStream_t st) {            \
    if constexpr (!std::is_same<T, long long>::value) {                                         \
      if (scaled_mode)                                                                          \
        return dispatch_range_nat<T, ModeScaling<T>::kOrtho, 0, Regime<T>::K1MAX>(m, seq, in, out, \
                                                                                  batch, scale, st); \
    }                                                                                           \
    return dispatch_range_nat<T, Scaling::kNone, 0, Regime<T>::K1MAX>(m, seq, in, out, batch, scale, st); \
  }

#define CHW_INSTANTIATE_K4(T)                                                                  \
  template <>                                                                                   \
  chw_status forward_k4<T>(int m, bool scaled_mode, const T* in, T* out, void* ws,              \
                           int64_t batch, typename IoTraits<T>::C scale, cudaStream_t st) {     \
    if constexpr (!std::is_same<T, long long>::value) {                                         \
      if (scaled_mode)                                                                          \
        return dispatch_range<T, ModeScaling<T>::kOrtho, Regime<T>::K1MAX + 1, kMaxM>(          \
            m, in, out, ws, batch, scale, st);                                                  \
    }                                                                                           \
    return dispatch_range<T, Scaling::kNone, Regime<T>::K1MAX + 1, kMaxM>(m, in, out, ws, batch, \
                                                                          scale, st);           \
  }                                                                                             \
  template <>                                                                                   \
  const char* plan_name<T>(int m) {                                                             \
    return plan_name_m<T>(m);                                                                   \
  }                                                                                             \
  template <>                                                                                   \
  size_t k4_workspace<T>(int m, int64_t batch) {                                                \
    return k4_workspace_m<T>(m, batch, sizeof(typename IoTraits<T>::C));                        \
  }

}  // namespace chwb
