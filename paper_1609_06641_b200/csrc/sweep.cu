// sweep.cu — host launcher of K9, the single-HBM-pass m = 24 row sweep
// (sweep.cuh), in its own translation unit.
#include "launch.cuh"
#include "sweep.cuh"

namespace chwb {

namespace {
// Workspace as [4][256][1024][16] floats (addr bits 22..23, 14..21, 4..13,
// 0..3 of layout P), box {16, 1, 256, 4}: one B tile of a layout-P row.
chw_status sweep_tmap(float* ws, TmapParam* t, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  TmapEncodeFn fn = nullptr;
  if (chw_status s = tmap_encoder(&fn)) return s;
  const cuuint64_t dims[4] = {16, 1024, 256, 4};
  const cuuint64_t strides[3] = {64, (cuuint64_t)1 << 16, (cuuint64_t)1 << 24};
  const cuuint32_t box[4] = {16, 1, 256, 4};
  const cuuint32_t e[4] = {1, 1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(t), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ws, dims, strides, box, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHW_ERR_CUDA, "chw_forward: cuTensorMapEncodeTiled (m = 24 sweep) failed");
  return CHW_OK;
}

template <bool SCALE, bool SEQ>
chw_status launch_sweep_t(const float* in, float* out, void* ws, int64_t batch, float scale, cudaStream_t st) {
  using P = SweepF32M24;
  constexpr auto k = sweep_m24_kernel<SCALE, SEQ>;
  constexpr int smem = 3 * P::TILE * 4 + P::TILE * 2;  // two A stages, one B stage, B transpose buffer
  if (((uintptr_t)in | (uintptr_t)out | (uintptr_t)ws) & 15u)
    return fail(CHW_ERR_ARGUMENT, "chw_forward: buffers and workspace must be 16-byte aligned");
  if (batch > 0x7fffffffLL) return fail(CHW_ERR_UNSUPPORTED, "chw_forward: batch too large for the m = 24 sweep");
  if (chw_status s = prep_kernel<k>(smem)) return s;
  int dev = 0, sms = 0;
  if (chw_status s = current_device(&dev)) return s;
  CHW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = (unsigned)std::min<int>(sms, (int)P::NTILES);
  if ((P::NTILES + grid - 1) / grid > 8) return fail(CHW_ERR_UNSUPPORTED, "chw_forward: too few SMs for the sweep");
  float* w = static_cast<float*>(ws);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + ((size_t)64 << 20));
  TmapParam tm;
  if (chw_status s = sweep_tmap(w, &tm)) return s;
  CHW_CUDA(cudaMemsetAsync(cnt, 0, (size_t)batch * 4, st));
  // Co-residency of all CTAs is required (B tiles wait for A tiles of other
  // CTAs): cooperative launch, one CTA per SM.
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(2 * P::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CHW_CUDA(cudaLaunchKernelEx(&cfg, k, in, out, w, cnt, (uint32_t)batch, scale, tm));
  return check_launch("sweep_m24_kernel");
}
// K9n (natural order): layout-Q rows are contiguous 64 KiB regions, loaded as
// [4096][256][16] floats, box {16, 256, 4}; both maps swizzle 64-byte rows
// (SweepNatF32M24::BStage).
chw_status sweep_nat_tmap_q(float* ws, TmapParam* t) {
  TmapEncodeFn fn = nullptr;
  if (chw_status s = tmap_encoder(&fn)) return s;
  const cuuint64_t dims[3] = {16, 256, 4096};
  const cuuint64_t strides[2] = {64, (cuuint64_t)1 << 14};
  const cuuint32_t box[3] = {16, 256, 4};
  const cuuint32_t e[3] = {1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(t), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ws, dims, strides, box, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHW_ERR_CUDA, "chw_forward: cuTensorMapEncodeTiled (m = 24 natural sweep) failed");
  return CHW_OK;
}

template <bool SCALE>
chw_status launch_sweep_nat(const float* in, float* out, void* ws, int64_t batch, float scale, cudaStream_t st) {
  using P = SweepNatF32M24;
  constexpr auto k = sweep_nat_m24_kernel<SCALE>;
  constexpr int smem = 3 * P::TILE * 4;  // two A stages, one B stage (transposed in place)
  if (((uintptr_t)in | (uintptr_t)out | (uintptr_t)ws) & 15u)
    return fail(CHW_ERR_ARGUMENT, "chw_forward: buffers and workspace must be 16-byte aligned");
  if (batch > 0x7fffffffLL) return fail(CHW_ERR_UNSUPPORTED, "chw_forward: batch too large for the m = 24 sweep");
  if (chw_status s = prep_kernel<k>(smem)) return s;
  int dev = 0, sms = 0;
  if (chw_status s = current_device(&dev)) return s;
  CHW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = (unsigned)std::min<int>(sms, (int)P::NTILES);
  if ((P::NTILES + grid - 1) / grid > 8) return fail(CHW_ERR_UNSUPPORTED, "chw_forward: too few SMs for the sweep");
  float* w = static_cast<float*>(ws);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + ((size_t)64 << 20));
  TmapParam tp, tq;
  if (chw_status s = sweep_tmap(w, &tp, CU_TENSOR_MAP_SWIZZLE_64B)) return s;
  if (chw_status s = sweep_nat_tmap_q(w, &tq)) return s;
  CHW_CUDA(cudaMemsetAsync(cnt, 0, (size_t)batch * 4, st));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(2 * P::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CHW_CUDA(cudaLaunchKernelEx(&cfg, k, in, out, w, cnt, (uint32_t)batch, scale, tp, tq));
  return check_launch("sweep_nat_m24_kernel");
}
}  // namespace

chw_status launch_sweep_m24(bool scale_mode, const float* in, float* out, void* ws, int64_t batch, float scale,
                            cudaStream_t st, int order) {
  if (order == 1)  // natural
    return scale_mode ? launch_sweep_nat<true>(in, out, ws, batch, scale, st)
                      : launch_sweep_nat<false>(in, out, ws, batch, scale, st);
  if (order == 2)  // sequency
    return scale_mode ? launch_sweep_t<true, true>(in, out, ws, batch, scale, st)
                      : launch_sweep_t<false, true>(in, out, ws, batch, scale, st);
  return scale_mode ? launch_sweep_t<true, false>(in, out, ws, batch, scale, st)
                    : launch_sweep_t<false, false>(in, out, ws, batch, scale, st);
}

}  // namespace chwb

#if CHW_SWEEP_TRACE
extern "C" int chw_b200_debug_sweep_trace(void* dev_buf) {
  return (int)cudaMemcpyToSymbol(chwb::g_sweep_trace, &dev_buf, sizeof(void*));
}
#endif
