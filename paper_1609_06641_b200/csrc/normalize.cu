// normalize.cu — device path of chw::normalize_inplace
// (proj/include/chw/transforms.hpp:202-210): y = x * c, c = 1 / sqrt(2^m),
// applied to `batch` rows of n = 2^m elements.  c is computed on the host with
// the reference's own expression, and every element sees exactly one
// IEEE multiply (DMUL for f64, no contraction), so the f64 result is
// bit-identical to the reference loop.  HBM-bound: 16 B/elem (f64) in one
// read + one write; grid = a multiple of the SM count, 16-byte vectors.
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "../../include/chw_b200.h"
#include "launch.cuh"

namespace chwb {
namespace {

template <class V, class S>
__global__ void __launch_bounds__(256) scale_kernel(V* __restrict__ x, uint64_t nvec, S c) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    V v = x[i];
    if constexpr (sizeof(V) == 16 && sizeof(S) == 8) {
      v.x = __dmul_rn(v.x, c);
      v.y = __dmul_rn(v.y, c);
    } else {
      v.x = __fmul_rn(v.x, c);
      v.y = __fmul_rn(v.y, c);
      v.z = __fmul_rn(v.z, c);
      v.w = __fmul_rn(v.w, c);
    }
    x[i] = v;
  }
}

template <class E, class S>
__global__ void __launch_bounds__(256) scale_tail_kernel(E* __restrict__ x, uint64_t n, S c) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * c;
}

}  // namespace

chw_status normalize_device(void* x, chw_dtype dtype, uint64_t total, double c, cudaStream_t st) {
  if (total == 0) return CHW_OK;
  int dev = 0, sms = 0;
  if (chw_status s = current_device(&dev)) return s;
  CHW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const uint64_t cap = (uint64_t)sms * 8;  // 8 resident 256-thread CTAs per SM
  if (dtype == CHW_F64) {
    const uint64_t nv = total / 2;
    if (nv) {
      const unsigned g = (unsigned)std::min<uint64_t>((nv + 255) / 256, cap);
      scale_kernel<double2, double><<<g, 256, 0, st>>>(static_cast<double2*>(x), nv, c);
      if (chw_status s = check_launch("scale_kernel<f64>")) return s;
    }
    if (total & 1) {
      scale_tail_kernel<double, double><<<1, 32, 0, st>>>(static_cast<double*>(x) + 2 * nv, 1, c);
      if (chw_status s = check_launch("scale_tail_kernel<f64>")) return s;
    }
    return CHW_OK;
  }
  if (dtype == CHW_F32) {
    const float cf = (float)c;
    const uint64_t nv = total / 4;
    if (nv) {
      const unsigned g = (unsigned)std::min<uint64_t>((nv + 255) / 256, cap);
      scale_kernel<float4, float><<<g, 256, 0, st>>>(static_cast<float4*>(x), nv, cf);
      if (chw_status s = check_launch("scale_kernel<f32>")) return s;
    }
    if (total & 3) {
      scale_tail_kernel<float, float><<<1, 32, 0, st>>>(static_cast<float*>(x) + 4 * nv, total & 3, cf);
      if (chw_status s = check_launch("scale_tail_kernel<f32>")) return s;
    }
    return CHW_OK;
  }
  return fail(CHW_ERR_UNSUPPORTED, "normalize: dtype not supported (f64, f32)");
}

}  // namespace chwb

extern "C" chw_status chw_b200_normalize(void* x, chw_dtype dtype, int64_t batch, uint64_t n, int m,
                                         void* stream) {
  // transforms.hpp:203-206: the length must equal 2^m (same wording).
  if (m < 0 || m > 62 || n != (uint64_t{1} << m))
    return chwb::fail(CHW_ERR_LENGTH, "normalize: signal length " + std::to_string(n) +
                                          " does not match level " + std::to_string(m));
  if (batch < 0) return chwb::fail(CHW_ERR_ARGUMENT, "normalize: negative batch");
  if (batch == 0) return CHW_OK;
  if (!x) return chwb::fail(CHW_ERR_ARGUMENT, "normalize: null buffer");
  if ((uintptr_t)x & 15u) return chwb::fail(CHW_ERR_ARGUMENT, "normalize: buffer must be 16-byte aligned");
  const double c = 1.0 / std::sqrt(std::ldexp(1.0, m));  // transforms.hpp:207
  return chwb::normalize_device(x, dtype, (uint64_t)batch * n, c, static_cast<cudaStream_t>(stream));
}
