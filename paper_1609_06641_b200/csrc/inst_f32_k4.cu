// inst_f32_k4.cu — multi-pass (K4) kernels for float (one TU per dtype x regime).
// The m = 16 and m = 24 schedules are instantiated in their own units
// (inst_f32_m16.cu, inst_f32_m24.cu) so the build parallelises.
#include "launch.cuh"

namespace chwb {
#define CHW_F32_EXTERN(M)                                                                                    \
  extern template chw_status launch_m<float, M, Scaling::kDeferred>(const float*, float*, void*, int64_t, float, \
                                                                    cudaStream_t);                           \
  extern template chw_status launch_m<float, M, Scaling::kNone>(const float*, float*, void*, int64_t, float,     \
                                                                cudaStream_t);
CHW_F32_EXTERN(16)
CHW_F32_EXTERN(24)
CHW_INSTANTIATE_K4(float)
}  // namespace chwb
