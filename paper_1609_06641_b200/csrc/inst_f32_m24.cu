// inst_f32_m24.cu — the f32 m = 24 schedules (split from inst_f32_k4.cu for build time).
#include "launch.cuh"

namespace chwb {
template chw_status launch_m<float, 24, Scaling::kDeferred>(const float*, float*, void*, int64_t, float, cudaStream_t);
template chw_status launch_m<float, 24, Scaling::kNone>(const float*, float*, void*, int64_t, float, cudaStream_t);
}  // namespace chwb
