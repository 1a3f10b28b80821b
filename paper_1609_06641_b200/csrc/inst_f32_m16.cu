// inst_f32_m16.cu — the f32 m = 16 schedules (split from inst_f32_k4.cu for build time).
#include "launch.cuh"

namespace chwb {
template chw_status launch_m<float, 16, Scaling::kDeferred>(const float*, float*, void*, int64_t, float, cudaStream_t);
template chw_status launch_m<float, 16, Scaling::kNone>(const float*, float*, void*, int64_t, float, cudaStream_t);
chw_status launch_rowpipe_m16_ordered(int order, bool scale_mode, const float* in, float* out, void* ws,
                                      int64_t batch, float scale, cudaStream_t st) {
  if (order == 1)
    return scale_mode ? launch_rowpipe_ws4_m16_x<true, 4, 6, 1, 1>(in, out, ws, batch, scale, st)
                      : launch_rowpipe_ws4_m16_x<false, 4, 6, 1, 1>(in, out, ws, batch, scale, st);
  return scale_mode ? launch_rowpipe_ws4_m16_x<true, 4, 6, 1, 2>(in, out, ws, batch, scale, st)
                    : launch_rowpipe_ws4_m16_x<false, 4, 6, 1, 2>(in, out, ws, batch, scale, st);
}
}  // namespace chwb
