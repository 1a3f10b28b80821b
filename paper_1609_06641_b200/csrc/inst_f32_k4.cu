// inst_f32_k4.cu — multi-pass (K4) kernels for float (one TU per dtype x regime).
#include "launch.cuh"

namespace chwb {
CHW_INSTANTIATE_K4(float)
}  // namespace chwb
