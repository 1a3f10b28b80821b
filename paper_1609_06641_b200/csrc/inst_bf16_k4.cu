// inst_bf16_k4.cu — multi-pass (K4) kernels for __nv_bfloat16 (one TU per dtype x regime).
#include "launch.cuh"

namespace chwb {
CHW_INSTANTIATE_K4(__nv_bfloat16)
}  // namespace chwb
