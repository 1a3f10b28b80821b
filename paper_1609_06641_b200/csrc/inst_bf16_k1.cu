// inst_bf16_k1.cu — single-pass (K1) kernels for __nv_bfloat16 (one TU per dtype x regime).
#include "launch.cuh"

namespace chwb {
CHW_INSTANTIATE_K1(__nv_bfloat16)
}  // namespace chwb
