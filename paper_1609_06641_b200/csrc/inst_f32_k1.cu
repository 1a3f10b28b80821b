// inst_f32_k1.cu — single-pass (K1) kernels for float (one TU per dtype x regime).
#include "launch.cuh"

namespace chwb {
CHW_INSTANTIATE_K1(float)
}  // namespace chwb
