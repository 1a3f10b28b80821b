// inst_f64_k1.cu — single-pass (K1) kernels for double (one TU per dtype x regime).
#include "launch.cuh"

namespace chwb {
CHW_INSTANTIATE_K1(double)
}  // namespace chwb
