// inst_f64_k4.cu — multi-pass (K4) kernels for double (one TU per dtype x regime).
#include "launch.cuh"

namespace chwb {
CHW_INSTANTIATE_K4(double)
}  // namespace chwb
