// inst_i64_k4.cu — multi-pass (K4) kernels for long long (one TU per dtype x regime).
#include "launch.cuh"

namespace chwb {
using i64_t = long long;
CHW_INSTANTIATE_K4(i64_t)
}  // namespace chwb
