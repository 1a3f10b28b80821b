// inst_i64_k1.cu — single-pass (K1) kernels for long long (one TU per dtype x regime).
#include "launch.cuh"

namespace chwb {
using i64_t = long long;
CHW_INSTANTIATE_K1(i64_t)
}  // namespace chwb
