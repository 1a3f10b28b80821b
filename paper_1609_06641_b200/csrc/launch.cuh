// launch.cuh — host-side launch templates shared by the per-dtype
// instantiation units (inst_*.cu).  Kernels for one dtype and one regime are
// compiled in their own translation unit so the build parallelises.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <string>
#include <type_traits>

#include "../../include/chw_b200.h"
#include "chw_kernels.cuh"

namespace chwb {

constexpr int kMaxM = 30;  // 2^30 elements per row (8 GiB of f64)

// Defined in chw_b200.cu.
chw_status fail(chw_status s, const std::string& msg);
chw_status cuda_fail(cudaError_t e, const char* where);
chw_status current_device(int* dev);
void count_launch();

#define CHW_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

inline chw_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, what);
  count_launch();
  return CHW_OK;
}

template <auto Kern>
chw_status prep_kernel(int smem) {
  // One-time (per kernel, per device) opt-in above 48 KiB of dynamic shared memory.
  static std::atomic<uint64_t> done_mask{0};
  if (smem <= 48 * 1024) return CHW_OK;
  int dev = 0;
  if (chw_status s = current_device(&dev)) return s;
  const uint64_t bit = 1ull << dev;
  if (done_mask.load(std::memory_order_acquire) & bit) return CHW_OK;
  CHW_CUDA(cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  done_mask.fetch_or(bit, std::memory_order_acq_rel);
  return CHW_OK;
}

// Output-order variants of a plan are produced by swapping the output map.
template <class T, int M, Scaling SC>
chw_status launch_k1(const T* in, T* out, int64_t batch, typename IoTraits<T>::C scale,
                     cudaStream_t st) {
  using Plan = typename K1Select<T, M>::Plan;
  constexpr int TB = Plan::kTB;
  constexpr int ROWS_PER_TILE = 1 << (TB - M);
  const uint64_t full = (uint64_t)batch / ROWS_PER_TILE;
  const uint64_t tail_rows = (uint64_t)batch % ROWS_PER_TILE;
  if (full > 0) {
    constexpr auto k = k1_kernel<Plan, SC, false>;
    if (chw_status s = prep_kernel<k>(Plan::SMEM_BYTES)) return s;
    for (uint64_t t0 = 0; t0 < full; t0 += 0x7fffffffull) {
      const unsigned g = (unsigned)std::min<uint64_t>(full - t0, 0x7fffffffull);
      k<<<g, Plan::NT, Plan::SMEM_BYTES, st>>>(in, out, t0, scale, 0);
      if (chw_status s = check_launch("k1_kernel")) return s;
    }
  }
  if (tail_rows > 0) {
    if constexpr (TB > M) {
      constexpr auto k = k1_kernel<Plan, SC, true>;
      if (chw_status s = prep_kernel<k>(Plan::SMEM_BYTES)) return s;
      k<<<1, Plan::NT, Plan::SMEM_BYTES, st>>>(in, out, full, scale,
                                               (uint32_t)(tail_rows << M));
      if (chw_status s = check_launch("k1_kernel(tail)")) return s;
    }
  }
  return CHW_OK;
}

template <class T, int M, Scaling SC, int p>
chw_status launch_k4_pass(const void* in, void* out, int64_t batch,
                          typename IoTraits<T>::C scale, cudaStream_t st) {
  using Sched = K4Sched<T, M>;
  using PassT = typename Sched::template Pass<p>;
  using MP = typename PassT::Plan;
  constexpr bool LAST = (p == Sched::NPASS - 1);
  constexpr auto k = pass_kernel<MP, SC, LAST && SC == Scaling::kDeferred>;
  if (chw_status s = prep_kernel<k>(MP::SMEM_BYTES)) return s;
  const uint64_t tiles = (uint64_t)batch << (M - PassT::TILE_BITS);
  if (tiles > 0x7fffffffull) return fail(CHW_ERR_UNSUPPORTED, "chw_forward: batch too large");
  k<<<(unsigned)tiles, MP::NT, MP::SMEM_BYTES, st>>>(
      static_cast<const typename MP::TIn*>(in), static_cast<typename MP::TOut*>(out), scale);
  return check_launch("pass_kernel");
}

template <class T, int M, Scaling SC, int p>
chw_status launch_k4_from(const T* in, T* out, void* ws, int64_t batch,
                          typename IoTraits<T>::C scale, cudaStream_t st) {
  using Sched = K4Sched<T, M>;
  constexpr int NP = Sched::NPASS;
  const void* src = (p == 0) ? static_cast<const void*>(in) : static_cast<const void*>(ws);
  void* dst = (p == NP - 1) ? static_cast<void*>(out) : ws;
  if (chw_status s = launch_k4_pass<T, M, SC, p>(src, dst, batch, scale, st)) return s;
  if constexpr (p + 1 < NP) return launch_k4_from<T, M, SC, p + 1>(in, out, ws, batch, scale, st);
  return CHW_OK;
}

template <class T, int M, Scaling SC>
chw_status launch_m(const T* in, T* out, void* ws, int64_t batch, typename IoTraits<T>::C scale,
                    cudaStream_t st) {
  if constexpr (M <= Regime<T>::K1MAX) {
    return launch_k1<T, M, SC>(in, out, batch, scale, st);
  } else {
    return launch_k4_from<T, M, SC, 0>(in, out, ws, batch, scale, st);
  }
}

template <class T, Scaling SC, int M, int MHI>
chw_status dispatch_range(int m, const T* in, T* out, void* ws, int64_t batch,
                          typename IoTraits<T>::C scale, cudaStream_t st) {
  if constexpr (M > MHI) {
    return fail(CHW_ERR_UNSUPPORTED, "chw_forward: unsupported length");
  } else {
    if (m == M) return launch_m<T, M, SC>(in, out, ws, batch, scale, st);
    return dispatch_range<T, SC, M + 1, MHI>(m, in, out, ws, batch, scale, st);
  }
}

template <class T, int M = 0>
const char* plan_name_m(int m) {
  if constexpr (M > kMaxM) {
    return "unsupported";
  } else {
    if (m != M) return plan_name_m<T, M + 1>(m);
    if constexpr (M <= Regime<T>::K1MAX) {
      return K1Select<T, M>::kTuned ? "k1-tuned" : "k1-generic";
    } else {
      static const std::string s = "k4-multipass:" + std::to_string(K4Sched<T, M>::NPASS);
      return s.c_str();
    }
  }
}


// Entry points per dtype, instantiated in inst_<dtype>_<regime>.cu:
//   forward_k1<T>: m in [0, K1MAX];  forward_k4<T>: m in (K1MAX, kMaxM].
template <class T>
chw_status forward_k1(int m, bool scaled_mode, const T* in, T* out, int64_t batch,
                      typename IoTraits<T>::C scale, cudaStream_t st);
template <class T>
chw_status forward_k4(int m, bool scaled_mode, const T* in, T* out, void* ws, int64_t batch,
                      typename IoTraits<T>::C scale, cudaStream_t st);
template <class T>
const char* plan_name(int m);

// scaled_mode: Orthonormal.  f64 scales per butterfly (bit-exact with the
// reference); f32/bf16 defer to one multiply; int64 is never scaled.
template <class T>
struct ModeScaling {
  static constexpr Scaling kOrtho = std::is_same<T, double>::value ? Scaling::kPerStage
                                                                   : Scaling::kDeferred;
};

#define CHW_INSTANTIATE_K1(T)                                                                 \
  template <>                                                                                  \
  chw_status forward_k1<T>(int m, bool scaled_mode, const T* in, T* out, int64_t batch,         \
                           typename IoTraits<T>::C scale, cudaStream_t st) {                    \
    if constexpr (!std::is_same<T, long long>::value) {                                         \
      if (scaled_mode)                                                                          \
        return dispatch_range<T, ModeScaling<T>::kOrtho, 0, Regime<T>::K1MAX>(                  \
            m, in, out, nullptr, batch, scale, st);                                             \
    }                                                                                           \
    return dispatch_range<T, Scaling::kNone, 0, Regime<T>::K1MAX>(m, in, out, nullptr, batch,    \
                                                                   scale, st);                   \
  }

#define CHW_INSTANTIATE_K4(T)                                                                  \
  template <>                                                                                   \
  chw_status forward_k4<T>(int m, bool scaled_mode, const T* in, T* out, void* ws,              \
                           int64_t batch, typename IoTraits<T>::C scale, cudaStream_t st) {     \
    if constexpr (!std::is_same<T, long long>::value) {                                         \
      if (scaled_mode)                                                                          \
        return dispatch_range<T, ModeScaling<T>::kOrtho, Regime<T>::K1MAX + 1, kMaxM>(          \
            m, in, out, ws, batch, scale, st);                                                  \
    }                                                                                           \
    return dispatch_range<T, Scaling::kNone, Regime<T>::K1MAX + 1, kMaxM>(m, in, out, ws, batch, \
                                                                          scale, st);           \
  }                                                                                             \
  template <>                                                                                   \
  const char* plan_name<T>(int m) {                                                             \
    return plan_name_m<T>(m);                                                                   \
  }

}  // namespace chwb
