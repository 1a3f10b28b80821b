// haar.cu — batched Haar wavelet transform Psi_m on the GPU.
//
// Replaces chw::haar_forward_inplace (proj/include/chw/transforms.hpp:49-80):
// for len = n, n/2, ..., 2 the pairs (2i, 2i+1) of the current smooth prefix
// give s = (a+b)k, d = (a-b)k (k = kInvSqrt2 in Orthonormal mode, 1 otherwise,
// transforms.hpp:62-70); d goes to position len/2 + i, s to position i.  The
// output row is [s, d_coarsest(1), ..., d_finest(n/2)].  Every operation is the
// reference's, in the same order, so f64 results are bit-exact.
//
// Rows with n <= kSmemMax run all levels in one CTA per row out of shared
// memory (one HBM read and write per element).  Longer rows first run global
// "level" kernels (each halves the smooth prefix, ping-ponging it through the
// workspace) until the prefix fits, then finish in shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "launch.cuh"

namespace chwb {
namespace {

template <class T>
struct HaarOps;
template <>
struct HaarOps<double> {
  __device__ static void bf(double a, double b, bool ortho, double& s, double& d) {
    s = __dadd_rn(a, b);
    d = __dsub_rn(a, b);
    if (ortho) {
      s = __dmul_rn(s, kInvSqrt2);
      d = __dmul_rn(d, kInvSqrt2);
    }
  }
};
template <>
struct HaarOps<float> {
  __device__ static void bf(float a, float b, bool ortho, float& s, float& d) {
    s = __fadd_rn(a, b);
    d = __fsub_rn(a, b);
    if (ortho) {
      s = __fmul_rn(s, (float)kInvSqrt2);
      d = __fmul_rn(d, (float)kInvSqrt2);
    }
  }
};
template <>
struct HaarOps<long long> {
  __device__ static void bf(long long a, long long b, bool, long long& s, long long& d) {
    s = a + b;
    d = a - b;
  }
};

constexpr int kSmemMaxBytes = 64 * 1024;  // smooth prefix handled in shared memory

// One CTA per row: levels len = n0 .. 2 on a prefix of length n0 held in smem.
// `src` holds the prefix (row stride src_stride), results go to `dst` rows
// (row stride dst_stride; d at [len/2, len), final s at [0]).
template <class T>
__global__ void haar_smem_kernel(const T* __restrict__ src, int64_t src_stride, T* __restrict__ dst,
                                 int64_t dst_stride, uint32_t n0, bool ortho) {
  extern __shared__ __align__(16) unsigned char hsm[];
  T* a = reinterpret_cast<T*>(hsm);
  T* b = a + n0;
  const uint64_t row = blockIdx.x;
  const T* s_in = src + row * src_stride;
  T* out = dst + row * dst_stride;
  for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) a[i] = s_in[i];
  __syncthreads();
  T* cur = a;
  T* nxt = b;
  for (uint32_t len = n0; len >= 2; len >>= 1) {
    const uint32_t half = len >> 1;
    for (uint32_t i = threadIdx.x; i < half; i += blockDim.x) {
      T s, d;
      HaarOps<T>::bf(cur[2 * i], cur[2 * i + 1], ortho, s, d);
      nxt[i] = s;
      out[half + i] = d;
    }
    __syncthreads();
    T* t = cur;
    cur = nxt;
    nxt = t;
  }
  if (threadIdx.x == 0) out[0] = cur[0];
}

// One level over all rows: pairs of the smooth prefix `src` (length len) ->
// smooth `s_out` (len/2) and details at dst[row][len/2 + i].
template <class T>
__global__ void haar_level_kernel(const T* __restrict__ src, int64_t src_stride, T* __restrict__ s_out,
                                  int64_t s_stride, T* __restrict__ dst, int64_t dst_stride, uint32_t len,
                                  uint64_t rows, bool ortho) {
  const uint32_t half = len >> 1;
  const uint64_t total = rows * half;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = t / half;
    const uint32_t i = (uint32_t)(t - row * half);
    T s, d;
    HaarOps<T>::bf(src[row * src_stride + 2 * i], src[row * src_stride + 2 * i + 1], ortho, s, d);
    s_out[row * s_stride + i] = s;
    dst[row * dst_stride + half + i] = d;
  }
}

// ---------------------------------------------------------------------------
// Inverse (transforms.hpp:85-120): for len = 2..n, x[2i], x[2i+1] from the
// smooth prefix s (length len/2) and the details d = x[len/2 + i]:
//   float Orthonormal: (s+d)k, (s-d)k;  float Unnormalized: (s+d)/2, (s-d)/2;
//   int64: sum = s+d must be even (else StructureError), sum/2, (s-d)/2.
// ---------------------------------------------------------------------------
template <class T>
struct InvOps;
template <>
struct InvOps<double> {
  __device__ static void op(double s, double d, bool ortho, double& a, double& b, int*) {
    if (ortho) {
      a = __dmul_rn(__dadd_rn(s, d), kInvSqrt2);
      b = __dmul_rn(__dsub_rn(s, d), kInvSqrt2);
    } else {
      a = __ddiv_rn(__dadd_rn(s, d), 2.0);
      b = __ddiv_rn(__dsub_rn(s, d), 2.0);
    }
  }
};
template <>
struct InvOps<float> {
  __device__ static void op(float s, float d, bool ortho, float& a, float& b, int*) {
    if (ortho) {
      a = __fmul_rn(__fadd_rn(s, d), (float)kInvSqrt2);
      b = __fmul_rn(__fsub_rn(s, d), (float)kInvSqrt2);
    } else {
      a = __fdiv_rn(__fadd_rn(s, d), 2.0f);
      b = __fdiv_rn(__fsub_rn(s, d), 2.0f);
    }
  }
};
template <>
struct InvOps<long long> {
  __device__ static void op(long long s, long long d, bool, long long& a, long long& b, int* err) {
    const long long sum = s + d;
    if (sum & 1) atomicExch(err, 1);
    a = sum / 2;
    b = (s - d) / 2;
  }
};

// One CTA per row, levels len = 2..n0 on the prefix x[0..n0) held in smem.
template <class T>
__global__ void haar_inv_smem_kernel(const T* __restrict__ src, int64_t src_stride, T* __restrict__ dst,
                                     int64_t dst_stride, uint32_t n0, bool ortho, int* err) {
  extern __shared__ __align__(16) unsigned char hsm[];
  T* x = reinterpret_cast<T*>(hsm);  // original prefix (s0 and the details)
  T* p = x + n0;                     // smooth ping
  T* q = p + n0;                     // smooth pong
  const uint64_t row = blockIdx.x;
  const T* in = src + row * src_stride;
  T* out = dst + row * dst_stride;
  for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) x[i] = in[i];
  __syncthreads();
  if (threadIdx.x == 0) p[0] = x[0];
  __syncthreads();
  T* cur = p;
  T* nxt = q;
  for (uint32_t len = 2; len <= n0; len <<= 1) {
    const uint32_t half = len >> 1;
    T* o = (len == n0) ? nullptr : nxt;
    for (uint32_t i = threadIdx.x; i < half; i += blockDim.x) {
      T a, b;
      InvOps<T>::op(cur[i], x[half + i], ortho, a, b, err);
      if (o) {
        o[2 * i] = a;
        o[2 * i + 1] = b;
      } else {
        out[2 * i] = a;
        out[2 * i + 1] = b;
      }
    }
    __syncthreads();
    T* t = cur;
    cur = nxt;
    nxt = t;
  }
}

// One level over all rows: smooth s (len/2) + details d_src[len/2 + i] -> dst (len).
template <class T>
__global__ void haar_inv_level_kernel(const T* __restrict__ s, int64_t s_stride, const T* __restrict__ d_src,
                                      int64_t d_stride, int64_t d_off, T* __restrict__ dst, int64_t dst_stride,
                                      uint32_t len, uint64_t rows, bool ortho, int* err) {
  const uint32_t half = len >> 1;
  const uint64_t total = rows * half;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = t / half;
    const uint32_t i = (uint32_t)(t - row * half);
    T a, b;
    InvOps<T>::op(s[row * s_stride + i], d_src[row * d_stride + d_off + i], ortho, a, b, err);
    dst[row * dst_stride + 2 * i] = a;
    dst[row * dst_stride + 2 * i + 1] = b;
  }
}

template <class T>
chw_status haar_inv_impl(const T* in, T* out, int64_t batch, uint64_t n, bool ortho, void* ws, int* err,
                         cudaStream_t st) {
  if (n == 1) {
    if (in != out) CHW_CUDA(cudaMemcpyAsync(out, in, (size_t)batch * sizeof(T), cudaMemcpyDeviceToDevice, st));
    return CHW_OK;
  }
  const uint64_t smem_max = kSmemMaxBytes / (3 * sizeof(T));
  uint64_t n0 = 1;
  while (n0 * 2 <= n && n0 * 2 <= smem_max) n0 *= 2;
  const bool big = n0 < n;
  T* bufs[2] = {static_cast<T*>(ws), static_cast<T*>(ws) + (size_t)batch * (n / 2)};
  T* dcopy = static_cast<T*>(ws) + 2 * (size_t)batch * (n / 2);  // in-place: top-level details
  const T* dsrc = in;
  if (big && in == out) {
    CHW_CUDA(cudaMemcpy2DAsync(dcopy, (n / 2) * sizeof(T), in + n / 2, n * sizeof(T), (n / 2) * sizeof(T),
                               (size_t)batch, cudaMemcpyDeviceToDevice, st));
  }
  // Levels 2..n0 in shared memory.
  T* first_dst = big ? bufs[0] : out;
  const int64_t first_stride = big ? (int64_t)n0 : (int64_t)n;
  const int smem = (int)(3 * n0 * sizeof(T));
  if (smem > 48 * 1024)
    CHW_CUDA(cudaFuncSetAttribute(haar_inv_smem_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int threads = (int)std::min<uint64_t>(256, std::max<uint64_t>(32, n0 / 2));
  for (int64_t r0 = 0; r0 < batch; r0 += 0x7fffffff) {
    const unsigned g = (unsigned)std::min<int64_t>(batch - r0, 0x7fffffff);
    haar_inv_smem_kernel<T><<<g, threads, smem, st>>>(in + r0 * (int64_t)n, (int64_t)n,
                                                       first_dst + r0 * first_stride, first_stride, (uint32_t)n0,
                                                       ortho, err);
    if (chw_status s = check_launch("haar_inv_smem_kernel")) return s;
  }
  // Larger levels through global memory.
  const T* s = bufs[0];
  int64_t s_stride = (int64_t)n0;
  int which = 1;
  for (uint64_t len = 2 * n0; len <= n; len <<= 1) {
    const bool last = (len == n);
    T* dst = last ? out : bufs[which];
    const int64_t dst_stride = last ? (int64_t)n : (int64_t)len;
    const T* d = (last && in == out) ? dcopy : dsrc;
    const int64_t d_stride = (last && in == out) ? (int64_t)(n / 2) : (int64_t)n;
    const int64_t d_off = (last && in == out) ? 0 : (int64_t)(len / 2);
    const uint64_t total = (uint64_t)batch * (len / 2);
    const unsigned grid = (unsigned)std::min<uint64_t>((total + 255) / 256, 148ull * 16);
    haar_inv_level_kernel<T><<<grid, 256, 0, st>>>(s, s_stride, d, d_stride, d_off, dst, dst_stride,
                                                    (uint32_t)len, (uint64_t)batch, ortho, err);
    if (chw_status r = check_launch("haar_inv_level_kernel")) return r;
    s = dst;
    s_stride = dst_stride;
    which ^= 1;
  }
  return CHW_OK;
}

template <class T>
chw_status haar_impl(const T* in, T* out, int64_t batch, uint64_t n, bool ortho, void* ws, cudaStream_t st) {
  if (n == 1) {
    if (in != out) CHW_CUDA(cudaMemcpyAsync(out, in, (size_t)batch * sizeof(T), cudaMemcpyDeviceToDevice, st));
    return CHW_OK;
  }
  const uint64_t smem_max = kSmemMaxBytes / (2 * sizeof(T));  // prefix + ping-pong half
  const T* src = in;
  int64_t src_stride = (int64_t)n;
  uint64_t len = n;
  T* bufs[2] = {static_cast<T*>(ws), static_cast<T*>(ws) + (size_t)batch * (n / 2)};
  int which = 0;
  if (len > smem_max && in == out) {
    // In place: the first level may not overwrite unread input, so it writes
    // its details to the workspace and they are copied into place after.
    const uint64_t half = len / 2;
    const uint64_t total = (uint64_t)batch * half;
    const unsigned grid = (unsigned)std::min<uint64_t>((total + 255) / 256, 148ull * 16);
    haar_level_kernel<T><<<grid, 256, 0, st>>>(src, src_stride, bufs[0], (int64_t)half, bufs[1] - half,
                                                (int64_t)half, (uint32_t)len, (uint64_t)batch, ortho);
    if (chw_status s = check_launch("haar_level_kernel")) return s;
    CHW_CUDA(cudaMemcpy2DAsync(out + half, n * sizeof(T), bufs[1], half * sizeof(T), half * sizeof(T),
                               (size_t)batch, cudaMemcpyDeviceToDevice, st));
    src = bufs[0];
    src_stride = (int64_t)half;
    len = half;
    which = 1;
  }
  while (len > smem_max) {
    T* s_out = bufs[which];
    const uint64_t total = (uint64_t)batch * (len / 2);
    const unsigned grid = (unsigned)std::min<uint64_t>((total + 255) / 256, 148ull * 16);
    haar_level_kernel<T><<<grid, 256, 0, st>>>(src, src_stride, s_out, (int64_t)(len / 2), out, (int64_t)n,
                                                (uint32_t)len, (uint64_t)batch, ortho);
    if (chw_status s = check_launch("haar_level_kernel")) return s;
    src = s_out;
    src_stride = (int64_t)(len / 2);
    len >>= 1;
    which ^= 1;
  }
  const int smem = (int)(len * sizeof(T) + (len / 2) * sizeof(T));
  if (smem > 48 * 1024) {
    CHW_CUDA(cudaFuncSetAttribute(haar_smem_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  const int threads = (int)std::min<uint64_t>(256, std::max<uint64_t>(32, len / 2));
  for (int64_t r0 = 0; r0 < batch; r0 += 0x7fffffff) {
    const unsigned g = (unsigned)std::min<int64_t>(batch - r0, 0x7fffffff);
    haar_smem_kernel<T><<<g, threads, smem, st>>>(src + r0 * src_stride, src_stride, out + r0 * (int64_t)n,
                                                   (int64_t)n, (uint32_t)len, ortho);
    if (chw_status s = check_launch("haar_smem_kernel")) return s;
  }
  return CHW_OK;
}

// ---------------------------------------------------------------------------
// Haar-Walsh map (transforms.hpp:187-198): a dyadic WHT of every scale block
// [2^j, 2^(j+1)), j = 1..m-1.  The blocks below 2^K of a row (K <= 13 or 14,
// whatever fits 64 KiB of shared memory) are done by ONE kernel, one CTA per
// row: level t = 0..K-2 combines (i, i | 2^t) for every i >= 2^(t+1) with bit
// t clear — block j takes part in levels t < j, the reference's level order —
// with the reference's per-butterfly scaling, and the store applies each
// block's own bit reversal.  One HBM read and write of the prefix instead of a
// gather, a transform and a scatter per block.
// ---------------------------------------------------------------------------
template <class T>
struct HwIo {
  using C = T;
  __device__ static C ld(const T* p) { return *p; }
  __device__ static void st(T* p, C v) { *p = v; }
};
template <>
struct HwIo<__nv_bfloat16> {
  using C = float;
  __device__ static float ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  __device__ static void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

template <class T>
__global__ void haar_walsh_smem_kernel(T* __restrict__ x, int64_t stride, uint32_t K, bool ortho) {
  using C = typename HwIo<T>::C;
  extern __shared__ __align__(16) unsigned char hw_smem[];
  C* s = reinterpret_cast<C*>(hw_smem);
  T* row = x + (int64_t)blockIdx.x * stride;
  const uint32_t n0 = 1u << K;
  for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) s[i] = HwIo<T>::ld(row + i);
  __syncthreads();
  for (uint32_t t = 0; t + 1 < K; ++t) {
    for (uint32_t p = threadIdx.x; p < n0 / 2; p += blockDim.x) {
      const uint32_t i = ((p >> t) << (t + 1)) | (p & ((1u << t) - 1u));
      if (i >= (2u << t)) {
        C a, b;
        HaarOps<C>::bf(s[i], s[i | (1u << t)], ortho, a, b);
        s[i] = a;
        s[i | (1u << t)] = b;
      }
    }
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) {
    uint32_t src = i;
    if (i >= 4) {  // blocks 0, 1 (one element) and j = 1 (two elements) are their own reversal
      const uint32_t j = 31u - (uint32_t)__clz((int)i);
      src = (1u << j) | (__brev(i - (1u << j)) >> (32u - j));
    }
    HwIo<T>::st(row + i, s[src]);
  }
}

template <class T>
chw_status haar_walsh_prefix_impl(T* x, int64_t batch, uint64_t n, int K, bool ortho, cudaStream_t st) {
  const int smem = (int)(((size_t)1 << K) * sizeof(typename HwIo<T>::C));
  if (smem > 48 * 1024)
    CHW_CUDA(cudaFuncSetAttribute(haar_walsh_smem_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int threads = (int)std::min<uint64_t>(512, std::max<uint64_t>(32, ((uint64_t)1 << K) / 2));
  for (int64_t r0 = 0; r0 < batch; r0 += 0x7fffffff) {
    const unsigned g = (unsigned)std::min<int64_t>(batch - r0, 0x7fffffff);
    haar_walsh_smem_kernel<T><<<g, threads, smem, st>>>(x + r0 * (int64_t)n, (int64_t)n, (uint32_t)K, ortho);
    if (chw_status s = check_launch("haar_walsh_smem_kernel")) return s;
  }
  return CHW_OK;
}

}  // namespace

size_t haar_inverse_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n) {
  const size_t es = (dtype == CHW_F32) ? 4 : 8;
  const uint64_t smem_max = kSmemMaxBytes / (3 * es);
  if (n <= smem_max || batch <= 0) return 256;  // error flag
  return 256 + 3 * (size_t)batch * (n / 2) * es;
}

chw_status haar_inverse_device(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                               chw_mode mode, void* ws, cudaStream_t st) {
  // ws layout: [0, 256) error flag, then the level buffers.
  int* err = static_cast<int*>(ws);
  void* bufs = static_cast<char*>(ws) + 256;
  CHW_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  const bool ortho = (mode == CHW_ORTHONORMAL);
  chw_status s = CHW_OK;
  switch (dtype) {
    case CHW_F64:
      s = haar_inv_impl<double>(static_cast<const double*>(in), static_cast<double*>(out), batch, n, ortho, bufs,
                                err, st);
      break;
    case CHW_F32:
      s = haar_inv_impl<float>(static_cast<const float*>(in), static_cast<float*>(out), batch, n, ortho, bufs,
                               err, st);
      break;
    case CHW_I64:
      s = haar_inv_impl<long long>(static_cast<const long long*>(in), static_cast<long long*>(out), batch, n,
                                   false, bufs, err, st);
      if (s == CHW_OK) {
        // The reference throws StructureError on an odd pair sum
        // (transforms.hpp:110-114): the integer inverse is synchronous.
        int h = 0;
        CHW_CUDA(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, st));
        CHW_CUDA(cudaStreamSynchronize(st));
        if (h) s = fail(CHW_ERR_STRUCTURE, "haar_inverse: signal is not an integer forward-transform output");
      }
      break;
    default:
      s = fail(CHW_ERR_UNSUPPORTED, "haar_inverse: dtype not supported (f64, f32, int64)");
  }
  return s;
}

size_t haar_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n) {
  const size_t es = (dtype == CHW_F32) ? 4 : 8;
  const uint64_t smem_max = kSmemMaxBytes / (2 * es);
  if (n <= smem_max || batch <= 0) return 0;
  return 2 * (size_t)batch * (n / 2) * es;
}

// Largest K such that the blocks below 2^K of a row fit the shared-memory kernel.
int haar_walsh_prefix_bits(chw_dtype dtype, int m) {
  const int es = (dtype == CHW_F64 || dtype == CHW_I64) ? 8 : 4;  // bf16 is computed in fp32
  int kmax = 0;
  while (((size_t)2 << kmax) * es <= (size_t)kSmemMaxBytes) ++kmax;
  return std::min(m, kmax);
}

// In place on x (rows of n): the Haar-Walsh map of the blocks below 2^K.
chw_status haar_walsh_prefix_device(void* x, chw_dtype dtype, int64_t batch, uint64_t n, int K, chw_mode mode,
                                    cudaStream_t st) {
  const bool ortho = (mode == CHW_ORTHONORMAL);
  switch (dtype) {
    case CHW_F64: return haar_walsh_prefix_impl(static_cast<double*>(x), batch, n, K, ortho, st);
    case CHW_F32: return haar_walsh_prefix_impl(static_cast<float*>(x), batch, n, K, ortho, st);
    case CHW_I64: return haar_walsh_prefix_impl(static_cast<long long*>(x), batch, n, K, false, st);
    case CHW_BF16: return haar_walsh_prefix_impl(static_cast<__nv_bfloat16*>(x), batch, n, K, ortho, st);
  }
  return fail(CHW_ERR_UNSUPPORTED, "haar_walsh_forward: unsupported dtype");
}

chw_status haar_forward_device(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                               chw_mode mode, void* ws, cudaStream_t st) {
  const bool ortho = (mode == CHW_ORTHONORMAL);
  switch (dtype) {
    case CHW_F64:
      return haar_impl<double>(static_cast<const double*>(in), static_cast<double*>(out), batch, n, ortho, ws,
                               st);
    case CHW_F32:
      return haar_impl<float>(static_cast<const float*>(in), static_cast<float*>(out), batch, n, ortho, ws, st);
    case CHW_I64:
      return haar_impl<long long>(static_cast<const long long*>(in), static_cast<long long*>(out), batch, n,
                                  false, ws, st);
    default:
      return fail(CHW_ERR_UNSUPPORTED, "haar_forward: dtype not supported (f64, f32, int64)");
  }
}

}  // namespace chwb
