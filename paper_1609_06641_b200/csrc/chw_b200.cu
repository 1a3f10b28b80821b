// chw_b200.cu — dispatch + C ABI (include/chw_b200.h).
//
// Host-side flow of chw_b200_forward (replaces chw::chw_forward_inplace,
// transforms.hpp:126-143, applied to every row of a batch):
//   validate (common.hpp:31-46 wording) -> pick the schedule for (dtype, m) ->
//   launch K1 (one pass) or the K4 passes on the caller's stream.
// No CPU fallback exists: without a device every call returns
// CHW_ERR_NO_DEVICE / CHW_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/chw_b200.h"
#include "launch.cuh"

using namespace chwb;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

bool is_pow2(uint64_t n) { return n != 0 && (n & (n - 1)) == 0; }
int level_of(uint64_t n) { return 63 - __builtin_clzll(n); }

size_t elem_size(chw_dtype d) {
  switch (d) {
    case CHW_F64:
    case CHW_I64:
      return 8;
    case CHW_F32:
      return 4;
    case CHW_BF16:
      return 2;
  }
  return 0;
}

}  // namespace

namespace chwb {
chw_status fail(chw_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
chw_status cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? CHW_ERR_NO_DEVICE
                                                                          : CHW_ERR_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}
chw_status current_device(int* dev) {
  CHW_CUDA(cudaGetDevice(dev));
  if (*dev < 0 || *dev >= 64) return fail(CHW_ERR_UNSUPPORTED, "device index out of range");
  return CHW_OK;
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace chwb

namespace chwb {
chw_status permute_order(const void* src, void* dst, size_t elem_bytes, chw_order order, int64_t batch, int m,
                         cudaStream_t st);
size_t haar_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n);
size_t haar_inverse_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n);
chw_status haar_inverse_device(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                               chw_mode mode, void* ws, cudaStream_t st);
int haar_walsh_prefix_bits(chw_dtype dtype, int m);
chw_status haar_walsh_prefix_device(void* x, chw_dtype dtype, int64_t batch, uint64_t n, int K, chw_mode mode,
                                    cudaStream_t st);
chw_status haar_forward_device(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                               chw_mode mode, void* ws, cudaStream_t st);
}  // namespace chwb

namespace {

// Reference validation order and text: require_pow2 then require_mode
// (transforms.hpp:127-130, common.hpp:31-46).
chw_status validate(const char* what, chw_dtype dtype, uint64_t n, chw_mode mode) {
  if (!is_pow2(n))
    return fail(CHW_ERR_LENGTH,
                std::string(what) + ": length " + std::to_string(n) + " is not a power of two");
  if (dtype == CHW_I64 && mode == CHW_ORTHONORMAL)
    return fail(CHW_ERR_MODE,
                std::string(what) + ": orthonormal mode requires a floating-point signal");
  if (dtype != CHW_F64 && dtype != CHW_F32 && dtype != CHW_BF16 && dtype != CHW_I64)
    return fail(CHW_ERR_UNSUPPORTED, std::string(what) + ": unknown dtype");
  if (mode != CHW_ORTHONORMAL && mode != CHW_UNNORMALIZED)
    return fail(CHW_ERR_ARGUMENT, std::string(what) + ": unknown scaling mode");
  if (level_of(n) > kMaxM)
    return fail(CHW_ERR_UNSUPPORTED, std::string(what) + ": length " + std::to_string(n) +
                                         " exceeds the supported maximum 2^" + std::to_string(kMaxM));
  return CHW_OK;
}

// 2^(-m/2): exact power of two for even m, one rounding of (2^-(m-1)/2)/sqrt2
// for odd m (the product of the reference's m per-butterfly kInvSqrt2 factors).
double ortho_scale(int m) {
  double s = std::ldexp(1.0, -(m / 2));
  if (m & 1) s *= 0.70710678118654752440;
  return s;
}

// ---------------------------------------------------------------------------
// Per-device state: SM count, lazily-grown workspace, streams for the host path.
// ---------------------------------------------------------------------------
struct DeviceState {
  std::mutex mu;  // serialises host-buffer calls (they own everything below)
  void* ws = nullptr;  // host path only: per-chunk workspaces of its two streams
  size_t ws_bytes = 0;
  int sms = 0;
  // host path
  cudaStream_t streams[2] = {nullptr, nullptr};
  void* dbuf[2] = {nullptr, nullptr};
  size_t dbuf_bytes = 0;
  void* pinned[2] = {nullptr, nullptr};
  size_t pinned_bytes = 0;
  cudaEvent_t done[2] = {nullptr, nullptr};
};
DeviceState g_dev[64];

// Library-managed scratch for calls made with workspace == NULL: stream-ordered
// allocations from a private per-device memory pool (cudaMallocFromPoolAsync
// on the caller's stream, cudaFreeAsync on the same stream after the last
// launch that uses it).  Concurrent calls on different streams therefore get
// disjoint buffers, and a buffer is reused only after the work that used it
// has completed in stream order — the reference's "concurrent calls on
// disjoint buffers are safe" contract without a shared buffer.
// The pool keeps its memory (release threshold = max), so steady-state calls
// do not reach the driver's allocator.
cudaMemPool_t g_pool[64] = {};
std::mutex g_pool_mu;

chw_status ws_pool(int dev, cudaMemPool_t* out) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    CHW_CUDA(cudaMemPoolCreate(&p, &props));
    uint64_t thr = ~0ull;
    CHW_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr));
    g_pool[dev] = p;
  }
  *out = g_pool[dev];
  return CHW_OK;
}

// RAII lease: `p` is the caller's workspace or a stream-ordered allocation
// that is released on `st` when the lease goes out of scope (after the
// launches that use it have been enqueued).
struct WsLease {
  void* p = nullptr;
  bool owned = false;
  cudaStream_t st = nullptr;
  WsLease() = default;
  WsLease(const WsLease&) = delete;
  WsLease& operator=(const WsLease&) = delete;
  ~WsLease() {
    if (owned && p) cudaFreeAsync(p, st);
  }
};

chw_status lease_workspace(const char* what, size_t need, void* caller_ws, size_t caller_bytes, cudaStream_t st,
                           WsLease* lease) {
  lease->st = st;
  if (need == 0) {
    lease->p = caller_ws;
    return CHW_OK;
  }
  if (caller_ws) {
    if (caller_bytes < need)
      return fail(CHW_ERR_WORKSPACE, std::string(what) + ": workspace of " + std::to_string(caller_bytes) +
                                         " bytes is smaller than the " + std::to_string(need) + " required");
    lease->p = caller_ws;
    return CHW_OK;
  }
  int dev = 0;
  if (chw_status s = current_device(&dev)) return s;
  cudaMemPool_t pool = nullptr;
  if (chw_status s = ws_pool(dev, &pool)) return s;
  void* p = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&p, need, pool, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CHW_ERR_RESOURCE, std::string(what) + ": cannot allocate " + std::to_string(need) +
                                      " bytes of workspace: " + cudaGetErrorString(e));
  }
  lease->p = p;
  lease->owned = true;
  return CHW_OK;
}

// The kernels move 16-byte vectors and TMA tiles: every device buffer must be
// 16-byte aligned (cudaMalloc and torch allocations are).  Checked once here,
// before any launch, so a misaligned view returns CHW_ERR_ARGUMENT instead of
// raising a sticky cudaErrorMisalignedAddress.
chw_status check_aligned(const char* what, const void* a, const void* b, const void* c) {
  if (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 15u)
    return fail(CHW_ERR_ARGUMENT, std::string(what) + ": buffers and workspace must be 16-byte aligned");
  return CHW_OK;
}

size_t workspace_for(chw_dtype dtype, int64_t batch, int m) {
  if (batch <= 0) return 0;
  switch (dtype) {
    case CHW_F64:
      return m <= Regime<double>::K1MAX ? 0 : k4_workspace<double>(m, batch);
    case CHW_I64:
      return m <= Regime<long long>::K1MAX ? 0 : k4_workspace<long long>(m, batch);
    case CHW_F32:
      return m <= Regime<float>::K1MAX ? 0 : k4_workspace<float>(m, batch);
    case CHW_BF16:
      return m <= Regime<__nv_bfloat16>::K1MAX ? 0 : k4_workspace<__nv_bfloat16>(m, batch);
  }
  return 0;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int k1max_of(chw_dtype dtype);
// NATURAL and SEQUENCY are folded into the single-pass kernels' stores.
bool order_fused(chw_dtype dtype, int m, chw_order order) {
  if (order == CHW_ORDER_DYADIC) return true;
  if (m <= k1max_of(dtype)) return true;
  // sequency is an XOR-linear map of the dyadic position: folded into the
  // f32 long-row kernels' stores (K6 m = 16, K9 m = 24); natural order needs
  // the second phase to carry j0..j3 so its runs stay whole 64-byte pieces:
  // K6 at m = 16, the K9n plan at m = 24
  if (dtype != CHW_F32) return false;
  if (order == CHW_ORDER_SEQUENCY) return m == 16 || m == 24;
  return order == CHW_ORDER_NATURAL && (m == 16 || m == 24);
}

size_t ordered_workspace(chw_dtype dtype, int64_t batch, int m, chw_order order) {
  const size_t inner = workspace_for(dtype, batch, m);
  if (order == CHW_ORDER_DYADIC || batch <= 0) return inner;
  // Orders folded into the kernel's store map need no gather buffer.
  if (order_fused(dtype, m, order)) return inner;
  return align256(inner) + (size_t)batch * ((size_t)1 << m) * elem_size(dtype);
}

chw_status dyadic_impl(const void* in, void* out, chw_dtype dtype, int64_t batch, int m, chw_mode mode,
                       void* ws, cudaStream_t st);

int k1max_of(chw_dtype dtype) {
  switch (dtype) {
    case CHW_F64: return Regime<double>::K1MAX;
    case CHW_I64: return Regime<long long>::K1MAX;
    case CHW_F32: return Regime<float>::K1MAX;
    case CHW_BF16: return Regime<__nv_bfloat16>::K1MAX;
  }
  return -1;
}

chw_status ordered_k1_impl(const void* in, void* out, chw_dtype dtype, int64_t batch, int m, chw_mode mode,
                           bool seq, cudaStream_t st) {
  const bool ortho = (mode == CHW_ORTHONORMAL);
  switch (dtype) {
    case CHW_F64:
      return forward_k1_natural<double>(m, ortho, seq, static_cast<const double*>(in), static_cast<double*>(out),
                                        batch, 1.0, st);
    case CHW_I64:
      return forward_k1_natural<long long>(m, false, seq, static_cast<const long long*>(in),
                                           static_cast<long long*>(out), batch, 1, st);
    case CHW_F32:
      return forward_k1_natural<float>(m, ortho, seq, static_cast<const float*>(in), static_cast<float*>(out), batch,
                                       (float)ortho_scale(m), st);
    case CHW_BF16:
      return forward_k1_natural<__nv_bfloat16>(m, ortho, seq, static_cast<const __nv_bfloat16*>(in),
                                               static_cast<__nv_bfloat16*>(out), batch, (float)ortho_scale(m),
                                               st);
  }
  return fail(CHW_ERR_UNSUPPORTED, "chw_forward: unknown dtype");
}

chw_status forward_impl(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                        chw_mode mode, chw_order order, void* workspace, size_t workspace_bytes,
                        cudaStream_t st) {
  if (chw_status s = validate("chw_forward", dtype, n, mode)) return s;
  if (batch < 0) return fail(CHW_ERR_ARGUMENT, "chw_forward: negative batch");
  if (order != CHW_ORDER_DYADIC && order != CHW_ORDER_NATURAL && order != CHW_ORDER_SEQUENCY)
    return fail(CHW_ERR_ARGUMENT, "chw_forward: unknown output order");
  if (batch == 0) return CHW_OK;
  if (!in || !out) return fail(CHW_ERR_ARGUMENT, "chw_forward: null buffer");
  const int m = level_of(n);
  const size_t need = ordered_workspace(dtype, batch, m, order);
  if (chw_status s = check_aligned("chw_forward", in, out, need ? workspace : nullptr)) return s;
  WsLease lease;
  if (chw_status s = lease_workspace("chw_forward", need, workspace, workspace_bytes, st, &lease)) return s;
  void* ws = lease.p;
  if (order == CHW_ORDER_DYADIC) return dyadic_impl(in, out, dtype, batch, m, mode, ws, st);
  // Natural / sequency order for single-pass sizes: the order is the kernel's
  // store map (identity / inverse Gray code), zero extra bytes.
  if (m <= k1max_of(dtype))
    return ordered_k1_impl(in, out, dtype, batch, m, mode, order == CHW_ORDER_SEQUENCY, st);
  if (order_fused(dtype, m, order)) {  // f32 natural / sequency at m = 16 (K6) and m = 24 (K9n / K9)
    const bool ortho = (mode == CHW_ORTHONORMAL);
    const float sc = (float)ortho_scale(m);
    auto* i = static_cast<const float*>(in);
    auto* o = static_cast<float*>(out);
    if (m == 16)
      return launch_rowpipe_m16_ordered(order == CHW_ORDER_NATURAL ? 1 : 2, ortho, i, o, ws, batch, sc, st);
    // (the sweep also serves the fused orders when CHW_B200_M24=t selects K4T for the dyadic order)
    return launch_sweep_m24(ortho, i, o, ws, batch, sc, st, order == CHW_ORDER_NATURAL ? 1 : 2);
  }
  // Other orders: dyadic result into the workspace, then one coalesced gather.
  void* tmp = static_cast<char*>(ws) + align256(workspace_for(dtype, batch, m));
  if (chw_status s = dyadic_impl(in, tmp, dtype, batch, m, mode, ws, st)) return s;
  return permute_order(tmp, out, elem_size(dtype), order, batch, m, st);
}

chw_status dyadic_impl(const void* in, void* out, chw_dtype dtype, int64_t batch, int m, chw_mode mode,
                       void* ws, cudaStream_t st) {
  const bool ortho = (mode == CHW_ORTHONORMAL);
  switch (dtype) {
    case CHW_F64: {
      auto* i = static_cast<const double*>(in);
      auto* o = static_cast<double*>(out);
      return m <= Regime<double>::K1MAX ? forward_k1<double>(m, ortho, i, o, batch, 1.0, st)
                                        : forward_k4<double>(m, ortho, i, o, ws, batch, 1.0, st);
    }
    case CHW_I64: {
      auto* i = static_cast<const long long*>(in);
      auto* o = static_cast<long long*>(out);
      return m <= Regime<long long>::K1MAX
                 ? forward_k1<long long>(m, false, i, o, batch, 1, st)
                 : forward_k4<long long>(m, false, i, o, ws, batch, 1, st);
    }
    case CHW_F32: {
      auto* i = static_cast<const float*>(in);
      auto* o = static_cast<float*>(out);
      const float sc = (float)ortho_scale(m);
      return m <= Regime<float>::K1MAX ? forward_k1<float>(m, ortho, i, o, batch, sc, st)
                                       : forward_k4<float>(m, ortho, i, o, ws, batch, sc, st);
    }
    case CHW_BF16: {
      auto* i = static_cast<const __nv_bfloat16*>(in);
      auto* o = static_cast<__nv_bfloat16*>(out);
      const float sc = (float)ortho_scale(m);
      return m <= Regime<__nv_bfloat16>::K1MAX
                 ? forward_k1<__nv_bfloat16>(m, ortho, i, o, batch, sc, st)
                 : forward_k4<__nv_bfloat16>(m, ortho, i, o, ws, batch, sc, st);
    }
  }
  return fail(CHW_ERR_UNSUPPORTED, "chw_forward: unknown dtype");
}

// ---------------------------------------------------------------------------
// Host-buffer path: rows are processed in chunks; chunk c uses stream c%2, so
// the H2D copy of chunk c+1, the kernels of chunk c and the D2H copy of chunk
// c-1 overlap (two copy engines + compute).
// ---------------------------------------------------------------------------
chw_status host_impl(const void* in_host, void* out_host, chw_dtype dtype, int64_t batch,
                     uint64_t n, chw_mode mode, chw_order order) {
  if (chw_status s = validate("chw_forward", dtype, n, mode)) return s;
  if (batch < 0) return fail(CHW_ERR_ARGUMENT, "chw_forward: negative batch");
  if (batch == 0) return CHW_OK;
  if (!in_host || !out_host) return fail(CHW_ERR_ARGUMENT, "chw_forward: null buffer");
  int dev = 0;
  if (chw_status s = current_device(&dev)) return s;
  DeviceState& d = g_dev[dev];
  std::lock_guard<std::mutex> lk(d.mu);

  const size_t es = elem_size(dtype);
  const size_t row_bytes = (size_t)n * es;
  const int m = level_of(n);
  // ~64 MiB chunks (at least one row).
  const size_t target = (size_t)64 << 20;
  int64_t rows_per_chunk = (int64_t)std::max<size_t>(1, target / row_bytes);
  rows_per_chunk = std::min<int64_t>(rows_per_chunk, batch);
  const size_t chunk_bytes = (size_t)rows_per_chunk * row_bytes;

  for (int i = 0; i < 2; ++i)
    if (!d.streams[i]) {
      CHW_CUDA(cudaStreamCreateWithFlags(&d.streams[i], cudaStreamNonBlocking));
      CHW_CUDA(cudaEventCreateWithFlags(&d.done[i], cudaEventDisableTiming));
    }
  if (d.dbuf_bytes < chunk_bytes) {
    for (int i = 0; i < 2; ++i) {
      if (d.dbuf[i]) cudaFree(d.dbuf[i]);
      d.dbuf[i] = nullptr;
    }
    d.dbuf_bytes = 0;
    for (int i = 0; i < 2; ++i)
      if (cudaMalloc(&d.dbuf[i], chunk_bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(CHW_ERR_RESOURCE, "chw_forward: cannot allocate device staging buffers");
      }
    d.dbuf_bytes = chunk_bytes;
  }
  // Workspace for multi-pass sizes, one per stream.
  // 256-byte aligned per-stream slices (the kernels use 16-byte vector accesses).
  const size_t ws_chunk = (ordered_workspace(dtype, rows_per_chunk, m, order) + 255) & ~size_t(255);
  std::vector<void*> wss(2, nullptr);
  void* ws_all = nullptr;
  if (ws_chunk > 0) {
    DeviceState& s = d;
    if (s.ws_bytes < 2 * ws_chunk) {
      if (s.ws) {
        // Only host calls (serialised by s.mu) use s.ws; drain their streams.
        for (int i = 0; i < 2; ++i) cudaStreamSynchronize(s.streams[i]);
        cudaFree(s.ws);
      }
      s.ws = nullptr;
      s.ws_bytes = 0;
      if (cudaMalloc(&s.ws, 2 * ws_chunk) != cudaSuccess) {
        cudaGetLastError();
        return fail(CHW_ERR_RESOURCE, "chw_forward: cannot allocate workspace");
      }
      s.ws_bytes = 2 * ws_chunk;
    }
    ws_all = s.ws;
    wss[0] = ws_all;
    wss[1] = static_cast<char*>(ws_all) + ws_chunk;
  }

  cudaPointerAttributes ai{}, ao{};
  const bool in_pinned = cudaPointerGetAttributes(&ai, in_host) == cudaSuccess &&
                         ai.type == cudaMemoryTypeHost;
  const bool out_pinned = cudaPointerGetAttributes(&ao, out_host) == cudaSuccess &&
                          ao.type == cudaMemoryTypeHost;
  cudaGetLastError();
  const bool staged = !(in_pinned && out_pinned);
  if (staged && d.pinned_bytes < chunk_bytes) {
    for (int i = 0; i < 2; ++i) {
      if (d.pinned[i]) cudaFreeHost(d.pinned[i]);
      d.pinned[i] = nullptr;
    }
    d.pinned_bytes = 0;
    for (int i = 0; i < 2; ++i)
      if (cudaMallocHost(&d.pinned[i], chunk_bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(CHW_ERR_RESOURCE, "chw_forward: cannot allocate pinned staging buffers");
      }
    d.pinned_bytes = chunk_bytes;
  }

  const char* src = static_cast<const char*>(in_host);
  char* dst = static_cast<char*>(out_host);
  const int64_t nchunks = (batch + rows_per_chunk - 1) / rows_per_chunk;
  // In the staged path chunk c's output must land in out_host before the
  // pinned buffer is reused for chunk c+2; the event wait below orders that.
  std::vector<int64_t> pending_rows(2, 0), pending_row0(2, 0);
  for (int64_t c = 0; c < nchunks; ++c) {
    const int b = (int)(c & 1);
    cudaStream_t st = d.streams[b];
    const int64_t r0 = c * rows_per_chunk;
    const int64_t rows = std::min<int64_t>(rows_per_chunk, batch - r0);
    const size_t bytes = (size_t)rows * row_bytes;
    if (staged) {
      // Drain the previous use of this buffer pair (chunk c-2).
      CHW_CUDA(cudaEventSynchronize(d.done[b]));
      if (pending_rows[b] > 0) {
        if (!out_pinned)
          std::memcpy(dst + (size_t)pending_row0[b] * row_bytes, d.pinned[b],
                      (size_t)pending_rows[b] * row_bytes);
        pending_rows[b] = 0;
      }
      const void* h_in = src + (size_t)r0 * row_bytes;
      if (!in_pinned) {
        std::memcpy(d.pinned[b], h_in, bytes);
        h_in = d.pinned[b];
      }
      CHW_CUDA(cudaMemcpyAsync(d.dbuf[b], h_in, bytes, cudaMemcpyHostToDevice, st));
    } else {
      CHW_CUDA(cudaMemcpyAsync(d.dbuf[b], src + (size_t)r0 * row_bytes, bytes,
                               cudaMemcpyHostToDevice, st));
    }
    if (chw_status s = forward_impl(d.dbuf[b], d.dbuf[b], dtype, rows, n, mode, order, wss[b], ws_chunk, st))
      return s;
    void* h_out = (staged && !out_pinned) ? d.pinned[b] : dst + (size_t)r0 * row_bytes;
    CHW_CUDA(cudaMemcpyAsync(h_out, d.dbuf[b], bytes, cudaMemcpyDeviceToHost, st));
    CHW_CUDA(cudaEventRecord(d.done[b], st));
    if (staged && !out_pinned) {
      pending_rows[b] = rows;
      pending_row0[b] = r0;
    }
  }
  for (int b = 0; b < 2; ++b) {
    CHW_CUDA(cudaEventSynchronize(d.done[b]));
    if (pending_rows[b] > 0)
      std::memcpy(dst + (size_t)pending_row0[b] * row_bytes, d.pinned[b],
                  (size_t)pending_rows[b] * row_bytes);
  }
  (void)ws_all;
  return CHW_OK;
}

}  // namespace

namespace {
// Synchronous host-buffer wrapper for the secondary transforms (compatibility
// path: one device copy of the batch, no pipelining).
template <class F>
chw_status host_stage(const void* in_host, void* out_host, chw_dtype dtype, int64_t batch, uint64_t n, F&& fn) {
  const size_t bytes = (size_t)batch * (size_t)n * elem_size(dtype);
  if (bytes == 0) return fn(nullptr);
  void* d = nullptr;
  if (cudaMalloc(&d, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(CHW_ERR_RESOURCE, "cannot allocate device buffer");
  }
  chw_status s = CHW_OK;
  cudaError_t e = cudaMemcpy(d, in_host, bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpy");
  if (s == CHW_OK) s = fn(d);
  if (s == CHW_OK) {
    e = cudaStreamSynchronize(nullptr);
    if (e != cudaSuccess) s = cuda_fail(e, "cudaStreamSynchronize");
  }
  if (s == CHW_OK) {
    e = cudaMemcpy(out_host, d, bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpy");
  }
  cudaFree(d);
  return s;
}

}  // namespace

extern "C" {

chw_status chw_b200_forward(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                            chw_mode mode, void* workspace, size_t workspace_bytes, void* stream) {
  return forward_impl(in, out, dtype, batch, n, mode, CHW_ORDER_DYADIC, workspace, workspace_bytes,
                      static_cast<cudaStream_t>(stream));
}

chw_status chw_b200_forward_ordered(const void* in, void* out, chw_dtype dtype, int64_t batch,
                                    uint64_t n, chw_mode mode, chw_order order, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  return forward_impl(in, out, dtype, batch, n, mode, order, workspace, workspace_bytes,
                      static_cast<cudaStream_t>(stream));
}

size_t chw_b200_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n) {
  if (!is_pow2(n)) return 0;
  return workspace_for(dtype, batch, level_of(n));
}

size_t chw_b200_workspace_bytes_ordered(chw_dtype dtype, int64_t batch, uint64_t n, chw_order order) {
  if (!is_pow2(n)) return 0;
  return ordered_workspace(dtype, batch, level_of(n), order);
}

chw_status chw_b200_forward_host(const void* in_host, void* out_host, chw_dtype dtype,
                                 int64_t batch, uint64_t n, chw_mode mode) {
  return host_impl(in_host, out_host, dtype, batch, n, mode, CHW_ORDER_DYADIC);
}

chw_status chw_b200_forward_host_ordered(const void* in_host, void* out_host, chw_dtype dtype, int64_t batch,
                                         uint64_t n, chw_mode mode, chw_order order) {
  return host_impl(in_host, out_host, dtype, batch, n, mode, order);
}

size_t chw_b200_haar_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n) {
  if (!is_pow2(n)) return 0;
  return haar_workspace_bytes(dtype, batch, n);
}

chw_status chw_b200_haar_forward(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                                 chw_mode mode, void* workspace, size_t workspace_bytes, void* stream) {
  // transforms.hpp:51-52: require_pow2 then require_mode, "haar_forward" wording.
  if (chw_status s = validate("haar_forward", dtype, n, mode)) return s;
  if (dtype == CHW_BF16) return fail(CHW_ERR_UNSUPPORTED, "haar_forward: bf16 is not supported");
  if (batch < 0) return fail(CHW_ERR_ARGUMENT, "haar_forward: negative batch");
  if (batch == 0) return CHW_OK;
  if (!in || !out) return fail(CHW_ERR_ARGUMENT, "haar_forward: null buffer");
  const size_t need = haar_workspace_bytes(dtype, batch, n);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (chw_status s = check_aligned("haar_forward", in, out, need ? workspace : nullptr)) return s;
  WsLease lease;
  if (chw_status s = lease_workspace("haar_forward", need, workspace, workspace_bytes, st, &lease)) return s;
  return haar_forward_device(in, out, dtype, batch, n, mode, lease.p, st);
}

chw_status chw_b200_haar_forward_host(const void* in_host, void* out_host, chw_dtype dtype, int64_t batch,
                                      uint64_t n, chw_mode mode) {
  if (chw_status s = validate("haar_forward", dtype, n, mode)) return s;
  if (dtype == CHW_BF16) return fail(CHW_ERR_UNSUPPORTED, "haar_forward: bf16 is not supported");
  if (batch < 0) return fail(CHW_ERR_ARGUMENT, "haar_forward: negative batch");
  if (batch == 0) return CHW_OK;
  if (!in_host || !out_host) return fail(CHW_ERR_ARGUMENT, "haar_forward: null buffer");
  // Compatibility path (synchronous, unpipelined): one device copy of the batch.
  const size_t bytes = (size_t)batch * (size_t)n * elem_size(dtype);
  void* d = nullptr;
  if (cudaMalloc(&d, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(CHW_ERR_RESOURCE, "haar_forward: cannot allocate device buffer");
  }
  chw_status s = CHW_OK;
  cudaError_t e = cudaMemcpy(d, in_host, bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpy");
  if (s == CHW_OK) s = chw_b200_haar_forward(d, d, dtype, batch, n, mode, nullptr, 0, nullptr);
  if (s == CHW_OK) {
    e = cudaMemcpy(out_host, d, bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpy");
  }
  cudaFree(d);
  return s;
}

size_t chw_b200_haar_inverse_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n) {
  if (!is_pow2(n)) return 0;
  return haar_inverse_workspace_bytes(dtype, batch, n);
}

chw_status chw_b200_haar_inverse(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                                 chw_mode mode, void* workspace, size_t workspace_bytes, void* stream) {
  // transforms.hpp:87-88: require_pow2 then require_mode, "haar_inverse" wording.
  if (chw_status s = validate("haar_inverse", dtype, n, mode)) return s;
  if (dtype == CHW_BF16) return fail(CHW_ERR_UNSUPPORTED, "haar_inverse: bf16 is not supported");
  if (batch < 0) return fail(CHW_ERR_ARGUMENT, "haar_inverse: negative batch");
  if (batch == 0) return CHW_OK;
  if (!in || !out) return fail(CHW_ERR_ARGUMENT, "haar_inverse: null buffer");
  const size_t need = haar_inverse_workspace_bytes(dtype, batch, n);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (chw_status s = check_aligned("haar_inverse", in, out, workspace)) return s;
  WsLease lease;
  if (chw_status s = lease_workspace("haar_inverse", need, workspace, workspace_bytes, st, &lease)) return s;
  return haar_inverse_device(in, out, dtype, batch, n, mode, lease.p, st);
}

chw_status chw_b200_haar_walsh_forward(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                                       chw_mode mode, void* stream) {
  // transforms.hpp:190-198: dyadic WHT of each scale block [2^j, 2^(j+1)), j = 1..m-1.
  if (chw_status s = validate("haar_walsh_forward", dtype, n, mode)) return s;
  if (batch < 0) return fail(CHW_ERR_ARGUMENT, "haar_walsh_forward: negative batch");
  if (batch == 0) return CHW_OK;
  if (!in || !out) return fail(CHW_ERR_ARGUMENT, "haar_walsh_forward: null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (chw_status s = check_aligned("haar_walsh_forward", in, out, nullptr)) return s;
  const size_t es = elem_size(dtype);
  if (in != out) CHW_CUDA(cudaMemcpyAsync(out, in, (size_t)batch * n * es, cudaMemcpyDeviceToDevice, st));
  const int m = level_of(n);
  if (m < 2) return CHW_OK;
  // Blocks j < K of every row: one shared-memory kernel (haar.cu), one HBM
  // read and write of the prefix.
  const int K = haar_walsh_prefix_bits(dtype, m);
  if (chw_status s = haar_walsh_prefix_device(out, dtype, batch, n, K, mode, st)) return s;
  if (K >= m) return CHW_OK;
  // Longer blocks j = K..m-1: gather block j of every row into a contiguous
  // [batch][2^j] buffer, run the batched dyadic kernel on it, scatter back.
  const size_t tmp_bytes = (size_t)batch * (n / 2) * es;
  size_t inner = 0;
  for (int j = K; j <= m - 1; ++j) inner = std::max(inner, workspace_for(dtype, batch, j));
  WsLease lease;
  if (chw_status s = lease_workspace("haar_walsh_forward", align256(tmp_bytes) + inner, nullptr, 0, st, &lease))
    return s;
  char* tmp = static_cast<char*>(lease.p);
  void* inner_ws = tmp + align256(tmp_bytes);
  char* o = static_cast<char*>(out);
  for (int j = K; j <= m - 1; ++j) {
    const size_t blk = ((size_t)1 << j) * es;
    CHW_CUDA(cudaMemcpy2DAsync(tmp, blk, o + blk, n * es, blk, (size_t)batch, cudaMemcpyDeviceToDevice, st));
    if (chw_status s = dyadic_impl(tmp, tmp, dtype, batch, j, mode, inner_ws, st)) return s;
    CHW_CUDA(cudaMemcpy2DAsync(o + blk, n * es, tmp, blk, blk, (size_t)batch, cudaMemcpyDeviceToDevice, st));
  }
  return CHW_OK;
}

chw_status chw_b200_haar_inverse_host(const void* in_host, void* out_host, chw_dtype dtype, int64_t batch,
                                      uint64_t n, chw_mode mode) {
  if (chw_status s = validate("haar_inverse", dtype, n, mode)) return s;
  if (batch <= 0) return batch < 0 ? fail(CHW_ERR_ARGUMENT, "haar_inverse: negative batch") : CHW_OK;
  return host_stage(in_host, out_host, dtype, batch, n, [&](void* d) {
    return chw_b200_haar_inverse(d, d, dtype, batch, n, mode, nullptr, 0, nullptr);
  });
}

chw_status chw_b200_haar_walsh_forward_host(const void* in_host, void* out_host, chw_dtype dtype, int64_t batch,
                                            uint64_t n, chw_mode mode) {
  if (chw_status s = validate("haar_walsh_forward", dtype, n, mode)) return s;
  if (batch <= 0) return batch < 0 ? fail(CHW_ERR_ARGUMENT, "haar_walsh_forward: negative batch") : CHW_OK;
  return host_stage(in_host, out_host, dtype, batch, n, [&](void* d) {
    return chw_b200_haar_walsh_forward(d, d, dtype, batch, n, mode, nullptr);
  });
}

chw_status chw_b200_parallel_execute(void* x, chw_dtype dtype, uint64_t n, int workers,
                                     chw_mode mode, void* stream) {
  // parallel.cpp:84-91: require_pow2, require_mode, then workers >= 1.
  if (chw_status s = validate("parallel_execute", dtype, n, mode)) return s;
  if (workers < 1)
    return fail(CHW_ERR_ARGUMENT,
                "parallel_execute: workers must be >= 1, got " + std::to_string(workers));
  return forward_impl(x, x, dtype, 1, n, mode, CHW_ORDER_DYADIC, nullptr, 0,
                      static_cast<cudaStream_t>(stream));
}

chw_status chw_b200_op_tally(int op, uint64_t n, chw_mode mode, uint64_t* additions,
                             uint64_t* multiplications) {
  if (!is_pow2(n)) return fail(CHW_ERR_LENGTH, "op_tally: length " + std::to_string(n) +
                                                   " is not a power of two");
  const uint64_t m = (uint64_t)level_of(n);
  uint64_t a = 0, mu = 0;
  const bool ortho = (mode == CHW_ORTHONORMAL);
  switch (op) {
    case 0:  // chw_forward: m levels of n adds (transforms.hpp:75-78)
      a = m * n;
      mu = ortho ? m * n : 0;
      break;
    case 1:  // haar_forward: sum_{len=n..2} len = 2(n-1)
      a = 2 * (n - 1);
      mu = ortho ? 2 * (n - 1) : 0;
      break;
    case 2:  // normalize: n multiplications (transforms.hpp:209)
      mu = n;
      break;
    default:
      return fail(CHW_ERR_ARGUMENT, "op_tally: unknown op");
  }
  if (additions) *additions = a;
  if (multiplications) *multiplications = mu;
  return CHW_OK;
}

const char* chw_b200_status_string(chw_status s) {
  switch (s) {
    case CHW_OK:
      return "ok";
    case CHW_ERR_LENGTH:
      return "length is not a power of two";
    case CHW_ERR_MODE:
      return "orthonormal mode requires a floating-point signal";
    case CHW_ERR_ARGUMENT:
      return "invalid argument";
    case CHW_ERR_UNSUPPORTED:
      return "unsupported";
    case CHW_ERR_WORKSPACE:
      return "workspace too small";
    case CHW_ERR_CUDA:
      return "CUDA error";
    case CHW_ERR_NO_DEVICE:
      return "no CUDA device";
    case CHW_ERR_RESOURCE:
      return "resource allocation failed";
    case CHW_ERR_STRUCTURE:
      return "structural precondition failed";
  }
  return "unknown status";
}

const char* chw_b200_last_error(void) { return g_last_error.c_str(); }

uint64_t chw_b200_launch_count(void) { return g_launches.load(); }

const char* chw_b200_plan_name(chw_dtype dtype, uint64_t n) {
  if (!is_pow2(n)) return "invalid";
  const int m = level_of(n);
  switch (dtype) {
    case CHW_F64:
      return plan_name<double>(m);
    case CHW_I64:
      return plan_name<long long>(m);
    case CHW_F32:
      return plan_name<float>(m);
    case CHW_BF16:
      return plan_name<__nv_bfloat16>(m);
  }
  return "invalid";
}

int chw_b200_abi_version(void) { return CHW_B200_ABI_VERSION; }

int chw_b200_is_device_pointer(const void* p) {
  if (!p) return 0;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? 1 : 0;
}

chw_status chw_b200_stream_synchronize(void* stream) {
  CHW_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return CHW_OK;
}

}  // extern "C"
