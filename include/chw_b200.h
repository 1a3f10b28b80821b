/*
 * chw_b200.h — C ABI of the B200-native batched CHW (dyadic-order WHT) library.
 *
 * The reference exposes only a C++20 header API (the proj/include/chw headers; no C
 * ABI, no FFI, no plugin registry — SURVEY §8b).  This header is the boundary a
 * foreign caller binds; include/chw_b200/chw.hpp re-exposes the reference's own
 * C++ signatures on top of it (the drop-in), and INTEGRATION.md shows both.
 *
 * Every entry point below replaces one reference interface:
 *
 *   chw_b200_forward        <- chw::chw_forward_inplace<T>
 *                              (proj/include/chw/transforms.hpp:126-143), batched:
 *                              `batch` contiguous rows of n elements, the loop the
 *                              reference leaves to its caller (chw_main.cpp:65).
 *                              Device pointers, stream-ordered, asynchronous.
 *   chw_b200_forward_host   <- the same call on HOST buffers, synchronous like the
 *                              reference (copies in and out are pipelined).
 *   chw_b200_parallel_execute <- chw::parallel_execute_inplace<T>
 *                              (proj/include/chw/parallel.hpp:16-17,
 *                              proj/src/parallel.cpp:84-97): same validation
 *                              (workers >= 1), same bitwise result as the serial
 *                              transform; runs the batched kernel with batch = 1.
 *   chw_b200_op_tally       <- chw::OpTally accounting (op_tally.hpp:12-22,
 *                              transforms.hpp:75-78) in closed form.
 *   chw_b200_workspace_bytes<- the optional `scratch` span of transforms.hpp:126-137
 *                              (caller-owned scratch, allocated when absent).
 *
 * Errors never cross this boundary as exceptions: each call returns a
 * chw_status and leaves the reference's exception text (same wording as
 * common.hpp:31-46, parallel.cpp:88-91) in a thread-local buffer,
 * chw_b200_last_error().  The C++ shim turns them back into the reference's
 * exception types.
 *
 * Thread safety: calls on different streams / disjoint buffers may run
 * concurrently.  A call made with workspace == NULL gets its own
 * stream-ordered scratch (cudaMallocFromPoolAsync on the caller's stream from a
 * private per-device pool, freed on that stream after its launches), so two
 * such calls never share scratch.  The host-buffer calls are synchronous and
 * serialised per device by an internal lock.
 */
#ifndef CHW_B200_H
#define CHW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHW_B200_ABI_VERSION 1

typedef enum chw_status {
  CHW_OK = 0,
  CHW_ERR_LENGTH = 1,      /* length not a power of two (incl. 0)  -> std::invalid_argument */
  CHW_ERR_MODE = 2,        /* Orthonormal on an integer signal       -> std::invalid_argument */
  CHW_ERR_ARGUMENT = 3,    /* other bad argument (workers < 1, null) -> std::invalid_argument */
  CHW_ERR_UNSUPPORTED = 4, /* dtype / size not supported by this build */
  CHW_ERR_WORKSPACE = 5,   /* caller workspace too small */
  CHW_ERR_CUDA = 6,        /* CUDA runtime error (text in last_error)  */
  CHW_ERR_NO_DEVICE = 7,   /* no CUDA device visible                   */
  CHW_ERR_RESOURCE = 8,    /* allocation failed                 -> chw::ResourceError */
  CHW_ERR_STRUCTURE = 9    /* int64 haar_inverse of a non-forward output -> chw::StructureError */
} chw_status;

/* Order matches chw::ScalingMode (proj/include/chw/common.hpp:15). */
typedef enum chw_mode { CHW_ORTHONORMAL = 0, CHW_UNNORMALIZED = 1 } chw_mode;

typedef enum chw_dtype {
  CHW_F64 = 0,  /* reference `double` path; Orthonormal is bit-exact with the reference */
  CHW_F32 = 1,  /* fp32 in/out, fp32 arithmetic, scale applied once at the end          */
  CHW_BF16 = 2, /* bf16 in/out, fp32 arithmetic, one rounding at the output           */
  CHW_I64 = 3   /* reference `std::int64_t` path: Unnormalized only, exact            */
} chw_dtype;

/* Output coefficient order.  DYADIC is the reference's
 * chw_forward order; NATURAL = fwht_natural (transforms.hpp:147-172);
 * SEQUENCY = dyadic_to_sequency applied to the dyadic output
 * (orderings.hpp:82-90, apply_permutation :92-102). */
typedef enum chw_order { CHW_ORDER_DYADIC = 0, CHW_ORDER_NATURAL = 1, CHW_ORDER_SEQUENCY = 2 } chw_order;

/* Batched CHW transform, dyadic order.  `in` and `out` are device pointers to
 * batch*n contiguous elements of `dtype` (in == out is allowed: in place).
 * `workspace` may be NULL (the library allocates and caches one per device) or
 * a device buffer of at least chw_b200_workspace_bytes(dtype, batch, n) bytes.
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Asynchronous.
 * Device buffers (in, out, workspace) must be 16-byte aligned, as cudaMalloc
 * and torch allocations are (the kernels move 16-byte vectors and TMA tiles). */
chw_status chw_b200_forward(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                            chw_mode mode, void* workspace, size_t workspace_bytes, void* stream);

/* Same, with an explicit output order (f2). */
chw_status chw_b200_forward_ordered(const void* in, void* out, chw_dtype dtype, int64_t batch,
                                    uint64_t n, chw_mode mode, chw_order order, void* workspace,
                                    size_t workspace_bytes, void* stream);

/* Workspace the device call needs (0 for single-pass sizes), and for a call
 * with an explicit order.  NATURAL and SEQUENCY are folded into the kernels'
 * stores — no extra workspace — for every single-pass size and for f32 rows
 * of 2^16 and 2^24; for the other long rows they add one batch-sized buffer
 * (the dyadic result is gathered into the requested order in one coalesced
 * pass). */
size_t chw_b200_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n);
size_t chw_b200_workspace_bytes_ordered(chw_dtype dtype, int64_t batch, uint64_t n, chw_order order);

/* Host-buffer call: copies `in_host` to the device, transforms, copies the
 * result to `out_host` (may equal in_host), and returns when done — the
 * reference's synchronous in-place contract.  Pinned host memory is used
 * directly; pageable memory is staged through internal pinned buffers.
 * Copies and kernels of consecutive row chunks overlap on two streams. */
chw_status chw_b200_forward_host(const void* in_host, void* out_host, chw_dtype dtype,
                                 int64_t batch, uint64_t n, chw_mode mode);

/* Batched Haar transform Psi_m <- chw::haar_forward_inplace
 * (proj/include/chw/transforms.hpp:49-80): output row [s, d_coarsest, ...,
 * d_finest], same operations and order as the reference (f64 bit-exact).
 * dtype F64/F32/I64 (I64: Unnormalized only).  Device pointers, in == out
 * allowed, asynchronous on `stream`.  Rows longer than 2^12 (f64) / 2^13
 * (f32) use a workspace (NULL = library-managed). */
chw_status chw_b200_haar_forward(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                                 chw_mode mode, void* workspace, size_t workspace_bytes, void* stream);
size_t chw_b200_haar_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n);
/* Batched inverse Haar transform <- chw::haar_inverse_inplace
 * (proj/include/chw/transforms.hpp:85-120); same operations and order (f64
 * bit-exact).  I64: an odd pair sum returns CHW_ERR_STRUCTURE (the reference's
 * StructureError), so the I64 call synchronizes `stream` before returning. */
chw_status chw_b200_haar_inverse(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                                 chw_mode mode, void* workspace, size_t workspace_bytes, void* stream);
size_t chw_b200_haar_inverse_workspace_bytes(chw_dtype dtype, int64_t batch, uint64_t n);

/* Batched Haar-to-Walsh map <- chw::haar_walsh_forward_inplace
 * (transforms.hpp:190-198): the dyadic WHT of each scale block
 * [2^j, 2^(j+1)), j = 1..m-1, of every row.  Device buffers, in == out allowed. */
chw_status chw_b200_haar_walsh_forward(const void* in, void* out, chw_dtype dtype, int64_t batch, uint64_t n,
                                       chw_mode mode, void* stream);

/* Host-buffer variants (synchronous). */
chw_status chw_b200_haar_inverse_host(const void* in_host, void* out_host, chw_dtype dtype, int64_t batch,
                                      uint64_t n, chw_mode mode);
chw_status chw_b200_haar_walsh_forward_host(const void* in_host, void* out_host, chw_dtype dtype,
                                            int64_t batch, uint64_t n, chw_mode mode);
/* Host-buffer Haar transform (synchronous). */
chw_status chw_b200_haar_forward_host(const void* in_host, void* out_host, chw_dtype dtype, int64_t batch,
                                      uint64_t n, chw_mode mode);

/* Host-buffer call with an explicit output order. */
chw_status chw_b200_forward_host_ordered(const void* in_host, void* out_host, chw_dtype dtype,
                                         int64_t batch, uint64_t n, chw_mode mode, chw_order order);

/* Device path of chw::normalize_inplace (proj/include/chw/transforms.hpp:202-210)
 * on `batch` rows of n = 2^m elements: x *= 1/sqrt(2^m), the reference's own
 * constant and one multiply per element (f64 bit-exact; F32 also accepted).
 * n != 2^m -> CHW_ERR_LENGTH with the reference's message.  Asynchronous on
 * `stream`; the buffer must be 16-byte aligned. */
chw_status chw_b200_normalize(void* x, chw_dtype dtype, int64_t batch, uint64_t n, int m, void* stream);

/* parallel_execute_inplace(x, workers, mode) on a DEVICE buffer of one signal.
 * Validation as parallel.cpp:84-91; the pool is replaced by the GPU. */
chw_status chw_b200_parallel_execute(void* x, chw_dtype dtype, uint64_t n, int workers,
                                     chw_mode mode, void* stream);

/* Closed-form OpTally of one length-n transform:
 *   op 0 = chw_forward  : adds m*2^m, mults m*2^m (Orthonormal) or 0
 *   op 1 = haar_forward : adds 2(n-1), mults 2(n-1) (Orthonormal) or 0
 *   op 2 = normalize    : adds 0, mults n
 * n == 1 leaves both at 0. */
chw_status chw_b200_op_tally(int op, uint64_t n, chw_mode mode, uint64_t* additions,
                             uint64_t* multiplications);

const char* chw_b200_status_string(chw_status s);
const char* chw_b200_last_error(void);

/* Number of kernels this library has launched in this process (all devices). */
uint64_t chw_b200_launch_count(void);

/* Name of the kernel family the dispatcher picks for (dtype, n): "k1-tuned",
 * "k1-generic", "k4-multipass:<passes>", ... (for reports; never NULL). */
const char* chw_b200_plan_name(chw_dtype dtype, uint64_t n);

int chw_b200_abi_version(void);

/* 1 if `p` is device (or managed) memory of the current CUDA context, 0 for
 * host memory (pinned or pageable).  Lets the C++ shim route spans without
 * including CUDA headers. */
int chw_b200_is_device_pointer(const void* p);

/* cudaStreamSynchronize(stream) (NULL = legacy default stream). */
chw_status chw_b200_stream_synchronize(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CHW_B200_H */
