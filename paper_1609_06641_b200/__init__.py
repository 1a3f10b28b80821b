"""paper_1609_06641_b200 — B200-native batched CHW (dyadic-order Walsh-Hadamard).

Python host-side mirror of the reference's transform API
(/root/reference/proj/include/chw/transforms.hpp, parallel.hpp, op_tally.hpp)
over the C ABI in include/chw_b200.h, implemented by the sm_100a kernels in
csrc/ and loaded from the in-tree libchw_b200.so.

There is NO CPU fallback: every transform runs on the GPU through the C ABI,
and importing this package raises if the shared library is missing.  torch is
used only for device memory and streams (plumbing).

Names and argument meaning follow the reference:
    ScalingMode.Orthonormal / Unnormalized        common.hpp:15
    chw_forward_inplace(x, mode, tally=None)      transforms.hpp:126-143
    chw_forward(x, mode, tally=None)              transforms.hpp:226-230
    parallel_execute(_inplace)(x, workers, mode)  parallel.hpp:16-22
    normalize(_inplace) / normalized              transforms.hpp:202-210, 250-260
    OpTally                                       op_tally.hpp:12-22
    stage_blocks(m, r) / BlockSlice               transforms.hpp:18-42
    bit_reverse, natural_to_dyadic                orderings.hpp:45-78
Errors: std::invalid_argument -> ValueError (same message text);
chw::ResourceError -> ResourceError.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field
from typing import List, Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
# CHW_B200_LIB overrides the library path (same-box A/B of alternative builds).
LIB_PATH = os.environ.get("CHW_B200_LIB") or os.path.join(_HERE, "libchw_b200.so")

# C-ABI enums (include/chw_b200.h)
CHW_OK = 0
CHW_ERR_LENGTH = 1
CHW_ERR_MODE = 2
CHW_ERR_ARGUMENT = 3
CHW_ERR_UNSUPPORTED = 4
CHW_ERR_WORKSPACE = 5
CHW_ERR_CUDA = 6
CHW_ERR_NO_DEVICE = 7
CHW_ERR_RESOURCE = 8
CHW_ERR_STRUCTURE = 9

DTYPE_F64, DTYPE_F32, DTYPE_BF16, DTYPE_I64 = 0, 1, 2, 3
ORDER_DYADIC, ORDER_NATURAL, ORDER_SEQUENCY = 0, 1, 2

# Every symbol include/chw_b200.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "chw_b200_forward",
    "chw_b200_forward_ordered",
    "chw_b200_workspace_bytes",
    "chw_b200_forward_host",
    "chw_b200_parallel_execute",
    "chw_b200_op_tally",
    "chw_b200_status_string",
    "chw_b200_last_error",
    "chw_b200_launch_count",
    "chw_b200_plan_name",
    "chw_b200_abi_version",
    "chw_b200_is_device_pointer",
    "chw_b200_haar_forward",
    "chw_b200_haar_workspace_bytes",
    "chw_b200_haar_forward_host",
    "chw_b200_workspace_bytes_ordered",
    "chw_b200_forward_host_ordered",
    "chw_b200_haar_inverse",
    "chw_b200_haar_inverse_workspace_bytes",
    "chw_b200_haar_walsh_forward",
    "chw_b200_haar_inverse_host",
    "chw_b200_haar_walsh_forward_host",
    "chw_b200_stream_synchronize",
    "chw_b200_normalize",
)


class ScalingMode(enum.IntEnum):
    """chw::ScalingMode (common.hpp:15)."""

    Orthonormal = 0
    Unnormalized = 1


class ResourceError(RuntimeError):
    """chw::ResourceError (errors.hpp:32-36)."""


class StructureError(RuntimeError):
    """chw::StructureError (errors.hpp:15-19)."""


class ChwCudaError(RuntimeError):
    """CUDA runtime failure inside the library."""


@dataclass
class OpTally:
    """chw::OpTally (op_tally.hpp:12-22): additions/subtractions and scaling
    multiplications.  Filled in closed form (the GPU does not count)."""

    additions: int = 0
    multiplications: int = 0

    def reset(self) -> None:
        self.additions = 0
        self.multiplications = 0


@dataclass(frozen=True)
class BlockSlice:
    """chw::BlockSlice (transforms.hpp:20-25)."""

    offset: int = 0
    size: int = 0


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    c = ctypes
    lib.chw_b200_forward.argtypes = [c.c_void_p, c.c_void_p, c.c_int, c.c_int64, c.c_uint64,
                                     c.c_int, c.c_void_p, c.c_size_t, c.c_void_p]
    lib.chw_b200_forward.restype = c.c_int
    lib.chw_b200_forward_ordered.argtypes = [c.c_void_p, c.c_void_p, c.c_int, c.c_int64,
                                             c.c_uint64, c.c_int, c.c_int, c.c_void_p,
                                             c.c_size_t, c.c_void_p]
    lib.chw_b200_forward_ordered.restype = c.c_int
    lib.chw_b200_workspace_bytes.argtypes = [c.c_int, c.c_int64, c.c_uint64]
    lib.chw_b200_workspace_bytes.restype = c.c_size_t
    lib.chw_b200_forward_host.argtypes = [c.c_void_p, c.c_void_p, c.c_int, c.c_int64,
                                          c.c_uint64, c.c_int]
    lib.chw_b200_forward_host.restype = c.c_int
    lib.chw_b200_parallel_execute.argtypes = [c.c_void_p, c.c_int, c.c_uint64, c.c_int, c.c_int,
                                              c.c_void_p]
    lib.chw_b200_parallel_execute.restype = c.c_int
    lib.chw_b200_op_tally.argtypes = [c.c_int, c.c_uint64, c.c_int, c.POINTER(c.c_uint64),
                                      c.POINTER(c.c_uint64)]
    lib.chw_b200_op_tally.restype = c.c_int
    lib.chw_b200_status_string.argtypes = [c.c_int]
    lib.chw_b200_status_string.restype = c.c_char_p
    lib.chw_b200_last_error.argtypes = []
    lib.chw_b200_last_error.restype = c.c_char_p
    lib.chw_b200_launch_count.argtypes = []
    lib.chw_b200_launch_count.restype = c.c_uint64
    lib.chw_b200_plan_name.argtypes = [c.c_int, c.c_uint64]
    lib.chw_b200_plan_name.restype = c.c_char_p
    lib.chw_b200_abi_version.argtypes = []
    lib.chw_b200_abi_version.restype = c.c_int
    lib.chw_b200_haar_forward.argtypes = [c.c_void_p, c.c_void_p, c.c_int, c.c_int64, c.c_uint64,
                                          c.c_int, c.c_void_p, c.c_size_t, c.c_void_p]
    lib.chw_b200_haar_forward.restype = c.c_int
    lib.chw_b200_haar_workspace_bytes.argtypes = [c.c_int, c.c_int64, c.c_uint64]
    lib.chw_b200_haar_workspace_bytes.restype = c.c_size_t
    lib.chw_b200_haar_forward_host.argtypes = [c.c_void_p, c.c_void_p, c.c_int, c.c_int64, c.c_uint64, c.c_int]
    lib.chw_b200_haar_forward_host.restype = c.c_int
    lib.chw_b200_workspace_bytes_ordered.argtypes = [c.c_int, c.c_int64, c.c_uint64, c.c_int]
    lib.chw_b200_workspace_bytes_ordered.restype = c.c_size_t
    lib.chw_b200_forward_host_ordered.argtypes = [c.c_void_p, c.c_void_p, c.c_int, c.c_int64, c.c_uint64,
                                                  c.c_int, c.c_int]
    lib.chw_b200_forward_host_ordered.restype = c.c_int
    lib.chw_b200_haar_inverse.argtypes = [c.c_void_p, c.c_void_p, c.c_int, c.c_int64, c.c_uint64,
                                          c.c_int, c.c_void_p, c.c_size_t, c.c_void_p]
    lib.chw_b200_haar_inverse.restype = c.c_int
    lib.chw_b200_haar_inverse_workspace_bytes.argtypes = [c.c_int, c.c_int64, c.c_uint64]
    lib.chw_b200_haar_inverse_workspace_bytes.restype = c.c_size_t
    lib.chw_b200_haar_walsh_forward.argtypes = [c.c_void_p, c.c_void_p, c.c_int, c.c_int64, c.c_uint64,
                                                c.c_int, c.c_void_p]
    lib.chw_b200_haar_walsh_forward.restype = c.c_int
    for name in ("chw_b200_haar_inverse_host", "chw_b200_haar_walsh_forward_host"):
        getattr(lib, name).argtypes = [c.c_void_p, c.c_void_p, c.c_int, c.c_int64, c.c_uint64, c.c_int]
        getattr(lib, name).restype = c.c_int
    lib.chw_b200_is_device_pointer.argtypes = [c.c_void_p]
    lib.chw_b200_is_device_pointer.restype = c.c_int
    lib.chw_b200_stream_synchronize.argtypes = [c.c_void_p]
    lib.chw_b200_stream_synchronize.restype = c.c_int
    lib.chw_b200_normalize.argtypes = [c.c_void_p, c.c_int, c.c_int64, c.c_uint64, c.c_int, c.c_void_p]
    lib.chw_b200_normalize.restype = c.c_int
    return lib


lib = _load()


def _check(status: int) -> None:
    if status == CHW_OK:
        return
    msg = lib.chw_b200_last_error().decode()
    if status in (CHW_ERR_LENGTH, CHW_ERR_MODE, CHW_ERR_ARGUMENT, CHW_ERR_WORKSPACE):
        raise ValueError(msg)
    if status == CHW_ERR_RESOURCE:
        raise ResourceError(msg)
    if status == CHW_ERR_STRUCTURE:
        raise StructureError(msg)
    if status == CHW_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise ChwCudaError(f"{lib.chw_b200_status_string(status).decode()}: {msg}")


def level_of(n: int) -> int:
    """common.hpp:25."""
    return n.bit_length() - 1


def is_pow2(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


def _tally_add(tally: Optional[OpTally], op: int, n: int, mode: int, rows: int = 1) -> None:
    if tally is None or n <= 1:
        return
    a = ctypes.c_uint64()
    m = ctypes.c_uint64()
    _check(lib.chw_b200_op_tally(op, n, int(mode), ctypes.byref(a), ctypes.byref(m)))
    tally.additions += a.value * rows
    tally.multiplications += m.value * rows


# --------------------------------------------------------------------------
# torch plumbing (device buffers and streams)
# --------------------------------------------------------------------------
def _torch():
    import torch  # noqa: WPS433 — plumbing only

    return torch


def dtype_code(t) -> int:
    torch = _torch()
    table = {torch.float64: DTYPE_F64, torch.float32: DTYPE_F32, torch.bfloat16: DTYPE_BF16,
             torch.int64: DTYPE_I64}
    if t.dtype not in table:
        raise ValueError(f"chw_forward: unsupported dtype {t.dtype} (float64, float32, bfloat16, int64)")
    return table[t.dtype]


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def chw_forward_batched_(x, mode: ScalingMode = ScalingMode.Orthonormal, tally: Optional[OpTally] = None,
                         out=None, stream=None, workspace=None, order: int = ORDER_DYADIC):
    """Batched in-place (or out-of-place via `out`) CHW over the LAST dim of a
    contiguous CUDA tensor — the batched overload the reference lacks
    (SURVEY §8b item 3).  Returns the output tensor."""
    torch = _torch()
    if not x.is_cuda:
        raise ValueError("chw_forward: expected a CUDA tensor (use chw_forward_host for host data)")
    if not x.is_contiguous():
        raise ValueError("chw_forward: expected a contiguous tensor")
    n = int(x.shape[-1]) if x.dim() > 0 else 1
    batch = x.numel() // n if n > 0 else 1
    dst = x if out is None else out
    if out is not None and (out.shape != x.shape or out.dtype != x.dtype or not out.is_contiguous()):
        raise ValueError("chw_forward: `out` must match the input's shape, dtype and layout")
    ws_ptr, ws_bytes = (None, 0)
    if workspace is not None:
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    with torch.cuda.device(x.device):
        _check(lib.chw_b200_forward_ordered(x.data_ptr(), dst.data_ptr(), dtype_code(x), batch, n,
                                            int(mode), int(order), ws_ptr, ws_bytes,
                                            _stream_ptr(stream)))
    _tally_add(tally, 0, n, mode, batch)
    return dst


def chw_forward_inplace(x, mode: ScalingMode = ScalingMode.Orthonormal, tally: Optional[OpTally] = None,
                        scratch=None):
    """transforms.hpp:126-143 on one signal (1-D) or a batch of rows (last dim).
    CUDA tensors are transformed on their device; numpy arrays / host tensors go
    through the synchronous host path (chw_b200_forward_host).  `scratch` is
    accepted for signature parity (the GPU manages its own workspace)."""
    torch = _torch()
    if isinstance(x, torch.Tensor) and x.is_cuda:
        chw_forward_batched_(x, mode, tally)
        torch.cuda.current_stream().synchronize()  # reference calls are synchronous
        return x
    return chw_forward_host_(x, mode, tally)


def _ordered_inplace(x, mode, tally, order):
    torch = _torch()
    if isinstance(x, torch.Tensor) and x.is_cuda:
        chw_forward_batched_(x, mode, tally, order=order)
        torch.cuda.current_stream().synchronize()
        return x
    t = torch.as_tensor(x)
    d = t.cuda()
    chw_forward_batched_(d, mode, tally, order=order)
    res = d.cpu()
    if isinstance(x, torch.Tensor):
        x.copy_(res)
    else:
        import numpy as np

        np.copyto(x, res.numpy())
    return x


def fwht_natural_inplace(x, mode: ScalingMode, tally: Optional[OpTally] = None):
    """transforms.hpp:147-172: WHT in natural (Sylvester) order = the CHW
    network without the final bit reversal (f2/f3)."""
    return _ordered_inplace(x, mode, tally, ORDER_NATURAL)


def fwht_natural(x, mode: ScalingMode, tally: Optional[OpTally] = None):
    torch = _torch()
    y = x.clone() if isinstance(x, torch.Tensor) else __import__("numpy").array(x, copy=True)
    return fwht_natural_inplace(y, mode, tally)


def fwht_dyadic_inplace(x, mode: ScalingMode, tally: Optional[OpTally] = None):
    """transforms.hpp:177-185: natural WHT + bit reversal == chw_forward."""
    return _ordered_inplace(x, mode, tally, ORDER_DYADIC)


def fwht_dyadic(x, mode: ScalingMode, tally: Optional[OpTally] = None):
    torch = _torch()
    y = x.clone() if isinstance(x, torch.Tensor) else __import__("numpy").array(x, copy=True)
    return fwht_dyadic_inplace(y, mode, tally)


def chw_forward_sequency(x, mode: ScalingMode = ScalingMode.Orthonormal, tally: Optional[OpTally] = None):
    """chw_forward followed by apply_permutation(dyadic_to_sequency(m), .)
    (orderings.hpp:82-102, the CLI's --order sequency, chw_main.cpp:76-89)."""
    torch = _torch()
    y = x.clone() if isinstance(x, torch.Tensor) else __import__("numpy").array(x, copy=True)
    return _ordered_inplace(y, mode, tally, ORDER_SEQUENCY)


def chw_forward(x, mode: ScalingMode = ScalingMode.Orthonormal, tally: Optional[OpTally] = None):
    """transforms.hpp:226-230: out-of-place wrapper (copy, then in place)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        y = x.clone()
    else:
        import numpy as np

        y = np.array(x, copy=True)
    return chw_forward_inplace(y, mode, tally)


def chw_forward_host_(x, mode: ScalingMode = ScalingMode.Orthonormal, tally: Optional[OpTally] = None,
                      out=None):
    """In-place transform of HOST memory (numpy array or CPU tensor, last dim =
    signal) through chw_b200_forward_host: H2D, kernel, D2H, synchronous."""
    import numpy as np

    torch = _torch()
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            raise ValueError("chw_forward_host: expected host memory")
        arr_ptr = x.data_ptr()
        code = dtype_code(x)
        n = int(x.shape[-1]) if x.dim() > 0 else 1
        numel = x.numel()
        if not x.is_contiguous():
            raise ValueError("chw_forward: expected a contiguous tensor")
        if out is not None and (not isinstance(out, torch.Tensor) or out.is_cuda or out.shape != x.shape
                                or out.dtype != x.dtype or not out.is_contiguous()):
            raise ValueError("chw_forward: `out` must be a host tensor matching the input's shape, "
                             "dtype and layout")
        dst_ptr = out.data_ptr() if out is not None else arr_ptr
    else:
        if not isinstance(x, np.ndarray):
            raise ValueError("chw_forward: expected a numpy array or tensor")
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("chw_forward: expected a contiguous array")
        codes = {np.dtype(np.float64): DTYPE_F64, np.dtype(np.float32): DTYPE_F32,
                 np.dtype(np.int64): DTYPE_I64}
        if x.dtype not in codes:
            raise ValueError(f"chw_forward: unsupported dtype {x.dtype}")
        code = codes[x.dtype]
        arr_ptr = x.ctypes.data
        n = int(x.shape[-1]) if x.ndim > 0 else 1
        numel = x.size
        if out is not None and (not isinstance(out, np.ndarray) or out.shape != x.shape
                                or out.dtype != x.dtype or not out.flags["C_CONTIGUOUS"]
                                or not out.flags["WRITEABLE"]):
            raise ValueError("chw_forward: `out` must be a writable array matching the input's shape, "
                             "dtype and layout")
        dst_ptr = out.ctypes.data if out is not None else arr_ptr
    batch = numel // n if n > 0 else 0
    if n == 0:
        batch = 1
    _check(lib.chw_b200_forward_host(arr_ptr, dst_ptr, code, batch, n, int(mode)))
    _tally_add(tally, 0, n, mode, batch)
    return x if out is None else out


def haar_forward_batched_(x, mode: ScalingMode = ScalingMode.Unnormalized, tally: Optional[OpTally] = None,
                          out=None, stream=None):
    """Batched Haar transform Psi_m (transforms.hpp:49-80) over the last dim of
    a contiguous CUDA tensor (float64, float32 or int64), in place or into `out`."""
    torch = _torch()
    if not x.is_cuda or not x.is_contiguous():
        raise ValueError("haar_forward: expected a contiguous CUDA tensor")
    n = int(x.shape[-1]) if x.dim() > 0 else 1
    batch = x.numel() // n if n > 0 else 1
    dst = x if out is None else out
    with torch.cuda.device(x.device):
        _check(lib.chw_b200_haar_forward(x.data_ptr(), dst.data_ptr(), dtype_code(x), batch, n, int(mode),
                                         None, 0, _stream_ptr(stream)))
    _tally_add(tally, 1, n, mode, batch)
    return dst


def haar_forward_inplace(x, mode: ScalingMode, tally: Optional[OpTally] = None, scratch=None):
    """transforms.hpp:49-80 on a signal (1-D) or rows (last dim); CUDA tensors
    in place on their device, host arrays staged through the device."""
    torch = _torch()
    if isinstance(x, torch.Tensor) and x.is_cuda:
        haar_forward_batched_(x, mode, tally)
        torch.cuda.current_stream().synchronize()
        return x
    import numpy as np

    a = x.numpy() if isinstance(x, torch.Tensor) else x
    if not isinstance(a, np.ndarray) or not a.flags["C_CONTIGUOUS"]:
        raise ValueError("haar_forward: expected a contiguous array")
    codes = {np.dtype(np.float64): DTYPE_F64, np.dtype(np.float32): DTYPE_F32, np.dtype(np.int64): DTYPE_I64}
    if a.dtype not in codes:
        raise ValueError(f"haar_forward: unsupported dtype {a.dtype}")
    n = int(a.shape[-1]) if a.ndim else 1
    batch = a.size // n if n else 1
    _check(lib.chw_b200_haar_forward_host(a.ctypes.data, a.ctypes.data, codes[a.dtype], batch, n, int(mode)))
    _tally_add(tally, 1, n, mode, batch)
    return x


def haar_forward(x, mode: ScalingMode, tally: Optional[OpTally] = None):
    """transforms.hpp:214-218: by-value wrapper."""
    torch = _torch()
    y = x.clone() if isinstance(x, torch.Tensor) else __import__("numpy").array(x, copy=True)
    return haar_forward_inplace(y, mode, tally)


def _device_rows(x):
    """(tensor on device, writer-back) for CUDA tensors, numpy arrays or CPU tensors."""
    torch = _torch()
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x, None
    t = torch.as_tensor(x)
    d = t.cuda()

    def back():
        res = d.cpu()
        if isinstance(x, torch.Tensor):
            x.copy_(res)
        else:
            import numpy as np

            np.copyto(x, res.numpy())

    return d, back


def haar_inverse_inplace(x, mode: ScalingMode, scratch=None):
    """transforms.hpp:85-120 (int64: StructureError on a non-forward output)."""
    torch = _torch()
    d, back = _device_rows(x)
    n = int(d.shape[-1]) if d.dim() > 0 else 1
    batch = d.numel() // n if n > 0 else 1
    with torch.cuda.device(d.device):
        _check(lib.chw_b200_haar_inverse(d.data_ptr(), d.data_ptr(), dtype_code(d), batch, n, int(mode),
                                         None, 0, _stream_ptr(None)))
    torch.cuda.current_stream().synchronize()
    if back:
        back()
    return x


def haar_inverse(y, mode: ScalingMode):
    torch = _torch()
    x = y.clone() if isinstance(y, torch.Tensor) else __import__("numpy").array(y, copy=True)
    return haar_inverse_inplace(x, mode)


def haar_walsh_forward_inplace(x, mode: ScalingMode, tally: Optional[OpTally] = None):
    """transforms.hpp:190-198: dyadic WHT of each scale block [2^j, 2^(j+1))."""
    torch = _torch()
    d, back = _device_rows(x)
    n = int(d.shape[-1]) if d.dim() > 0 else 1
    batch = d.numel() // n if n > 0 else 1
    with torch.cuda.device(d.device):
        _check(lib.chw_b200_haar_walsh_forward(d.data_ptr(), d.data_ptr(), dtype_code(d), batch, n, int(mode),
                                               _stream_ptr(None)))
    torch.cuda.current_stream().synchronize()
    if tally is not None and n > 2:
        for j in range(1, level_of(n)):
            _tally_add(tally, 0, 1 << j, mode, batch)
    if back:
        back()
    return x


def haar_walsh_forward(h, mode: ScalingMode, tally: Optional[OpTally] = None):
    torch = _torch()
    x = h.clone() if isinstance(h, torch.Tensor) else __import__("numpy").array(h, copy=True)
    return haar_walsh_forward_inplace(x, mode, tally)


def parallel_execute_inplace(x, workers: int, mode: ScalingMode, tally: Optional[OpTally] = None):
    """parallel.hpp:16-17 / parallel.cpp:84-97: same validation and the same
    result as the serial transform; the thread pool is replaced by the GPU."""
    torch = _torch()
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        t = torch.as_tensor(x)
        d = t.cuda()
        parallel_execute_inplace(d, workers, mode, tally)
        res = d.cpu()
        if isinstance(x, torch.Tensor):
            x.copy_(res)
            return x
        import numpy as np

        np.copyto(x, res.numpy())
        return x
    n = x.numel()
    with torch.cuda.device(x.device):
        _check(lib.chw_b200_parallel_execute(x.data_ptr(), dtype_code(x), n, int(workers), int(mode),
                                             _stream_ptr(None)))
    torch.cuda.current_stream().synchronize()
    _tally_add(tally, 0, n, mode)
    return x


def parallel_execute(x, workers: int, mode: ScalingMode, tally: Optional[OpTally] = None):
    """parallel.hpp:20-22: by-value wrapper."""
    torch = _torch()
    y = x.clone() if isinstance(x, torch.Tensor) else __import__("numpy").array(x, copy=True)
    return parallel_execute_inplace(y, workers, mode, tally)


def normalize_inplace(x, m: int, tally: Optional[OpTally] = None):
    """transforms.hpp:202-210: x *= 1/sqrt(2^m) on an Unnormalized output."""
    n = x.shape[-1] if hasattr(x, "shape") and len(x.shape) else len(x)
    if m < 0 or n != (1 << m):
        raise ValueError(f"normalize: signal length {n} does not match level {m}")
    import math

    torch = _torch()
    rows = 1
    if isinstance(x, torch.Tensor) and x.is_cuda:
        # Device path: one multiply per element in the library's kernel
        # (chw_b200_normalize; bit-identical to the reference loop for f64).
        if not x.is_contiguous():
            raise ValueError("normalize: expected a contiguous tensor")
        rows = x.numel() // n if n else 0
        with torch.cuda.device(x.device):
            _check(lib.chw_b200_normalize(x.data_ptr(), dtype_code(x), rows, n, m,
                                          _stream_ptr(None)))
        torch.cuda.current_stream().synchronize()
    else:
        if hasattr(x, "shape") and len(x.shape) > 1:
            rows = int(__import__("numpy").prod(x.shape[:-1]))
        x *= 1.0 / math.sqrt(math.ldexp(1.0, m))
    if tally is not None:
        tally.multiplications += int(n) * rows
    return x


def normalized(x, m: int, tally: Optional[OpTally] = None):
    """transforms.hpp:250-260 (int64 input is converted to double)."""
    import numpy as np

    torch = _torch()
    if isinstance(x, torch.Tensor):
        y = x.to(torch.float64).clone()
    else:
        y = np.array(x, dtype=np.float64, copy=True)
    return normalize_inplace(y, m, tally)


def stage_blocks(m: int, r: int) -> List[BlockSlice]:
    """transforms.hpp:30-42 (cascade geometry, the reference's own contract)."""
    if r < 1 or r > m - 1:
        raise ValueError(f"stage_blocks: stage {r} out of range for m={m}")
    size = 1 << (m - r)
    return [BlockSlice(q * 2 * size + size, size) for q in range(1 << (r - 1))]


def bit_reverse(v: int, bits: int) -> int:
    """orderings.hpp:45-52."""
    r = 0
    for _ in range(bits):
        r = (r << 1) | (v & 1)
        v >>= 1
    return r


def natural_to_dyadic(m: int) -> List[int]:
    """orderings.hpp:70-78 (map[i] = bit_reverse(i, m))."""
    if m < 0 or m > 31:
        raise ValueError(f"natural_to_dyadic: level {m} out of range")
    return [bit_reverse(i, m) for i in range(1 << m)]


def workspace_bytes(dtype: int, batch: int, n: int) -> int:
    return int(lib.chw_b200_workspace_bytes(dtype, batch, n))


def workspace_bytes_ordered(dtype: int, batch: int, n: int, order: int) -> int:
    return int(lib.chw_b200_workspace_bytes_ordered(dtype, batch, n, order))


def plan_name(dtype: int, n: int) -> str:
    return lib.chw_b200_plan_name(dtype, n).decode()


def launch_count() -> int:
    return int(lib.chw_b200_launch_count())


__all__ = [
    "ScalingMode", "OpTally", "BlockSlice", "ResourceError", "ChwCudaError",
    "chw_forward", "chw_forward_inplace", "chw_forward_batched_", "chw_forward_host_",
    "haar_forward", "haar_forward_inplace", "haar_forward_batched_",
    "haar_inverse", "haar_inverse_inplace", "haar_walsh_forward", "haar_walsh_forward_inplace",
    "StructureError", "fwht_natural", "fwht_natural_inplace", "fwht_dyadic", "fwht_dyadic_inplace", "chw_forward_sequency",
    "parallel_execute", "parallel_execute_inplace", "normalize_inplace", "normalized",
    "stage_blocks", "bit_reverse", "natural_to_dyadic", "workspace_bytes", "workspace_bytes_ordered", "plan_name",
    "launch_count", "lib", "LIB_PATH", "EXPORTED_SYMBOLS",
]
