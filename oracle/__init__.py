"""oracle — CPU checkers for the CHW hot path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the timed
CPU baseline; the product (paper_1609_06641_b200) never touches it.

Two backends, same numpy-facing API:
  * "port": liboracle_chw.so — the plain-C restatement in chw_oracle.c,
    pinned against tests/golden/golden.npz (generated from the reference);
  * "reference": _ref/libchw_ref.so — the UNMODIFIED reference headers and
    src/parallel.cpp compiled by oracle/Makefile (present wherever it was built;
    the .so travels to the GPU box with the repo snapshot).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle_chw.so")
REF_PATH = os.path.join(HERE, "_ref", "libchw_ref.so")

ORTHONORMAL, UNNORMALIZED = 0, 1

_c = ctypes
_dp = _c.POINTER(_c.c_double)
_ip = _c.POINTER(_c.c_int64)
_up = _c.POINTER(_c.c_uint64)


def build() -> None:
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Backend:
    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = _c.CDLL(path)

    def fn(self, name: str):
        return getattr(self.lib, self.prefix + name)


_port = None
_ref = None


def port() -> _Backend:
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            build()
        b = _Backend(PORT_PATH, "chw_oracle_")
        for name in ("chw_forward_f64", "haar_forward_f64"):
            b.fn(name).argtypes = [_dp, _c.c_size_t, _c.c_int, _up, _up]
        for name in ("chw_forward_i64", "haar_forward_i64"):
            b.fn(name).argtypes = [_ip, _c.c_size_t, _c.c_int, _up, _up]
        for name in ("fwht_natural_f64", "fwht_dyadic_f64", "haar_walsh_forward_f64",
                     "haar_inverse_f64", "network_f64"):
            b.fn(name).argtypes = [_dp, _c.c_size_t, _c.c_int]
        for name in ("fwht_natural_i64", "fwht_dyadic_i64", "haar_walsh_forward_i64",
                     "haar_inverse_i64"):
            b.fn(name).argtypes = [_ip, _c.c_size_t, _c.c_int]
        b.fn("normalize_f64").argtypes = [_dp, _c.c_size_t, _c.c_int]
        b.fn("chw_batch_f64").argtypes = [_dp, _c.c_size_t, _c.c_size_t, _c.c_int, _c.c_int]
        b.fn("chw_batch_i64").argtypes = [_ip, _c.c_size_t, _c.c_size_t, _c.c_int, _c.c_int]
        b.fn("bit_reverse").argtypes = [_c.c_uint64, _c.c_int]
        b.fn("bit_reverse").restype = _c.c_uint64
        _port = b
    return _port


def have_reference() -> bool:
    return os.path.exists(REF_PATH)


def reference() -> _Backend:
    global _ref
    if _ref is None:
        if not have_reference():
            raise FileNotFoundError(f"{REF_PATH} not built (reference tree absent when building)")
        b = _Backend(REF_PATH, "ref_")
        for name in ("chw_forward_f64", "haar_forward_f64"):
            b.fn(name).argtypes = [_dp, _c.c_size_t, _c.c_int, _up, _up]
        for name in ("chw_forward_i64", "haar_forward_i64"):
            b.fn(name).argtypes = [_ip, _c.c_size_t, _c.c_int, _up, _up]
        for name in ("fwht_natural_f64", "fwht_dyadic_f64", "haar_walsh_forward_f64",
                     "haar_inverse_f64"):
            b.fn(name).argtypes = [_dp, _c.c_size_t, _c.c_int]
        for name in ("fwht_natural_i64", "fwht_dyadic_i64", "haar_walsh_forward_i64",
                     "haar_inverse_i64"):
            b.fn(name).argtypes = [_ip, _c.c_size_t, _c.c_int]
        b.fn("normalize_f64").argtypes = [_dp, _c.c_size_t, _c.c_int, _up]
        b.fn("parallel_execute_f64").argtypes = [_dp, _c.c_size_t, _c.c_int, _c.c_int, _up, _up]
        b.fn("parallel_execute_i64").argtypes = [_ip, _c.c_size_t, _c.c_int, _c.c_int, _up, _up]
        b.fn("chw_batch_f64").argtypes = [_dp, _c.c_size_t, _c.c_size_t, _c.c_int, _c.c_int]
        b.fn("chw_batch_i64").argtypes = [_ip, _c.c_size_t, _c.c_size_t, _c.c_int, _c.c_int]
        b.fn("last_error").restype = _c.c_char_p
        b.fn("hardware_concurrency").restype = _c.c_int
        _ref = b
    return _ref


def _ptr(a: np.ndarray):
    if a.dtype == np.float64:
        return a.ctypes.data_as(_dp)
    if a.dtype == np.int64:
        return a.ctypes.data_as(_ip)
    raise TypeError(a.dtype)


def _sfx(a: np.ndarray) -> str:
    return "f64" if a.dtype == np.float64 else "i64"


class OracleError(ValueError):
    pass


def _rc(rc: int, what: str) -> None:
    if rc != 0:
        raise OracleError(f"{what}: oracle returned {rc}")


def chw_forward(x, mode: int = ORTHONORMAL, backend: str = "port", tally: bool = False):
    """chw_forward_inplace (transforms.hpp:126-143) on a copy of a 1-D signal."""
    a = np.array(x, copy=True)
    if a.dtype not in (np.float64, np.int64):
        a = a.astype(np.float64)
    b = port() if backend == "port" else reference()
    adds = _c.c_uint64(0)
    mults = _c.c_uint64(0)
    rc = b.fn("chw_forward_" + _sfx(a))(_ptr(a), a.size, mode, _c.byref(adds), _c.byref(mults))
    _rc(rc, "chw_forward")
    return (a, adds.value, mults.value) if tally else a


def chw_batch(x: np.ndarray, mode: int = ORTHONORMAL, backend: str = "port", threads: int = 0) -> np.ndarray:
    """Row-wise chw_forward over a [rows][n] array (copy), threaded over rows."""
    a = np.ascontiguousarray(x)
    a = np.array(a, dtype=np.float64 if a.dtype != np.int64 else np.int64, copy=True)
    rows, n = a.shape
    b = port() if backend == "port" else reference()
    _rc(b.fn("chw_batch_" + _sfx(a))(_ptr(a), rows, n, mode, threads), "chw_batch")
    return a


def chw_batch_inplace(a: np.ndarray, mode: int = ORTHONORMAL, backend: str = "port", threads: int = 0) -> None:
    rows, n = a.shape
    b = port() if backend == "port" else reference()
    _rc(b.fn("chw_batch_" + _sfx(a))(_ptr(a), rows, n, mode, threads), "chw_batch")


def simple(name: str, x, mode: int = UNNORMALIZED, backend: str = "port") -> np.ndarray:
    """fwht_natural / fwht_dyadic / haar_walsh_forward / haar_inverse / network."""
    a = np.array(x, copy=True)
    if a.dtype not in (np.float64, np.int64):
        a = a.astype(np.float64)
    b = port() if backend == "port" else reference()
    _rc(b.fn(f"{name}_{_sfx(a)}")(_ptr(a), a.size, mode), name)
    return a


def haar_forward(x, mode: int = UNNORMALIZED, backend: str = "port", tally: bool = False):
    a = np.array(x, copy=True)
    b = port() if backend == "port" else reference()
    adds = _c.c_uint64(0)
    mults = _c.c_uint64(0)
    _rc(b.fn("haar_forward_" + _sfx(a))(_ptr(a), a.size, mode, _c.byref(adds), _c.byref(mults)),
        "haar_forward")
    return (a, adds.value, mults.value) if tally else a


def bit_reverse(v: int, bits: int) -> int:
    return int(port().fn("bit_reverse")(v, bits))


def online_cores() -> int:
    return os.cpu_count() or 1
