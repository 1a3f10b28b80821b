"""C-ABI boundary checks that need no GPU: the in-tree library loads, exports
every function include/chw_b200.h declares, and validates like the reference
(common.hpp:31-46, parallel.cpp:88-91) before touching any device."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1609_06641_b200 as chw

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "chw_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(chw_b200_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_what_the_package_binds():
    assert declared_functions() == sorted(chw.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", chw.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (chw_b200_\w+)", out))
    missing = [s for s in declared_functions() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(chw.LIB_PATH)
    for s in declared_functions():
        assert getattr(lib, s) is not None


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", chw.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_abi_version():
    assert chw.lib.chw_b200_abi_version() == 1


@pytest.mark.parametrize("n", [0, 3, 6, 1000, 12345])
def test_length_validation_message(n):
    rc = chw.lib.chw_b200_forward(None, None, chw.DTYPE_F64, 1, n, 0, None, 0, None)
    assert rc == chw.CHW_ERR_LENGTH
    assert chw.lib.chw_b200_last_error().decode() == f"chw_forward: length {n} is not a power of two"


def test_mode_validation_message():
    rc = chw.lib.chw_b200_forward(None, None, chw.DTYPE_I64, 1, 4, 0, None, 0, None)
    assert rc == chw.CHW_ERR_MODE
    assert chw.lib.chw_b200_last_error().decode() == "chw_forward: orthonormal mode requires a floating-point signal"


def test_parallel_execute_validation():
    # parallel.cpp:84-91 order: length, mode, workers
    assert chw.lib.chw_b200_parallel_execute(None, chw.DTYPE_I64, 3, 2, 1, None) == chw.CHW_ERR_LENGTH
    assert chw.lib.chw_b200_parallel_execute(None, chw.DTYPE_I64, 4, 2, 0, None) == chw.CHW_ERR_MODE
    assert chw.lib.chw_b200_parallel_execute(None, chw.DTYPE_I64, 4, 0, 1, None) == chw.CHW_ERR_ARGUMENT
    assert chw.lib.chw_b200_last_error().decode() == "parallel_execute: workers must be >= 1, got 0"


def test_zero_batch_is_a_noop():
    assert chw.lib.chw_b200_forward(None, None, chw.DTYPE_F32, 0, 4096, 0, None, 0, None) == chw.CHW_OK


def test_python_api_raises_reference_exceptions():
    with pytest.raises(ValueError, match="length 3 is not a power of two"):
        chw.chw_forward(np.zeros(3, np.int64), chw.ScalingMode.Unnormalized)
    with pytest.raises(ValueError, match="orthonormal mode requires a floating-point signal"):
        chw.chw_forward(np.zeros(4, np.int64), chw.ScalingMode.Orthonormal)
    with pytest.raises(ValueError, match="stage 0 out of range for m=4"):
        chw.stage_blocks(4, 0)


@pytest.mark.parametrize("m", range(0, 21))
def test_op_tally_closed_form(m):
    # transforms.hpp:75-78 (chw: m*2^m), :49-80 (haar: 2(n-1)), :209 (normalize: n)
    n = 1 << m
    a, mu = ctypes.c_uint64(), ctypes.c_uint64()
    for mode, mults in ((0, m * n), (1, 0)):
        assert chw.lib.chw_b200_op_tally(0, n, mode, ctypes.byref(a), ctypes.byref(mu)) == 0
        assert (a.value, mu.value) == (m * n, mults)
        assert chw.lib.chw_b200_op_tally(1, n, mode, ctypes.byref(a), ctypes.byref(mu)) == 0
        assert a.value == 2 * (n - 1) and mu.value == (2 * (n - 1) if mode == 0 else 0)
    assert chw.lib.chw_b200_op_tally(2, n, 0, ctypes.byref(a), ctypes.byref(mu)) == 0
    assert (a.value, mu.value) == (0, n)


def test_plan_selection():
    # defaults (no CHW_B200_* schedule overrides in the environment)
    assert chw.plan_name(chw.DTYPE_F32, 4096) == "k1t-tma"
    assert chw.plan_name(chw.DTYPE_BF16, 128) == "k7tc-tcgen05"
    assert chw.plan_name(chw.DTYPE_F64, 1024).startswith("k1")
    assert chw.plan_name(chw.DTYPE_F32, 1 << 24) == "k9-row-sweep"
    assert chw.plan_name(chw.DTYPE_F32, 1 << 16) == "k6-rowpipe"
    assert chw.plan_name(chw.DTYPE_F32, 1 << 20).startswith("k4-multipass")


def test_workspace_bytes():
    assert chw.workspace_bytes(chw.DTYPE_F32, 65536, 4096) == 0
    assert chw.workspace_bytes(chw.DTYPE_F32, 256, 1 << 24) >= 256 * (1 << 24) * 4 or \
        chw.workspace_bytes(chw.DTYPE_F32, 256, 1 << 24) > 0


def test_python_mirrors_reference_helpers():
    assert [chw.bit_reverse(i, 2) for i in range(4)] == [0, 2, 1, 3]
    assert chw.natural_to_dyadic(2) == [0, 2, 1, 3]
    assert chw.stage_blocks(4, 2) == [chw.BlockSlice(4, 4), chw.BlockSlice(12, 4)]
    t = chw.OpTally(5, 7)
    t.reset()
    assert t == chw.OpTally()
    y = chw.normalized(np.array([1, 1, 1, 1], np.int64), 2)
    assert y.tolist() == [0.5, 0.5, 0.5, 0.5]
    with pytest.raises(ValueError, match="normalize: signal length 4 does not match level 3"):
        chw.normalize_inplace(np.zeros(4), 3)
