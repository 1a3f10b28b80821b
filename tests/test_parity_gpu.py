"""GPU parity: the sm_100a kernels (through the C ABI) vs the oracle.

Bars (BASELINE.json north_star): f64 BIT-EXACT with the reference (stricter
than the 1e-12 relative-L2 bar), int64 exact, fp32 relative
L2 <= 1e-5, bf16 relative L2 <= 1e-2, and the dyadic output order checked
bit-exactly through the Unnormalized integer probe (a wrong permutation cannot
pass).  Inputs are seeded; sizes are ones the oracle finishes in seconds.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

O, U = oracle.ORTHONORMAL, oracle.UNNORMALIZED
F32_TOL = 1e-5
BF16_TOL = 1e-2


def _chw():
    import paper_1609_06641_b200 as chw

    return chw


def _gpu(x, cuda):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(cuda)


def _run(x, mode, cuda, dtype=None):
    import torch

    chw = _chw()
    t = _gpu(x, cuda)
    if dtype is not None:
        t = t.to(dtype)
    chw.chw_forward_batched_(t, chw.ScalingMode(mode))
    torch.cuda.synchronize()
    return t


def _rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _rows_for(m, elems=1 << 16):
    return max(1, min(37, elems >> m))


# ---------------------------------------------------------------------------
# f64: bit-exact against the reference algorithm (Orthonormal and Unnormalized)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m", list(range(0, 21)))
@pytest.mark.parametrize("mode", [O, U])
def test_f64_bitexact(cuda, m, mode):
    rng = np.random.default_rng(100 + m)
    rows = _rows_for(m) if m < 17 else 1
    x = rng.uniform(-1, 1, size=(rows, 1 << m))
    y = _run(x, mode, cuda).cpu().numpy()
    ref = oracle.chw_batch(x, mode)
    assert np.array_equal(y.view(np.uint64), ref.view(np.uint64)), (
        f"m={m} mode={mode}: max abs diff {np.max(np.abs(y - ref))}")


def test_f64_golden_cfg1_rows(cuda, golden):
    x = golden["cfg1_rows16_in"].reshape(16, 1024)
    y = _run(x, O, cuda).cpu().numpy()
    assert np.array_equal(y.view(np.uint64), golden["cfg1_rows16_out"].reshape(16, 1024).view(np.uint64))


@pytest.mark.parametrize("m", range(0, 15))
def test_f64_golden_sweep(cuda, golden, m):
    x = golden[f"sweep_f64_m{m}_in"][None, :]
    for mode, key in ((O, "ortho"), (U, "unnorm")):
        y = _run(x, mode, cuda).cpu().numpy()[0]
        assert np.array_equal(y.view(np.uint64), golden[f"sweep_f64_m{m}_{key}"].view(np.uint64))


# ---------------------------------------------------------------------------
# int64 (f1): exact
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m", list(range(0, 21)))
def test_i64_exact(cuda, m):
    rng = np.random.default_rng(200 + m)
    rows = _rows_for(m) if m < 17 else 1
    x = rng.integers(-1000, 1001, size=(rows, 1 << m), dtype=np.int64)
    y = _run(x, U, cuda).cpu().numpy()
    assert np.array_equal(y, oracle.chw_batch(x, U))


@pytest.mark.parametrize("m", range(0, 9))
def test_i64_golden_dense(cuda, golden, m):
    # transforms_test.cpp:123-132 through the GPU
    x = golden[f"dense_int_m{m}_in"].reshape(20, 1 << m)
    y = _run(x, U, cuda).cpu().numpy()
    assert np.array_equal(y, golden[f"dense_int_m{m}_dense"].reshape(20, 1 << m))


def test_i64_orthonormal_rejected(cuda):
    chw = _chw()
    import torch

    t = torch.zeros(4, dtype=torch.int64, device=cuda)
    with pytest.raises(ValueError, match="orthonormal mode requires a floating-point signal"):
        chw.chw_forward_batched_(t, chw.ScalingMode.Orthonormal)


# ---------------------------------------------------------------------------
# fp32: tolerance + exact order probe
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m", list(range(0, 25)))
def test_f32_tolerance(cuda, m):
    import torch

    rng = np.random.default_rng(300 + m)
    rows = _rows_for(m, 1 << 18) if m < 20 else 1
    x = rng.standard_normal(size=(rows, 1 << m)).astype(np.float32)
    y = _run(x, O, cuda, torch.float32).cpu().numpy()
    ref = oracle.chw_batch(x.astype(np.float64), O)
    per_row = [_rel_l2(y[r], ref[r]) for r in range(rows)]
    assert max(per_row) <= F32_TOL, f"m={m}: worst row rel L2 {max(per_row):.3e}"


@pytest.mark.parametrize("m", list(range(0, 25)))
def test_f32_order_probe_exact(cuda, m):
    """Unnormalized on integers with |x| <= 2^(24-m): every partial sum is exact
    in fp32, so the output must equal the int64 oracle bit for bit."""
    import torch

    rng = np.random.default_rng(400 + m)
    bound = max(1, 1 << max(0, 24 - m - 1))
    rows = _rows_for(m, 1 << 18) if m < 20 else 1
    xi = rng.integers(-bound, bound + 1, size=(rows, 1 << m), dtype=np.int64)
    y = _run(xi.astype(np.float32), U, cuda, torch.float32).cpu().numpy()
    ref = oracle.chw_batch(xi, U)
    assert np.array_equal(y.astype(np.int64), ref)
    assert np.array_equal(y, ref.astype(np.float32))


def test_f32_basis_vectors(cuda):
    """e_j -> column j of H_dy: y[i] = 2^(-m/2) (-1)^popcount(rev(i) & j)."""
    import torch

    m = 12
    n = 1 << m
    js = [0, 1, 2, 3, 5, 100, 2047, 4095]
    x = np.zeros((len(js), n), np.float32)
    for r, j in enumerate(js):
        x[r, j] = 1
    y = _run(x, O, cuda, torch.float32).cpu().numpy()
    rev = np.array([oracle.bit_reverse(i, m) for i in range(n)])
    for r, j in enumerate(js):
        sign = 1 - 2 * (np.array([bin(int(v) & j).count("1") & 1 for v in rev]))
        assert np.array_equal(y[r], (sign * 2.0 ** (-m / 2)).astype(np.float32))


# ---------------------------------------------------------------------------
# bf16
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m", list(range(0, 21)))
def test_bf16_tolerance(cuda, m):
    import torch

    rng = np.random.default_rng(500 + m)
    rows = _rows_for(m, 1 << 18) if m < 18 else 1
    x = torch.from_numpy(rng.standard_normal(size=(rows, 1 << m)).astype(np.float32)).to(torch.bfloat16)
    xd = x.to(torch.float64).numpy()  # exact upcast of the same bf16 bytes
    y = _run(x.numpy() if False else x.to(torch.float32).numpy(), O, cuda, torch.bfloat16)
    y = y.to(torch.float64).cpu().numpy()
    ref = oracle.chw_batch(xd, O)
    per_row = [_rel_l2(y[r], ref[r]) for r in range(rows)]
    assert max(per_row) <= BF16_TOL, f"m={m}: worst row rel L2 {max(per_row):.3e}"


@pytest.mark.parametrize("m", list(range(0, 8)))
def test_bf16_order_probe_exact(cuda, m):
    """x in {-1,0,1}, m <= 7: |y| <= 128, exact in bf16."""
    import torch

    rng = np.random.default_rng(600 + m)
    rows = 4099
    xi = rng.integers(-1, 2, size=(rows, 1 << m), dtype=np.int64)
    y = _run(xi.astype(np.float32), U, cuda, torch.bfloat16).to(torch.float64).cpu().numpy()
    assert np.array_equal(y.astype(np.int64), oracle.chw_batch(xi, U))


# ---------------------------------------------------------------------------
# API behaviour: in place vs out of place, host path, parallel_execute, errors
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m", [3, 10, 12, 16])
def test_out_of_place_equals_in_place(cuda, m):
    import torch

    chw = _chw()
    rng = np.random.default_rng(700 + m)
    x = _gpu(rng.uniform(-1, 1, size=(5, 1 << m)), cuda)
    out = torch.empty_like(x)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=out)
    inplace = x.clone()
    chw.chw_forward_batched_(inplace, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()
    assert torch.equal(out, inplace)


@pytest.mark.parametrize("dtype", ["f64", "f32", "i64"])
@pytest.mark.parametrize("m", [0, 7, 12, 16])
def test_host_path(cuda, dtype, m):
    chw = _chw()
    rng = np.random.default_rng(800 + m)
    rows = 9
    if dtype == "i64":
        x = rng.integers(-1000, 1001, size=(rows, 1 << m), dtype=np.int64)
        mode = U
    else:
        x = rng.uniform(-1, 1, size=(rows, 1 << m)).astype(np.float64 if dtype == "f64" else np.float32)
        mode = O
    y = x.copy()
    chw.chw_forward_host_(y, chw.ScalingMode(mode))
    dev = _run(x, mode, cuda).cpu().numpy()
    assert np.array_equal(y, dev)


def test_kats_through_reference_api(cuda):
    chw = _chw()
    import torch

    t = chw.OpTally()
    y = chw.chw_forward(np.array([1, 0, 0, 0], np.int64), chw.ScalingMode.Unnormalized, t)
    assert y.tolist() == [1, 1, 1, 1] and t.additions == 8
    assert chw.chw_forward(np.array([0, 1, 0, 0], np.int64), chw.ScalingMode.Unnormalized).tolist() == [1, 1, -1, -1]
    t.reset()
    assert chw.chw_forward(np.array([9], np.int64), chw.ScalingMode.Unnormalized, t).tolist() == [9]
    assert t == chw.OpTally()
    with pytest.raises(ValueError, match="length 3 is not a power of two"):
        chw.chw_forward_inplace(torch.zeros(3, dtype=torch.int64, device=cuda), chw.ScalingMode.Unnormalized)
    with pytest.raises(ValueError, match="length 0 is not a power of two"):
        chw.chw_forward_inplace(torch.zeros(0, dtype=torch.int64, device=cuda), chw.ScalingMode.Unnormalized)


def test_parallel_execute_contract(cuda):
    # parallel_test.cpp:21-91 restated
    chw = _chw()
    import torch

    rng = np.random.default_rng(9)
    for m in (2, 5, 9, 13):
        x = rng.integers(-1000, 1001, size=1 << m, dtype=np.int64)
        serial = oracle.chw_forward(x, U)
        for workers in (1, 2, 4, 8):
            t = chw.OpTally()
            y = chw.parallel_execute(torch.from_numpy(x).to(cuda), workers, chw.ScalingMode.Unnormalized, t)
            assert np.array_equal(y.cpu().numpy(), serial)
            assert t.additions == m << m and t.multiplications == 0
    for m in (3, 8, 11):
        x = rng.uniform(-1, 1, size=1 << m)
        serial = oracle.chw_forward(x, O)
        y = chw.parallel_execute(torch.from_numpy(x).to(cuda), 4, chw.ScalingMode.Orthonormal).cpu().numpy()
        assert np.array_equal(y.view(np.uint64), serial.view(np.uint64))
    assert chw.parallel_execute(torch.tensor([1, 2], device=cuda), 8, chw.ScalingMode.Unnormalized).tolist() == [3, -1]
    with pytest.raises(ValueError, match="workers must be >= 1, got 0"):
        chw.parallel_execute(torch.tensor([1, 2, 3, 4], device=cuda), 0, chw.ScalingMode.Unnormalized)
    with pytest.raises(ValueError, match="not a power of two"):
        chw.parallel_execute(torch.tensor([1, 2, 3], device=cuda), 2, chw.ScalingMode.Unnormalized)
    with pytest.raises(ValueError, match="orthonormal mode requires"):
        chw.parallel_execute(torch.tensor([1, 2, 3, 4], device=cuda), 2, chw.ScalingMode.Orthonormal)


def test_determinism(cuda):
    # parallel_test.cpp:60-65 analogue: repeated runs are bitwise identical.
    import torch

    rng = np.random.default_rng(8)
    x = rng.standard_normal(size=(64, 1 << 16)).astype(np.float32)
    first = _run(x, O, cuda, torch.float32)
    for _ in range(5):
        assert torch.equal(_run(x, O, cuda, torch.float32), first)


def test_launches_counted(cuda):
    chw = _chw()
    import torch

    before = chw.launch_count()
    _run(np.zeros((4, 1 << 12), np.float32), O, cuda, torch.float32)
    assert chw.launch_count() > before


# ---------------------------------------------------------------------------
# K5 fused two-phase kernel (m = 16, 24): several row chunks, a ragged last
# chunk, in place and out of place, exact order probe, host path.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m,rows", [(16, 1), (16, 33), (16, 70), (16, 97), (24, 1), (24, 3)])
def test_fused_chunks(cuda, m, rows):
    import torch

    chw = _chw()
    rng = np.random.default_rng(900 + m + rows)
    x = rng.standard_normal(size=(rows, 1 << m)).astype(np.float32)
    t = torch.from_numpy(x).to(cuda)
    out = torch.empty_like(t)
    chw.chw_forward_batched_(t, chw.ScalingMode.Orthonormal, out=out)
    inplace = t.clone()
    chw.chw_forward_batched_(inplace, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()
    assert torch.equal(out, inplace)
    y = out.cpu().numpy()
    ref = oracle.chw_batch(x.astype(np.float64), O)
    for r in range(rows):
        assert _rel_l2(y[r], ref[r]) <= F32_TOL
    host = x.copy()
    chw.chw_forward_host_(host, chw.ScalingMode.Orthonormal)
    assert np.array_equal(host, y)
    # order probe on integers (exact)
    bound = 1 << max(0, 24 - m - 1)
    xi = rng.integers(-bound, bound + 1, size=(rows, 1 << m), dtype=np.int64)
    ti = torch.from_numpy(xi.astype(np.float32)).to(cuda)
    chw.chw_forward_batched_(ti, chw.ScalingMode.Unnormalized)
    torch.cuda.synchronize()
    assert np.array_equal(ti.cpu().numpy().astype(np.int64), oracle.chw_batch(xi, U))


def test_user_workspace_too_small_is_rejected(cuda):
    import torch

    chw = _chw()
    x = torch.zeros(4, 1 << 16, device=cuda)
    need = chw.workspace_bytes(chw.DTYPE_F32, 4, 1 << 16)
    assert need > 0
    ws = torch.empty(need - 1, dtype=torch.uint8, device=cuda)
    with pytest.raises(ValueError, match="workspace"):
        chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, workspace=ws)


# ---------------------------------------------------------------------------
# a2: batched Haar transform Psi_m (transforms.hpp:49-80)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m", list(range(0, 19)))
def test_haar_f64_bitexact(cuda, m):
    import torch

    chw = _chw()
    rng = np.random.default_rng(1100 + m)
    rows = max(1, min(9, (1 << 16) >> m))
    x = rng.uniform(-1, 1, size=(rows, 1 << m))
    for mode in (O, U):
        t = torch.from_numpy(x).to(cuda)
        out = torch.empty_like(t)
        chw.haar_forward_batched_(t, chw.ScalingMode(mode), out=out)   # out of place
        chw.haar_forward_batched_(t, chw.ScalingMode(mode))            # in place
        torch.cuda.synchronize()
        ref = np.stack([oracle.haar_forward(x[r], mode) for r in range(rows)])
        assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64))
        assert np.array_equal(t.cpu().numpy().view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("m", [0, 1, 5, 12, 14, 17])
def test_haar_i64_and_f32(cuda, m):
    import torch

    chw = _chw()
    rng = np.random.default_rng(1200 + m)
    xi = rng.integers(-1000, 1001, size=(3, 1 << m), dtype=np.int64)
    ti = torch.from_numpy(xi).to(cuda)
    chw.haar_forward_batched_(ti, chw.ScalingMode.Unnormalized)
    torch.cuda.synchronize()
    assert np.array_equal(ti.cpu().numpy(), np.stack([oracle.haar_forward(r, U) for r in xi]))
    xf = rng.standard_normal(size=(3, 1 << m)).astype(np.float32)
    tf = torch.from_numpy(xf).to(cuda)
    chw.haar_forward_batched_(tf, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()
    ref = np.stack([oracle.haar_forward(r.astype(np.float64), O) for r in xf])
    for r in range(3):
        assert _rel_l2(tf.cpu().numpy()[r], ref[r]) <= F32_TOL


def test_haar_kats_and_validation(cuda):
    # transforms_test.cpp:27-45, tally_test.cpp:30-36 and :70-77
    chw = _chw()
    t = chw.OpTally()
    assert chw.haar_forward(np.array([7], np.int64), chw.ScalingMode.Unnormalized, t).tolist() == [7]
    assert t.additions == 0
    assert chw.haar_forward(np.array([1, 0, 0, 0], np.int64), chw.ScalingMode.Unnormalized, t).tolist() == [1, 1, 1, 0]
    assert t.additions == 6
    t = chw.OpTally()
    chw.haar_forward(np.random.default_rng(4).uniform(-1, 1, 16), chw.ScalingMode.Orthonormal, t)
    assert (t.additions, t.multiplications) == (30, 30)
    with pytest.raises(ValueError, match="haar_forward: length 3 is not a power of two"):
        chw.haar_forward(np.zeros(3, np.int64), chw.ScalingMode.Unnormalized)
    with pytest.raises(ValueError, match="haar_forward: orthonormal mode requires a floating-point signal"):
        chw.haar_forward(np.zeros(2, np.int64), chw.ScalingMode.Orthonormal)


# ---------------------------------------------------------------------------
# f2: natural and sequency orders (orderings_test.cpp:79-84, :35-65)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m", list(range(0, 21)))
def test_orders_bitexact(cuda, m):
    import torch

    chw = _chw()
    rng = np.random.default_rng(1300 + m)
    rows = max(1, min(5, (1 << 15) >> m))
    x = rng.uniform(-1, 1, size=(rows, 1 << m))
    n = 1 << m
    gray = np.array([i ^ (i >> 1) for i in range(n)])
    for mode in (O, U):
        nat = torch.from_numpy(x).to(cuda)
        seq = nat.clone()
        chw.chw_forward_batched_(nat, chw.ScalingMode(mode), order=chw.ORDER_NATURAL)
        chw.chw_forward_batched_(seq, chw.ScalingMode(mode), order=chw.ORDER_SEQUENCY)
        torch.cuda.synchronize()
        ref_nat = np.stack([oracle.simple("fwht_natural", x[r], mode) for r in range(rows)])
        ref_dy = oracle.chw_batch(x, mode)
        assert np.array_equal(nat.cpu().numpy().view(np.uint64), ref_nat.view(np.uint64))
        assert np.array_equal(seq.cpu().numpy().view(np.uint64), ref_dy[:, gray].view(np.uint64))


@pytest.mark.parametrize("m,rows", [(2, 37), (7, 300), (12, 149), (13, 5), (16, 150), (24, 3)])
def test_sequency_fused_f32(cuda, m, rows):
    """f2: sequency order folded into the store map (inverse Gray code of the
    dyadic position): bit-exact integer probe against the reference permutation
    (orderings.hpp:82-102) on batches that leave partial tiles / CTAs with 0-3
    rows, in place and out of place, and with no extra gather launch."""
    import torch

    chw = _chw()
    rng = np.random.default_rng(1500 + m)
    bound = 1 << max(0, 24 - m)
    xi = rng.integers(-bound, bound + 1, size=(rows, 1 << m), dtype=np.int64)
    dy = oracle.chw_batch(xi, U)
    gray = np.array([i ^ (i >> 1) for i in range(1 << m)])
    ref = dy[:, gray]
    t = torch.from_numpy(xi).to(cuda).to(torch.float32)
    out = torch.empty_like(t)
    n_dy = chw.launch_count()
    chw.chw_forward_batched_(t.clone(), chw.ScalingMode.Unnormalized)
    n_dy = chw.launch_count() - n_dy
    n_seq = chw.launch_count()
    chw.chw_forward_batched_(t, chw.ScalingMode.Unnormalized, out=out, order=chw.ORDER_SEQUENCY)
    n_seq = chw.launch_count() - n_seq
    chw.chw_forward_batched_(t, chw.ScalingMode.Unnormalized, order=chw.ORDER_SEQUENCY)  # in place
    torch.cuda.synchronize()
    assert np.array_equal(out.to(torch.float64).cpu().numpy().astype(np.int64), ref)
    assert np.array_equal(t.to(torch.float64).cpu().numpy().astype(np.int64), ref)
    assert n_seq == n_dy, "sequency must not add a gather pass"
    assert chw.workspace_bytes_ordered(chw.DTYPE_F32, rows, 1 << m, chw.ORDER_SEQUENCY) == \
        chw.workspace_bytes(chw.DTYPE_F32, rows, 1 << m)


@pytest.mark.parametrize("rows", [1, 3, 149, 150])
def test_natural_fused_f32_m16(cuda, rows):
    """f2: natural order folded into the m = 16 row pipeline (K6) — bit-exact
    integer probe against the reference's fwht_natural order, in place and out
    of place, no extra gather launch or workspace."""
    import torch

    chw = _chw()
    m = 16
    rng = np.random.default_rng(1600 + rows)
    xi = rng.integers(-256, 257, size=(rows, 1 << m), dtype=np.int64)
    dy = oracle.chw_batch(xi, U)
    rev = np.array([oracle.bit_reverse(i, m) for i in range(1 << m)])
    ref = dy[:, rev]
    t = torch.from_numpy(xi).to(cuda).to(torch.float32)
    out = torch.empty_like(t)
    n_dy = chw.launch_count()
    chw.chw_forward_batched_(t.clone(), chw.ScalingMode.Unnormalized)
    n_dy = chw.launch_count() - n_dy
    n_nat = chw.launch_count()
    chw.chw_forward_batched_(t, chw.ScalingMode.Unnormalized, out=out, order=chw.ORDER_NATURAL)
    n_nat = chw.launch_count() - n_nat
    chw.chw_forward_batched_(t, chw.ScalingMode.Unnormalized, order=chw.ORDER_NATURAL)
    torch.cuda.synchronize()
    assert np.array_equal(out.to(torch.float64).cpu().numpy().astype(np.int64), ref)
    assert np.array_equal(t.to(torch.float64).cpu().numpy().astype(np.int64), ref)
    assert n_nat == n_dy
    # orthonormal f32 within tolerance of the reference natural FWHT
    x = rng.uniform(-1, 1, size=(rows, 1 << m)).astype(np.float32)
    tx = torch.from_numpy(x).to(cuda)
    chw.chw_forward_batched_(tx, chw.ScalingMode.Orthonormal, order=chw.ORDER_NATURAL)
    got = tx.cpu().numpy().astype(np.float64)
    want = np.stack([oracle.simple("fwht_natural", x[r].astype(np.float64), O) for r in range(rows)])
    assert _rel_l2(got, want) <= F32_TOL


@pytest.mark.parametrize("rows", [1, 3])
def test_natural_fused_f32_m24(cuda, rows):
    """f2: natural order folded into the m = 24 row sweep (K9n: the second
    phase carries j0..j3, in-place tile transposes, swizzling tensor maps) —
    bit-exact integer probe against the dyadic result permuted by bit
    reversal (orderings.hpp:45-78), in place and out of place, one launch, no
    gather workspace; orthonormal f32 within tolerance of the reference's
    natural FWHT."""
    import torch

    chw = _chw()
    m = 24
    rng = np.random.default_rng(2400 + rows)
    xi = rng.integers(-3, 4, size=(rows, 1 << m), dtype=np.int64)
    dy = oracle.chw_batch(xi, U)
    idx = np.arange(1 << m, dtype=np.int64)
    rev = np.zeros_like(idx)
    for b in range(m):
        rev |= ((idx >> b) & 1) << (m - 1 - b)
    ref = dy[:, rev]
    t = torch.from_numpy(xi).to(cuda).to(torch.float32)
    out = torch.empty_like(t)
    n_dy = chw.launch_count()
    chw.chw_forward_batched_(t.clone(), chw.ScalingMode.Unnormalized)
    n_dy = chw.launch_count() - n_dy
    n_nat = chw.launch_count()
    chw.chw_forward_batched_(t, chw.ScalingMode.Unnormalized, out=out, order=chw.ORDER_NATURAL)
    n_nat = chw.launch_count() - n_nat
    chw.chw_forward_batched_(t, chw.ScalingMode.Unnormalized, order=chw.ORDER_NATURAL)
    torch.cuda.synchronize()
    assert np.array_equal(out.to(torch.float64).cpu().numpy().astype(np.int64), ref)
    assert np.array_equal(t.to(torch.float64).cpu().numpy().astype(np.int64), ref)
    assert n_nat == n_dy, "natural order must not add a gather pass"
    assert chw.workspace_bytes_ordered(chw.DTYPE_F32, rows, 1 << m, chw.ORDER_NATURAL) == \
        chw.workspace_bytes(chw.DTYPE_F32, rows, 1 << m)
    x = rng.standard_normal(size=(1, 1 << m)).astype(np.float32)
    tx = torch.from_numpy(x).to(cuda)
    chw.chw_forward_batched_(tx, chw.ScalingMode.Orthonormal, order=chw.ORDER_NATURAL)
    got = tx.cpu().numpy().astype(np.float64)
    want = oracle.simple("fwht_natural", x[0].astype(np.float64), O)[None, :]
    assert _rel_l2(got, want) <= F32_TOL


@pytest.mark.parametrize("dt", ["f32", "bf16", "i64"])
@pytest.mark.parametrize("m", [3, 10, 12, 16])
def test_orders_other_dtypes(cuda, dt, m):
    import torch

    chw = _chw()
    rng = np.random.default_rng(1400 + m)
    xi = rng.integers(-1, 2, size=(4, 1 << m), dtype=np.int64)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "i64": torch.int64}[dt]
    if dt == "bf16" and m > 7:
        pytest.skip("exact bf16 probe only for m <= 7")
    dy = oracle.chw_batch(xi, U)
    rev = np.array([oracle.bit_reverse(i, m) for i in range(1 << m)])
    gray = np.array([i ^ (i >> 1) for i in range(1 << m)])
    for order, ref in ((chw.ORDER_NATURAL, dy[:, rev]), (chw.ORDER_SEQUENCY, dy[:, gray])):
        t = torch.from_numpy(xi).to(cuda).to(tdt)
        chw.chw_forward_batched_(t, chw.ScalingMode.Unnormalized, order=order)
        torch.cuda.synchronize()
        assert np.array_equal(t.to(torch.float64).cpu().numpy().astype(np.int64), ref)


def test_fwht_reference_api(cuda):
    chw = _chw()
    t = chw.OpTally()
    assert chw.fwht_natural(np.array([1, 0], np.int64), chw.ScalingMode.Unnormalized, t).tolist() == [1, 1]
    assert t.additions == 2
    x = np.array([0, 1, 0, 0], np.int64)
    assert chw.fwht_dyadic(x, chw.ScalingMode.Unnormalized).tolist() == [1, 1, -1, -1]
    nat = chw.fwht_natural(x, chw.ScalingMode.Unnormalized)
    assert nat[[0, 2, 1, 3]].tolist() == [1, 1, -1, -1]


# ---------------------------------------------------------------------------
# f3: Haar inverse and Haar-Walsh (transforms_test.cpp:59-75, :172-192)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m", list(range(0, 18)))
def test_haar_inverse_bitexact(cuda, m):
    chw = _chw()
    rng = np.random.default_rng(1500 + m)
    rows = max(1, min(4, (1 << 15) >> m))
    x = rng.uniform(-1, 1, size=(rows, 1 << m))
    for mode in (O, U):
        y = x.copy()
        chw.haar_inverse_inplace(y, chw.ScalingMode(mode))
        ref = np.stack([oracle.simple("haar_inverse", x[r], mode) for r in range(rows)])
        assert np.array_equal(y.view(np.uint64), ref.view(np.uint64))
    xi = rng.integers(-1000, 1001, size=(rows, 1 << m), dtype=np.int64)
    h = np.stack([oracle.haar_forward(r, U) for r in xi])
    back = chw.haar_inverse(h, chw.ScalingMode.Unnormalized)
    assert np.array_equal(back, xi)  # integer round trip is exact


def test_haar_inverse_structure_error(cuda):
    chw = _chw()
    assert chw.haar_inverse(np.array([5], np.int64), chw.ScalingMode.Unnormalized).tolist() == [5]
    assert chw.haar_inverse(chw.haar_forward(np.array([1, 2, 3, 4], np.int64), chw.ScalingMode.Unnormalized),
                            chw.ScalingMode.Unnormalized).tolist() == [1, 2, 3, 4]
    with pytest.raises(chw.StructureError, match="not an integer forward-transform output"):
        chw.haar_inverse(np.array([1, 0], np.int64), chw.ScalingMode.Unnormalized)
    xf = np.random.default_rng(33).uniform(-1, 1, 64)
    rt = chw.haar_inverse(chw.haar_forward(xf, chw.ScalingMode.Orthonormal), chw.ScalingMode.Orthonormal)
    assert np.max(np.abs(rt - xf)) <= 1e-12


@pytest.mark.parametrize("m", [1, 2, 5, 10, 14, 15])
def test_haar_walsh_f32(cuda, m):
    """f32 Haar-Walsh map: the one-kernel shared-memory prefix (blocks below
    2^14) plus the per-block path above it, within the fp32 tolerance of the
    reference (transforms.hpp:187-198) in both scaling modes."""
    chw = _chw()
    rng = np.random.default_rng(1700 + m)
    x = rng.uniform(-1, 1, size=(3, 1 << m)).astype(np.float32)
    for mode, om in ((chw.ScalingMode.Orthonormal, O), (chw.ScalingMode.Unnormalized, U)):
        got = chw.haar_walsh_forward(x, mode).astype(np.float64)
        ref = np.stack([oracle.simple("haar_walsh_forward", r.astype(np.float64), om) for r in x])
        assert _rel_l2(got, ref) <= F32_TOL


@pytest.mark.parametrize("m", list(range(0, 17)))
def test_haar_walsh(cuda, golden, m):
    chw = _chw()
    rng = np.random.default_rng(1600 + m)
    x = rng.integers(-1000, 1001, size=(3, 1 << m), dtype=np.int64)
    got = chw.haar_walsh_forward(x, chw.ScalingMode.Unnormalized)
    ref = np.stack([oracle.simple("haar_walsh_forward", r, U) for r in x])
    assert np.array_equal(got, ref)
    # composition: haar_walsh(haar(x)) == chw(x) (transforms_test.cpp:181-184)
    h = chw.haar_forward(x, chw.ScalingMode.Unnormalized)
    assert np.array_equal(chw.haar_walsh_forward(h, chw.ScalingMode.Unnormalized), oracle.chw_batch(x, U))
    if m == 7:
        assert np.array_equal(chw.haar_walsh_forward(golden["haarwalsh_m7_in"], chw.ScalingMode.Unnormalized),
                              golden["haarwalsh_m7_dense"])
    xf = rng.uniform(-1, 1, size=(2, 1 << m))
    gf = chw.haar_walsh_forward(xf, chw.ScalingMode.Orthonormal)
    rf = np.stack([oracle.simple("haar_walsh_forward", r, O) for r in xf])
    assert np.array_equal(gf.view(np.uint64), rf.view(np.uint64))
