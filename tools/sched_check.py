"""Parity check of one schedule variant (selected by the CHW_B200_* env vars of
this process) against the oracle: f32 Orthonormal rel-L2 <= 1e-5 per row,
in-place == out-of-place, exact dyadic order through the Unnormalized integer
probe.  Used by tests/test_schedules_gpu.py (one subprocess per variant, since
the library reads the variant once per process).

    CHW_B200_M16=r1 python tools/sched_check.py --m 16 --rows 1 2 3 149 300
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1609_06641_b200 as chw  # noqa: E402


def check_bf16(m, rows, dev):
    """bf16 in/out: rel-L2 <= 1e-2 per sampled row, in-place == out-of-place,
    exact order through small-integer inputs (exact in bf16 for m <= 7)."""
    rng = np.random.default_rng(4343 + m + rows)
    x = rng.standard_normal(size=(rows, 1 << m)).astype(np.float32)
    t = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    xb = t.float().cpu().numpy()
    out = torch.empty_like(t)
    chw.chw_forward_batched_(t, chw.ScalingMode.Orthonormal, out=out)
    inplace = t.clone()
    chw.chw_forward_batched_(inplace, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()
    assert torch.equal(out, inplace), "in-place != out-of-place"
    y = out.float().cpu().numpy()
    pick = sorted({0, rows - 1, rows // 2})
    ref = oracle.chw_batch(xb[pick].astype(np.float64), oracle.ORTHONORMAL)
    for k, r in enumerate(pick):
        err = np.linalg.norm(y[r] - ref[k]) / np.linalg.norm(ref[k])
        assert err <= 1e-2, f"row {r}: rel L2 {err}"
    xi = rng.integers(-1, 2, size=(rows, 1 << m), dtype=np.int64)
    ti = torch.from_numpy(xi.astype(np.float32)).to(dev).to(torch.bfloat16)
    chw.chw_forward_batched_(ti, chw.ScalingMode.Unnormalized)
    torch.cuda.synchronize()
    got = ti.float().cpu().numpy().astype(np.int64)
    ref_i = oracle.chw_batch(xi[pick], oracle.UNNORMALIZED)
    for k, r in enumerate(pick):
        assert np.array_equal(got[r], ref_i[k]), f"order probe row {r}"
    e_in = (xb.astype(np.float64) ** 2).sum(1)
    e_out = (y.astype(np.float64) ** 2).sum(1)
    assert np.allclose(e_in, e_out, rtol=3e-2), "Parseval failed on some row"


def check(m, rows, dev):
    rng = np.random.default_rng(4242 + m + rows)
    x = rng.standard_normal(size=(rows, 1 << m)).astype(np.float32)
    t = torch.from_numpy(x).to(dev)
    out = torch.empty_like(t)
    chw.chw_forward_batched_(t, chw.ScalingMode.Orthonormal, out=out)
    inplace = t.clone()
    chw.chw_forward_batched_(inplace, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()
    assert torch.equal(out, inplace), "in-place != out-of-place"
    y = out.cpu().numpy()
    # oracle on a sample of rows (first, last, a middle one) keeps it fast
    pick = sorted({0, rows - 1, rows // 2})
    ref = oracle.chw_batch(x[pick].astype(np.float64), oracle.ORTHONORMAL)
    for k, r in enumerate(pick):
        err = np.linalg.norm(y[r] - ref[k]) / np.linalg.norm(ref[k])
        assert err <= 1e-5, f"row {r}: rel L2 {err}"
    bound = 1 << max(0, 24 - m - 1)
    xi = rng.integers(-bound, bound + 1, size=(rows, 1 << m), dtype=np.int64)
    ti = torch.from_numpy(xi.astype(np.float32)).to(dev)
    chw.chw_forward_batched_(ti, chw.ScalingMode.Unnormalized)
    torch.cuda.synchronize()
    got = ti.cpu().numpy().astype(np.int64)
    ref_i = oracle.chw_batch(xi[pick], oracle.UNNORMALIZED)
    for k, r in enumerate(pick):
        assert np.array_equal(got[r], ref_i[k]), f"order probe row {r}"
    # every row, not just the sampled ones: rows are independent and identical
    # in distribution, so compare row sums of squares (Parseval) as a cheap net
    e_in = (x.astype(np.float64) ** 2).sum(1)
    e_out = (y.astype(np.float64) ** 2).sum(1)
    assert np.allclose(e_in, e_out, rtol=1e-5), "Parseval failed on some row"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--rows", type=int, nargs="+", default=[1, 2, 3, 149, 300])
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    for rows in args.rows:
        (check_bf16 if args.dtype == "bf16" else check)(args.m, rows, dev)
    plan = chw.plan_name(2 if args.dtype == "bf16" else 1, 1 << args.m)
    print(f"sched ok: m={args.m} rows={args.rows} plan={plan}")


if __name__ == "__main__":
    main()
