"""Quick check of the fused NATURAL order at f32 m = 24 (K9n): against the
dyadic result permuted by bit reversal (exact with integer inputs), repeat
runs, in place, launch count, timing."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch

import paper_1609_06641_b200 as chw

dev = torch.device("cuda:0")
m = 24
n = 1 << m
idx = torch.arange(n, device=dev, dtype=torch.int64)
rev = torch.zeros_like(idx)
for b in range(m):
    rev |= ((idx >> b) & 1) << (m - 1 - b)
ok = True
for rows in (1, 2, 3, 5):
    g = torch.Generator(device=dev)
    g.manual_seed(rows)
    xi = torch.randint(-3, 4, (rows, n), device=dev, generator=g).float()
    d = torch.empty_like(xi)
    chw.chw_forward_batched_(xi, chw.ScalingMode.Unnormalized, out=d)
    before = chw.launch_count()
    nat = torch.empty_like(xi)
    chw.chw_forward_batched_(xi, chw.ScalingMode.Unnormalized, out=nat, order=chw.ORDER_NATURAL)
    launches = chw.launch_count() - before
    torch.cuda.synchronize()
    exact = bool(torch.equal(nat, d[:, rev]))
    x = torch.randn(rows, n, device=dev, generator=g)
    d2 = torch.empty_like(x)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=d2)
    n2 = torch.empty_like(x)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=n2, order=chw.ORDER_NATURAL)
    n3 = x.clone()
    chw.chw_forward_batched_(n3, chw.ScalingMode.Orthonormal, order=chw.ORDER_NATURAL)
    torch.cuda.synchronize()
    err = float((n2 - d2[:, rev]).norm() / d2.norm())
    inpl = bool(torch.equal(n2, n3))
    print(f"rows {rows}: exact {exact} launches {launches} rel {err:.2e} inplace {inpl}")
    ok &= exact and err < 1e-6 and inpl
x = torch.randn(32, n, device=dev)
o = torch.empty_like(x)
for order, name in ((chw.ORDER_DYADIC, "dyadic"), (chw.ORDER_NATURAL, "natural"), (chw.ORDER_SEQUENCY, "sequency")):
    for _ in range(2):
        chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=o, order=order)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=o, order=order)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {ms:.3f} ms / 32 rows  frac {32 * n * 8 / (ms * 1e-3) / 1e9 / 6544.7:.3f}")
print("OK" if ok else "FAIL")
sys.exit(0 if ok else 1)
