"""Repeatability stress of the kernels added in round 2 session 4: K10
(cluster/DSMEM, CHW_B200_M16=c in the environment), K9n (natural order at
m = 24) and the Haar-Walsh prefix kernel — many runs on fresh random inputs,
each compared bitwise with the first run of the same input and (sampled) with
the oracle."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

import oracle
import paper_1609_06641_b200 as chw

dev = torch.device("cuda:0")
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
bad = 0
print("m16 plan", chw.plan_name(1, 1 << 16))
g = torch.Generator(device=dev)
for it in range(iters):
    g.manual_seed(1000 + it)
    rows = [1, 3, 4, 33, 67, 149, 300, 445][it % 8]
    x = torch.randn(rows, 1 << 16, device=dev, generator=g)
    a = torch.empty_like(x)
    b = torch.empty_like(x)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=a)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=b)
    torch.cuda.synchronize()
    if not torch.equal(a, b):
        bad += 1
        print("m16 mismatch between runs", it, rows)
    if it % 5 == 0:
        ref = oracle.chw_batch(x[:2].cpu().numpy().astype(np.float64), oracle.ORTHONORMAL)
        err = np.linalg.norm(a[:2].cpu().numpy() - ref) / np.linalg.norm(ref)
        if err > 1e-5:
            bad += 1
            print("m16 oracle mismatch", it, err)
n = 1 << 24
for it in range(max(2, iters // 4)):
    g.manual_seed(2000 + it)
    rows = [1, 2, 3, 5][it % 4]
    x = torch.randn(rows, n, device=dev, generator=g)
    a = torch.empty_like(x)
    b = torch.empty_like(x)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=a, order=chw.ORDER_NATURAL)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=b, order=chw.ORDER_NATURAL)
    d = torch.empty_like(x)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=d)
    torch.cuda.synchronize()
    if not torch.equal(a, b):
        bad += 1
        print("m24 natural mismatch between runs", it, rows)
    # Parseval against the dyadic result (a permutation of the same values up to rounding)
    if abs(float(a.double().pow(2).sum() - d.double().pow(2).sum())) > 1e-6 * float(d.double().pow(2).sum()):
        bad += 1
        print("m24 natural energy mismatch", it)
print("stress", "OK" if bad == 0 else f"FAIL ({bad})")
sys.exit(1 if bad else 0)
