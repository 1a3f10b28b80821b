"""Quick parity + timing check of the f32 m = 16 schedule selected by
CHW_B200_M16 (c = K10 cluster/DSMEM, default K6): rows vs the C oracle,
repeatability, and a short timing loop."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
import torch

import oracle
import paper_1609_06641_b200 as chw

dev = torch.device("cuda:0")
print("plan", chw.plan_name(1, 1 << 16))
rng = np.random.default_rng(16)
ok = True
for rows in (1, 2, 3, 4, 5, 37, 148, 300, 1000):
    x = rng.uniform(-1, 1, size=(rows, 1 << 16)).astype(np.float32)
    t = torch.from_numpy(x).to(dev)
    o = torch.empty_like(t)
    chw.chw_forward_batched_(t, chw.ScalingMode.Orthonormal, out=o)
    torch.cuda.synchronize()
    y = o.cpu().numpy()
    nchk = min(rows, 6)
    idx = sorted(set(list(range(min(3, rows))) + list(range(max(0, rows - 3), rows))))
    ref = oracle.chw_batch(x[idx].astype(np.float64), oracle.ORTHONORMAL)
    err = np.linalg.norm(y[idx] - ref) / np.linalg.norm(ref)
    o2 = torch.empty_like(t)
    chw.chw_forward_batched_(t, chw.ScalingMode.Orthonormal, out=o2)
    same = bool(torch.equal(o, o2))
    # in place
    t2 = t.clone()
    chw.chw_forward_batched_(t2, chw.ScalingMode.Orthonormal)
    inpl = bool(torch.equal(o, t2))
    print(f"rows {rows:5d} rel L2 {err:.2e} repeat {same} inplace {inpl}")
    ok &= err < 1e-5 and same and inpl
# exact order probe (Unnormalized, small integers)
xi = rng.integers(-3, 4, size=(5, 1 << 16)).astype(np.float32)
ti = torch.from_numpy(xi).to(dev)
chw.chw_forward_batched_(ti, chw.ScalingMode.Unnormalized)
ri = oracle.chw_batch(xi.astype(np.float64), oracle.UNNORMALIZED)
exact = bool(np.array_equal(ti.cpu().numpy().astype(np.float64), ri))
print("order probe exact", exact)
ok &= exact
x = torch.randn(4096, 1 << 16, device=dev)
o = torch.empty_like(x)
for _ in range(5):
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=o)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"cfg4: {ms:.4f} ms/step  {2**31 / (ms * 1e-3) / 1e9:.1f} GB/s  frac {2**31 / (ms * 1e-3) / 1e9 / 6544.7:.3f}")
print("OK" if ok else "FAIL")
sys.exit(0 if ok else 1)
