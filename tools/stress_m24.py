"""Stress check of the m = 24 path at the full cfg5 batch: repeated device
runs must agree bit for bit with each other and with the host-buffer path;
prints the differing rows (debug tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_06641_b200 as chw  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(11)
x = torch.randn(rows, 1 << 24, generator=g, device=dev)
ref = torch.empty_like(x)
chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=ref)
out = torch.empty_like(x)
for k in range(reps):
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=out)
    torch.cuda.synchronize()
    bad = (out != ref).any(dim=1).nonzero().flatten().tolist()
    print("device rep", k, "OK" if not bad else f"rows differ {bad[:20]} ({len(bad)})", flush=True)
del out
# independent check of a few rows (incl. any that differed) against the C port
import numpy as np  # noqa: E402

import oracle  # noqa: E402 (debug tool: checker only)

for r in sorted({0, rows // 2, rows - 1, min(196, rows - 1)}):
    want = oracle.chw_batch(x[r:r + 1].double().cpu().numpy(), oracle.ORTHONORMAL)
    got = ref[r:r + 1].double().cpu().numpy()
    print("oracle row", r, "rel l2", float(np.linalg.norm(got - want) / np.linalg.norm(want)), flush=True)
hx = x.cpu().pin_memory()
hy = torch.empty_like(hx).pin_memory()
for k in range(2):
    chw.chw_forward_host_(hx, chw.ScalingMode.Orthonormal, out=hy)
    d = hy.to(dev)
    bad = (d != ref).any(dim=1).nonzero().flatten().tolist()
    print("host rep", k, "OK" if not bad else f"rows differ {bad[:20]} ({len(bad)})", flush=True)
    if bad:
        r = bad[0]
        diff = (d[r] != ref[r]).nonzero().flatten()
        print("  row", r, "n diff", diff.numel(), "first idx", diff[:8].tolist(),
              "max abs", float((d[r] - ref[r]).abs().max()))
    del d
