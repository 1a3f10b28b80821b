"""Debug helper: m = 24 device out-of-place vs in-place vs host path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_06641_b200 as chw

dev = torch.device("cuda:0")
for rows in (1, 2, 4, 9):
    g = torch.Generator(device=dev); g.manual_seed(rows)
    x = torch.randn(rows, 1 << 24, generator=g, device=dev)
    ref = torch.empty_like(x)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=ref)
    ip = x.clone()
    chw.chw_forward_batched_(ip, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()
    hx = x.cpu().pin_memory(); hy = torch.empty_like(hx).pin_memory()
    chw.chw_forward_host_(hx, chw.ScalingMode.Orthonormal, out=hy)
    hyd = hy.to(dev)
    for name, t in (("inplace", ip), ("host", hyd)):
        bad = (t != ref).any(dim=1).nonzero().flatten().tolist()
        print(rows, name, "equal" if not bad else f"rows differ {bad}", float((t - ref).abs().max()))
    # host in place, pageable
    h2 = x.cpu()
    chw.chw_forward_host_(h2, chw.ScalingMode.Orthonormal)
    print(rows, "host-pageable", bool(torch.equal(h2.to(dev), ref)))
