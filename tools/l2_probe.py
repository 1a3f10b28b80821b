"""Probe SM<->L2 bandwidth: device copies whose footprint fits in L2 vs HBM.
Prints GB/s (read + write bytes) for several sizes.  Used to decide whether an
L2-resident intermediate can beat the HBM roofline."""
import torch

def bw(nbytes, reps=50):
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    for _ in range(5):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    return 2 * nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9

for mb in (4, 8, 16, 32, 48, 64, 128, 1024, 4096):
    print(f"{mb:6d} MiB footprint x2: {bw(mb << 20):9.1f} GB/s")
