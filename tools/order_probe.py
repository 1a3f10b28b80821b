"""Time the f32 m = 12 (cfg2-shaped) transform in dyadic and natural order
with CUDA events (2 GiB in + out per step, 50 steps): isolates the cost of the
dyadic store pattern.  Schedules come from the CHW_B200_* env of the process."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_06641_b200 as chw  # noqa: E402

x = torch.randn(65536, 4096, device="cuda")
o = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tag = os.environ.get("TAG", "")
for name, order in (("dyadic", chw.ORDER_DYADIC), ("natural", chw.ORDER_NATURAL)):
    def f():
        chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=o, order=order)
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"{tag} {name}: {ms:.4f} ms/step, {65536 * 4096 / ms / 1e6:.1f} Gelem/s, "
          f"{2 * 65536 * 4096 * 4 / ms / 1e6:.0f} GB/s")
