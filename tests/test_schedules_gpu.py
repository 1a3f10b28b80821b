"""GPU parity of every selectable schedule of the long-row paths, one
subprocess per variant (the library reads CHW_B200_* once per process).

m = 16 (cfg4): K6 row pipeline variants r1..r7 (default r6), the K3 cluster
kernel (c) and the K5 fused dataflow kernel (f); m = 24 (cfg5): the TMA two-pass
schedule (t, default), K4P (p) and the fused one (f).  Each run checks f32 Orthonormal
against the oracle (rel-L2 <= 1e-5), in-place == out-of-place, the exact
dyadic order through the integer probe, and Parseval on every row, for batch
sizes that leave some CTAs with 0, 1, 2 or 3 rows (tools/sched_check.py).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra, m, rows):
    env = dict(os.environ)
    env.update(env_extra)
    cmd = [sys.executable, os.path.join(REPO, "tools", "sched_check.py"), "--m", str(m), "--rows"] + [
        str(r) for r in rows]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert "sched ok" in p.stdout
    return p.stdout


@pytest.mark.parametrize("variant", ["r1", "r2", "r3", "r4", "r5", "r6", "r7", "c", "f"])
def test_m16_schedules(cuda, variant):
    out = _run({"CHW_B200_M16": variant}, 16, [1, 2, 3, 149, 300, 445])
    want = {"r": "k6-rowpipe", "c": "k3-cluster-dsmem", "f": "k5-fused-2phase"}[variant[0]]
    assert want in out


def test_m16_default_is_rowpipe(cuda):
    env = {k: v for k, v in os.environ.items() if k != "CHW_B200_M16"}
    p = subprocess.run([sys.executable, os.path.join(REPO, "tools", "sched_check.py"), "--m", "16", "--rows", "5"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "k6-rowpipe" in p.stdout


@pytest.mark.parametrize("variant", ["default", "t", "p", "f"])
def test_m24_schedules(cuda, variant):
    env = {k: v for k, v in os.environ.items() if k != "CHW_B200_M24"}
    if variant != "default":
        env["CHW_B200_M24"] = variant
    cmd = [sys.executable, os.path.join(REPO, "tools", "sched_check.py"), "--m", "24", "--rows", "1", "3", "17"]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    want = {"default": "k4t-two-pass-tma", "t": "k4t-two-pass-tma", "p": "k4p-two-pass-pipelined",
            "f": "k5-fused-2phase"}[variant]
    assert want in p.stdout


@pytest.mark.parametrize("variant", ["0", "1", "2", "3", "4"])
def test_m12_k1t_variants(cuda, variant):
    """f32 m = 12 (cfg2): K1T variants (TMA-fed, default 1) and K1P (0)."""
    out = _run({"CHW_B200_K1T": variant}, 12, [1, 5, 148, 149, 1000, 4097])
    assert ("k1t-tma" in out) == (variant != "0")


@pytest.mark.parametrize("variant", ["0", "1", "2", "3"])
def test_m7_bf16_k1t_variants(cuda, variant):
    """bf16 m = 7 (cfg3): K1 (0, default) and the TMA-fed K1T variants."""
    env = dict(os.environ)
    env["CHW_B200_K1T_BF16"] = variant
    p = subprocess.run([sys.executable, os.path.join(REPO, "tools", "sched_check.py"), "--m", "7", "--dtype", "bf16",
                        "--rows", "1", "31", "32", "33", "4737"], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert ("k1t-tma" in p.stdout) == (variant != "0")


# ---------------------------------------------------------------------------
# Boundary cases of the TMA-fed default kernels (K1T m=12, K6 m=16, K4T m=24).
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("m,rows", [(12, 300), (16, 150), (24, 2)])
def test_exact_user_workspace_and_side_stream(cuda, m, rows):
    """A caller workspace of exactly chw_b200_workspace_bytes() bytes and a
    non-default stream give the same bits as the library-managed default."""
    import numpy as np
    import torch

    import paper_1609_06641_b200 as chw

    g = torch.Generator(device=cuda)
    g.manual_seed(m * 1000 + rows)
    x = torch.randn(rows, 1 << m, device=cuda, generator=g)
    ref = torch.empty_like(x)
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=ref)
    need = chw.workspace_bytes(chw.DTYPE_F32, rows, 1 << m)
    ws = torch.empty(max(need, 1), dtype=torch.uint8, device=cuda)
    side = torch.cuda.Stream()
    out = torch.empty_like(x)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=out, stream=side,
                                 workspace=ws if need else None)
    side.synchronize()
    assert torch.equal(out, ref)
    assert np.isfinite(out.cpu().numpy()).all()


@pytest.mark.parametrize("m", [12, 16, 24])
def test_misaligned_buffers_rejected(cuda, m):
    """The TMA paths need 16-byte aligned rows; a 4-byte-offset view must be
    rejected with an argument error, never fault."""
    import torch

    import paper_1609_06641_b200 as chw

    rows = 2
    base = torch.zeros(rows * (1 << m) + 4, device=cuda)
    x = base[1:1 + rows * (1 << m)].view(rows, 1 << m)
    assert x.data_ptr() % 16 == 4
    with pytest.raises(ValueError, match="aligned"):
        chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()


def test_empty_batch_is_a_no_op(cuda):
    import torch

    import paper_1609_06641_b200 as chw

    for m in (12, 16, 24):
        x = torch.zeros(0, 1 << m, device=cuda)
        chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()
