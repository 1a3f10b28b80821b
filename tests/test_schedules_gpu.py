"""GPU parity of the long-row schedules, one subprocess per schedule (the
library reads CHW_B200_* once per process).

m = 16 (cfg4): the K6 row pipeline; m = 24 (cfg5): the K9 single-pass row
sweep (default) and the K4T two-pass schedule (t); m = 12 (cfg2): K1T.  Each
run checks f32 Orthonormal against the oracle (rel-L2 <= 1e-5), in-place ==
out-of-place, the exact dyadic order through the integer probe, and Parseval
on every row, for batch sizes that leave some CTAs with 0, 1, 2 or 3 rows
(tools/sched_check.py).  (The measured-and-superseded variants of round 1 —
K1P, K3, K5, K6e, K4P — were removed from the library in round 2.)
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


def test_m16_rowpipe(cuda):
    out = _run({}, 16, [1, 2, 3, 149, 300, 445])
    assert "k6-rowpipe" in out


def test_m16_cluster_dsmem(cuda):
    """K10 (CHW_B200_M16=c): 4-CTA clusters, the row exchanged through
    distributed shared memory; batches below, at and across the cluster count."""
    out = _run({"CHW_B200_M16": "c"}, 16, [1, 2, 3, 5, 33, 67, 300, 445])
    assert "k10-cluster-dsmem" in out


def test_m16_default_is_rowpipe(cuda):
    env = {k: v for k, v in os.environ.items() if k != "CHW_B200_M16"}
    p = subprocess.run([sys.executable, os.path.join(REPO, "tools", "sched_check.py"), "--m", "16", "--rows", "5"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "k6-rowpipe" in p.stdout


@pytest.mark.parametrize("variant", ["default", "t"])
def test_m24_schedules(cuda, variant):
    env = {k: v for k, v in os.environ.items() if k != "CHW_B200_M24"}
    if variant != "default":
        env["CHW_B200_M24"] = variant
    cmd = [sys.executable, os.path.join(REPO, "tools", "sched_check.py"), "--m", "24", "--rows", "1", "2", "3", "17"]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    want = {"default": "k9-row-sweep", "t": "k4t-two-pass-tma"}[variant]
    assert want in p.stdout


def test_m12_k1t(cuda):
    """f32 m = 12 (cfg2): the TMA-fed K1T kernel, batches that wrap its ring."""
    out = _run({}, 12, [1, 5, 148, 149, 1000, 4097])
    assert "k1t-tma" in out


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
