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
