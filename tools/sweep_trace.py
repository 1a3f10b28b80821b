"""Timeline of the K9 m = 24 sweep (debug build ab/lib_trace.so, compiled
with -DCHW_SWEEP_TRACE=1): per-tile %globaltimer stamps of CTA 0 and 1, both
groups, summarised as per-phase durations (us).

    CHW_B200_LIB=$PWD/ab/lib_trace.so python tools/sweep_trace.py [rows]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1609_06641_b200 as chw  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dev = torch.device("cuda:0")
buf = torch.zeros(2 * 2 * 512 * 8, dtype=torch.int64, device=dev)
chw.lib.chw_b200_debug_sweep_trace.argtypes = [ctypes.c_void_p]
x = torch.randn(rows, 1 << 24, device=dev)
out = torch.empty_like(x)
for _ in range(2):
    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=out)
torch.cuda.synchronize()
assert chw.lib.chw_b200_debug_sweep_trace(buf.data_ptr()) == 0
chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=out)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(2, 2, 512, 8).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1000.0, np.nan)  # us
nt = 7
for cta in range(2):
    A = t[cta, 0]
    B = t[cta, 1]
    n = rows * nt
    a_wait_in = A[:n, 1] - A[:n, 0]
    a_comp = A[:n, 2] - A[:n, 1]
    a_wait_rf = A[:n, 3] - A[:n, 2]
    a_store = A[:n, 4] - A[:n, 3]
    b_issue = B[:n, 1] - B[:n, 0]
    b_wait = B[:n, 2] - B[:n, 1]
    b_comp = B[:n, 3] - B[:n, 2]
    b_l0 = B[:n, 4] - B[:n, 2]
    b_b0 = B[:n, 5] - B[:n, 4]
    b_h0 = B[:n, 6] - B[:n, 5]
    b_h1 = B[:n, 3] - B[:n, 6]
    span = np.nanmax(B[:n, 3]) - np.nanmin(A[:n, 0])
    print(f"CTA {cta}: span {span:.1f} us for {rows} rows = {span / rows:.2f} us/row")
    for name, arr in [("A wait input", a_wait_in), ("A compute", a_comp), ("A wait regionfree", a_wait_rf),
                      ("A store+signal", a_store), ("B wait cnt/issue", b_issue), ("B wait data", b_wait),
                      ("B compute+store", b_comp), ("  B LDS L0+bar", b_l0), ("  B B0 bfly", b_b0),
                      ("  B half0 T+B1+STG", b_h0), ("  B half1 T+B1+STG", b_h1)]:
        print(f"   {name:18s} mean {np.nanmean(arr):6.2f}  sum/row {np.nansum(arr) / rows:6.2f}")
    # per row: when B of row r starts (tile 0 data ready) vs when A of row r finished
    for r in range(min(rows, 4)):
        a_end = np.nanmax(A[r * nt:(r + 1) * nt, 4])
        b_start = B[r * nt, 2]
        b_end = B[(r + 1) * nt - 1, 3]
        print(f"   row {r}: A done {a_end:7.2f}  B first data {b_start:7.2f}  B done {b_end:7.2f}")
