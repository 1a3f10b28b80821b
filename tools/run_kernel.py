"""Minimal driver for ncu / compute-sanitizer: transforms one BASELINE config
through the C ABI `--reps` times (no CPU baseline, no e2e, no copy kernel), so a
profiler sees only this library's kernels.

    python tools/run_kernel.py --config cfg2 --reps 3
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1609_06641_b200 as chw  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", choices=sorted(bench.CONFIGS))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rows", type=int, default=0, help="override the batch (0 = config's)")
    ap.add_argument("--mode", default="ortho", choices=["ortho", "unnorm"])
    args = ap.parse_args()
    name, dt, rows, m, _ = bench.CONFIGS[args.config]
    rows = args.rows or rows
    dev = torch.device("cuda:0")
    x = bench.make_input(torch, args.config, 0, rows, dev)
    out = torch.empty_like(x)
    mode = chw.ScalingMode.Orthonormal if args.mode == "ortho" else chw.ScalingMode.Unnormalized
    for _ in range(args.reps):
        chw.chw_forward_batched_(x, mode, out=out)
    torch.cuda.synchronize()
    print(f"{name}: {args.reps} reps ok, plan {chw.plan_name({'f64': 0, 'f32': 1, 'bf16': 2}[dt], 1 << m)}")


if __name__ == "__main__":
    main()
