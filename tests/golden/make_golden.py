"""Regenerate tests/golden/golden.npz from the UNMODIFIED reference.

Runs oracle/_ref/make_golden (built by `make -C oracle` from
/root/reference/proj/include; see oracle/make_golden.cpp for the cases and the
reference test lines each one mirrors) and packs its raw arrays into one
compressed .npz.  Only runnable where /root/reference exists (the builder
container); the GPU box only reads the committed golden.npz.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
DTYPES = {"f64": np.float64, "i64": np.int64, "u64": np.uint64}


def main() -> int:
    subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)
    exe = os.path.join(REPO, "oracle", "_ref", "make_golden")
    if not os.path.exists(exe):
        print("reference absent: cannot regenerate golden vectors", file=sys.stderr)
        return 1
    arrays = {}
    with tempfile.TemporaryDirectory() as d:
        subprocess.run([exe, d], check=True)
        with open(os.path.join(d, "index.txt")) as f:
            for line in f:
                name, dt, count = line.split()
                a = np.fromfile(os.path.join(d, name + ".bin"), dtype=DTYPES[dt])
                assert a.size == int(count), name
                arrays[name] = a
    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **arrays)
    print(f"wrote {len(arrays)} arrays to {out} ({os.path.getsize(out)} bytes)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
