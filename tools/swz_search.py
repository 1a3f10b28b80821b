"""Search XOR swizzles (pairs src->dst on the tile index) that make a
layout-change round trip through shared memory bank-conflict free
(tools/plan_check.py cost model).  Used to pick the K9 (m = 24 row sweep) tile
swizzles; prints the best candidates.

    python tools/swz_search.py
"""
import itertools
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from plan_check import Layout, Plan, check, smem_cost  # noqa: E402


def search(l0, l1, T, vb_keep, max_pairs=3, dsts=(2, 3, 4)):
    srcs = [b for b in range(vb_keep, T) if b not in dsts]
    best = []
    for k in range(0, max_pairs + 1):
        for ds in itertools.combinations(dsts, k):
            for ss in itertools.permutations(srcs, k):
                swz = list(zip(ss, ds))
                st = smem_cost(l0, swz, 4, 2, nwarps_check=2)
                ld = smem_cost(l1, swz, 4, 2, nwarps_check=2)
                score = st[0] / st[1] * (4 >> st[2] if False else 1), ld[0] / ld[1]
                best.append(((st[0] + ld[0]) / (st[1] + ld[1]), swz, st, ld))
    best.sort(key=lambda t: t[0])
    return best[:5]


if __name__ == "__main__":
    A0 = Layout([0, 1, 5, 6, 7, 8, 9], [2, 3, 4, 10, 11, 12, 13])
    A1 = Layout([2, 3, 4, 10, 11, 12, 13], [5, 6, 0, 1, 7, 8, 9])
    print("A (L0 -> L1):")
    for r in search(A0, A1, 14, 2):
        print("  ", r[0], r[1], "sts", r[2], "lds", r[3])
    B0 = Layout([0, 1, 7, 8, 9, 10, 11], [2, 3, 4, 5, 6, 12, 13])
    B1 = Layout([13, 12, 4, 5, 6, 0, 1], [11, 10, 9, 8, 7, 2, 3])
    print("B (L0 -> L1):")
    for r in search(B0, B1, 14, 2):
        print("  ", r[0], r[1], "sts", r[2], "lds", r[3])
