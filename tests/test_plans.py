"""CPU checks of the round-2 tile plans with the offline cost model
(tools/plan_check.py): every shared-memory round trip of the K9 row sweep
(dyadic and natural-order plans) and of the K10 cluster kernel is
bank-conflict free (wavefronts == ideal), every global access moves
whole 32-byte sectors, and every butterfly bit is covered exactly once."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from plan_check import Layout, global_cost, smem_cost  # noqa: E402

# K9 (csrc/sweep.cuh: SweepF32M24)
A0 = Layout([0, 1, 5, 6, 7, 8, 9], [2, 3, 4, 10, 11, 12, 13])
A1 = Layout([2, 3, 4, 10, 11, 12, 13], [5, 6, 0, 1, 7, 8, 9])
AS = [(5, 2), (6, 3), (7, 4)]
A_OUT_P = [4, 5, 0, 1, 9, 2, 3, 6, 7, 8, 10, 11, 12, 13]
A_OUT_Q = [14, 15, 0, 1, 19, 2, 3, 16, 17, 18, 20, 21, 22, 23]
B0 = Layout([0, 1, 7, 8, 9, 10, 11], [2, 3, 4, 5, 6, 12, 13])
BH0 = Layout([0, 6, 7, 8, 9, 10], [1, 2, 3, 4, 5, 11, 12])
BH1 = Layout([12, 11, 3, 4, 5, 0], [10, 9, 8, 7, 6, 1, 2])
BHS = [(7, 1), (8, 2), (9, 3), (10, 4)]
B_OUT_H = [20, 18, 17, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0]


def _ideal(c):
    wf, ideal, _ = c
    return wf == ideal


def test_k9_shared_round_trips_conflict_free():
    assert _ideal(smem_cost(A0, [], 4, 2))           # A stage read (natural order)
    assert _ideal(smem_cost(A0, AS, 4, 2))           # A transpose store
    assert _ideal(smem_cost(A1, AS, 4, 2))           # A transpose load
    assert _ideal(smem_cost(B0, [], 4, 2))           # B stage read
    assert _ideal(smem_cost(BH0, BHS, 4, 2))         # B half transposes
    assert _ideal(smem_cost(BH1, BHS, 4, 2))


@pytest.mark.parametrize("lay,pos", [(A1, A_OUT_P), (A1, A_OUT_Q), (BH1, B_OUT_H)])
def test_k9_global_accesses_whole_sectors(lay, pos):
    g = global_cost(lay, lambda b: pos[b], 4, 2)
    assert g["vec_bytes"] == 16
    assert g["partial_sectors_per_instr"] == 0
    assert g["sectors_per_instr"] == 16


def test_k9_butterfly_coverage():
    # A: j0, j1, j4..j13 (passengers j2, j3 go to B); B: t0, t1 (= j2, j3) and
    # t4..t13 (= j14..j23): together every j bit exactly once.
    a_bits = {0, 1, 5, 6, 7, 8, 9} | {4, 10, 11, 12, 13}
    b_bits_t = {0, 1, 7, 8, 9, 10, 11} | {4, 5, 6, 12, 13}
    t_to_j = {0: 2, 1: 3, 2: 5, 3: 6, **{k: 10 + k for k in range(4, 14)}}
    b_bits = {t_to_j[t] for t in b_bits_t}
    assert a_bits.isdisjoint(b_bits)
    assert a_bits | b_bits == set(range(24))


def test_k9n_natural_plan():
    """K9n (csrc/sweep.cuh: SweepNatF32M24): natural order folded into the
    sweep — 16-byte accesses on both sides of A's transpose, B's first layout
    conflict-free under TMA's 64-byte swizzle, in-place transpose, scalar
    stores in whole sectors; every row bit butterflied exactly once."""
    a0 = Layout([0, 1, 5, 6, 7, 8, 9], [2, 3, 4, 10, 11, 12, 13])
    a1 = Layout([0, 1, 4, 10, 11, 12, 13], [2, 3, 5, 6, 7, 8, 9])
    a_s = [(5, 4)]
    for c in (smem_cost(a0, [], 4, 2, 4), smem_cost(a0, a_s, 4, 2, 4), smem_cost(a1, a_s, 4, 2, 4)):
        assert _ideal(c) and c[2] == 2          # all three are 16-byte vector accesses
    out_p = list(range(14))
    out_q = [0, 1, 2, 3] + list(range(14, 24))
    for pos in (out_p, out_q):
        g = global_cost(a1, lambda b: pos[b], 4, 2, 4)
        assert g["vec_bytes"] == 16 and g["partial_sectors_per_instr"] == 0
    b0 = Layout([0, 1, 2, 3, 7, 8, 9], [4, 5, 6, 10, 11, 12, 13])
    b1 = Layout([4, 5, 6, 10, 11, 12, 13], [0, 1, 2, 3, 7, 8, 9])
    tma64 = [(5, 2), (6, 3)]                    # CU_TENSOR_MAP_SWIZZLE_64B on float-index bits
    bs = [(5, 2), (6, 3), (7, 4)]
    assert _ideal(smem_cost(b0, tma64, 4, 2, 4))
    assert _ideal(smem_cost(b0, bs, 4, 2, 4)) and _ideal(smem_cost(b1, bs, 4, 2, 4))
    g = global_cost(b1, lambda b: out_q[b], 4, 2, 4)   # natural position of B tile bit t
    assert g["partial_sectors_per_instr"] == 0 and g["sectors_per_instr"] == 4
    a_bits = {0, 1, 5, 6, 7, 8, 9} | {4, 10, 11, 12, 13}
    t_to_j = {0: 0, 1: 1, 2: 2, 3: 3, **{k: 10 + k for k in range(4, 14)}}
    b_bits = {t_to_j[t] for t in ({2, 3, 7, 8, 9} | {4, 5, 6, 10, 11, 12, 13})}
    assert a_bits.isdisjoint(b_bits) and a_bits | b_bits == set(range(24))


def test_k10_cluster_plan():
    """K10 (csrc/clusterm16.cuh: ClusterF32M16): the in-quarter transpose, the
    exchange blocks (writer side per destination, reader side) and the output
    stores are conflict-free / whole sectors, and the three layouts cover all
    16 row bits exactly once."""
    l0 = Layout([0, 1, 9, 10, 11, 12], [2, 3, 4, 5, 6, 7, 8, 13])
    l1 = Layout([2, 3, 4, 5, 6, 13], [7, 8, 9, 0, 1, 10, 11, 12])
    s1 = [(7, 2), (8, 3), (9, 4)]
    assert _ideal(smem_cost(l0, [], 4, 2, 8))    # stage read (natural order)
    assert _ideal(smem_cost(l0, s1, 4, 2, 8))    # transpose store
    assert _ideal(smem_cost(l1, s1, 4, 2, 8))    # transpose load (scalar)
    lw = Layout([0, 1, 9, 10, 11, 8], [2, 3, 4, 5, 6, 7])
    lr = Layout([13, 12, 2, 3, 0, 1], [4, 5, 6, 7, 8, 9, 10, 11])
    sx = [(5, 2), (6, 3)]
    assert _ideal(smem_cost(lw, sx, 4, 2, 2))    # exchange block store
    assert _ideal(smem_cost(lr, sx, 4, 2, 8))    # exchange read
    out = [13, 12, 8, 7, 6, 5, 4, 3, 2, 11, 10, 9, 1, 0]
    g = global_cost(lr, lambda b: out[b], 4, 2, 8)
    assert g["vec_bytes"] == 16 and g["partial_sectors_per_instr"] == 0 and g["sectors_per_instr"] == 16
    # exchange-tile bit e_k -> row bit j
    e_to_j = [2, 3, 7, 8, 9, 10, 11, 12, 13, 4, 5, 6, 14, 15]
    bits = [0, 1, 9, 10, 11, 12] + [2, 3, 4, 5, 6, 13] + [e_to_j[e] for e in (13, 12, 2, 3)]
    assert sorted(bits) == list(range(16))
    # the dyadic position of row bit j is 15 - j; the CTA rank supplies j0, j1
    assert [15 - e_to_j[e] for e in range(14)] == out
