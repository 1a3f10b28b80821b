"""CPU check of the K6 row-pipeline synchronisation protocol (csrc/rowpipe.cuh)
through its executable model (tools/rowpipe_model.py): random interleavings of
the producer and compute roles with hardware mbarrier parity semantics must
never deadlock, consume a stale stage, break RAW (B(i, .) before A(i, .) is
stored) or WAR (A(i, k) before B(i-1, k) has landed).  The model also shows
why K6f requires even ring depths (enforced by a static_assert)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

import rowpipe_model as rm  # noqa: E402


@pytest.mark.parametrize("depths", [(2, 2), (4, 6), (6, 4), (8, 2), (5, 5), (7, 3)])
def test_one_group_per_stream(depths):
    assert rm.sweep(1, [depths], [1, 2, 3], range(8)) == []


@pytest.mark.parametrize("depths", [(2, 2), (4, 6), (6, 4), (8, 2)])
def test_two_groups_even_depths(depths):
    assert rm.sweep(2, [depths], [1, 2, 3], range(8)) == []


def test_two_groups_odd_depths_are_unsafe():
    assert rm.sweep(2, [(5, 5), (7, 3), (3, 3)], [2, 3], range(40)) != []
