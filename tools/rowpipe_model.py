"""Executable model of the K6 row-pipeline synchronisation protocol
(paper_1609_06641_b200/csrc/rowpipe.cuh: rowpipe_ws_kernel / rowpipe_ws4_kernel).

Every role of one CTA is a Python generator that yields at the points where the
kernel blocks (mbarrier parity waits); a seeded random scheduler interleaves
them, and TMA copies complete at random later times.  mbarriers follow the
hardware rule the kernel relies on: a phase completes when its pending arrival
count reaches zero AND its expected transaction bytes have landed;
`try_wait.parity(P)` succeeds iff the barrier's current phase parity differs
from P (i.e. it cannot tell "one phase ago" from "three phases ago").

Checked on every run:
  * no deadlock (all roles finish);
  * every consumed stage holds the item the consumer expects (no stale data);
  * RAW: a B(i, k) copy starts only after all 16 A(i, .) tiles were stored;
  * WAR: an A(i, k) store happens only after the B(i-1, k) copy that reads the
    same workspace region has landed.

    python tools/rowpipe_model.py            # sweeps groups/ring depths/rows/seeds
"""
from __future__ import annotations

import random


class MBar:
    def __init__(self, count):
        self.count = count
        self.pending = count
        self.tx = 0
        self.phase = 0  # completed phases

    def _maybe_complete(self):
        if self.pending == 0 and self.tx == 0:
            self.phase += 1
            self.pending = self.count

    def arrive(self):
        self.pending -= 1
        assert self.pending >= 0, "arrival beyond the barrier count"
        self._maybe_complete()

    def arrive_expect_tx(self, nbytes):
        self.tx += nbytes
        self.arrive()

    def complete_tx(self, nbytes):
        self.tx -= nbytes
        self._maybe_complete()

    def test_parity(self, parity):
        return (self.phase & 1) != parity


class Violation(Exception):
    pass


def run(groups_per_stream: int, sa: int, sb: int, rows: int, seed: int) -> None:
    """Simulate one CTA owning `rows` rows; raise Violation on any failure."""
    rng = random.Random(seed)
    nst = 16 * rows
    full_a = [MBar(1) for _ in range(sa)]
    empty_a = [MBar(1) for _ in range(sa)]
    full_b = [MBar(1) for _ in range(sb)]
    empty_b = [MBar(1) for _ in range(sb)]
    regionfree = [MBar(1) for _ in range(16)]
    rowstored = MBar(groups_per_stream)
    stage_a = [None] * sa       # item held by each ring stage (after its copy lands)
    stage_b = [None] * sb
    stored = set()              # A(i, k) tiles stored to the workspace
    landed_b = set()            # B(i, k) copies that have landed
    inflight = []               # pending copies: (ring, stage, item, bar)

    def wait(bar, parity):
        while not bar.test_parity(parity):
            yield

    def producer_a():
        for t in range(nst):
            st = t % sa
            if t >= sa:
                yield from wait(empty_a[st], ((t // sa) - 1) & 1)
            full_a[st].arrive_expect_tx(1)
            inflight.append(("a", st, t, full_a[st]))
            yield

    def producer_b():
        for t in range(nst):
            i, k = divmod(t, 16)
            if k == 0:
                yield from wait(rowstored, i & 1)
            st = t % sb
            if t >= sb:
                yield from wait(empty_b[st], ((t // sb) - 1) & 1)
            if any((i, kk) not in stored for kk in range(16)):
                raise Violation(f"RAW: B({i},{k}) copy issued before row {i} was stored")
            full_b[st].arrive_expect_tx(1)
            inflight.append(("b", st, t, full_b[st]))
            yield

    def group_a(par):
        for t in range(par, nst, groups_per_stream):
            st = t % sa
            i, k = divmod(t, 16)
            yield from wait(full_a[st], (t // sa) & 1)
            if stage_a[st] != t:
                raise Violation(f"stale A stage: wanted item {t}, stage holds {stage_a[st]}")
            yield
            empty_a[st].arrive()
            if i >= 1:
                yield from wait(regionfree[k], (i - 1) & 1)
                if (i - 1, k) not in landed_b:
                    raise Violation(f"WAR: A({i},{k}) stored before B({i - 1},{k}) landed")
            stored.add((i, k))
            yield
            if k >= 16 - groups_per_stream:  # this group's last tile of the row
                rowstored.arrive()

    def group_b(par):
        for t in range(par, nst, groups_per_stream):
            st = t % sb
            i, k = divmod(t, 16)
            yield from wait(full_b[st], (t // sb) & 1)
            if stage_b[st] != t:
                raise Violation(f"stale B stage: wanted item {t}, stage holds {stage_b[st]}")
            yield
            empty_b[st].arrive()
            regionfree[k].arrive()

    roles = [producer_a(), producer_b()]
    roles += [group_a(p) for p in range(groups_per_stream)]
    roles += [group_b(p) for p in range(groups_per_stream)]
    live = list(roles)
    idle = 0
    while live or inflight:
        # land a random in-flight copy now and then
        if inflight and (not live or rng.random() < 0.3):
            ring, st, t, bar = inflight.pop(rng.randrange(len(inflight)))
            if ring == "a":
                stage_a[st] = t
            else:
                stage_b[st] = t
                landed_b.add(divmod(t, 16))
            bar.complete_tx(1)
            idle = 0
            continue
        if not live:
            break
        r = rng.choice(live)
        try:
            next(r)
        except StopIteration:
            live.remove(r)
            idle = 0
            continue
        idle += 1
        if idle > 200000:
            raise Violation("deadlock: no role can make progress")
    if live:
        raise Violation("deadlock")


def sweep(groups_per_stream, depths, rows_list, seeds):
    bad = []
    for sa, sb in depths:
        for rows in rows_list:
            for seed in seeds:
                try:
                    run(groups_per_stream, sa, sb, rows, seed)
                except Violation as e:
                    bad.append((sa, sb, rows, seed, str(e)))
                    break
    return bad


if __name__ == "__main__":
    even = [(2, 2), (4, 4), (4, 6), (6, 4), (8, 2)]
    odd = [(5, 5), (7, 3), (3, 3)]
    print("K6e (1 group per stream), any depth:", sweep(1, even + odd, [1, 2, 3], range(20)) or "ok")
    print("K6f (2 groups per stream), even depths:", sweep(2, even, [1, 2, 3], range(20)) or "ok")
    found = sweep(2, odd, [2, 3], range(40))
    print("K6f with odd depths (rejected at compile time):", f"{len(found)} violating configs, e.g. {found[:1]}")
