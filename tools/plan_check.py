"""Offline checker for CHW tile plans (the layouts in csrc/plans.cuh).

For a plan — a sequence of layouts over T tile bits, a shared-memory XOR
swizzle, input/output position maps — it reports, per access instruction:
  * shared memory: wavefronts per warp instruction vs the conflict-free ideal
    (32 banks x 4 B; a 16-byte vector access serves 8 lanes per wavefront),
  * global memory: 32-byte sectors and 128-byte lines touched per warp
    instruction, and whether every touched sector is fully written/read by
    that instruction,
and checks that every butterfly bit is processed exactly once while held in
registers (or lanes, for shuffle butterflies).

    python tools/plan_check.py            # checks the plans named below
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence


@dataclass
class Layout:
    regs: Sequence[int]       # tile bit per register-index bit
    thr: Sequence[int]        # tile bit per thread-index bit (lanes = first 5)

    @property
    def e(self):
        return len(self.regs)


def apply_swz(x: int, swz: Sequence[tuple]) -> int:
    y = x
    for s, d in swz:
        y ^= ((x >> s) & 1) << d
    return y


def vec_bits(lay: Layout, pos, cap: int) -> int:
    vb = 0
    while vb < cap and any(pos(r) == vb for r in lay.regs):
        vb += 1
    return vb


def warp_addresses(lay: Layout, warp: int, r: int, pos):
    """Element positions touched by the 32 lanes for register index r."""
    out = []
    for lane in range(32):
        t = lane | (warp << 5)
        k = 0
        for i, b in enumerate(lay.regs):
            if (r >> i) & 1:
                k |= 1 << pos(b)
        for i, b in enumerate(lay.thr):
            if (t >> i) & 1:
                k |= 1 << pos(b)
        out.append(k)
    return out


def smem_cost(lay: Layout, swz, word_bytes: int, vcap: int, nwarps_check: int = 2):
    """(wavefronts, ideal) summed over all vector instructions of warps 0..n-1."""
    ident = lambda b: b  # noqa: E731
    vb = vec_bits(lay, ident, vcap)
    # vectors must not be split by the swizzle
    while vb > 0 and any(s < vb or d < vb for s, d in swz):
        vb -= 1
    vbytes = word_bytes << vb
    heads = [r for r in range(1 << lay.e)
             if all(((r >> lay.regs.index(q)) & 1) == 0 for q in range(vb))]
    wf = ideal = 0
    nw = min(nwarps_check, 1 << max(0, len(lay.thr) - 5))
    for w in range(nw):
        for r in heads:
            addrs = [apply_swz(a, swz) * word_bytes for a in warp_addresses(lay, w, r, ident)]
            lanes_per_wf = max(1, min(32, 128 // vbytes))
            for g in range(0, 32, lanes_per_wf):
                grp = addrs[g:g + lanes_per_wf]
                # bank conflict degree: max distinct 4-byte words per bank
                banks: Dict[int, set] = {}
                for a in grp:
                    for wb in range(0, vbytes, 4):
                        banks.setdefault(((a + wb) // 4) % 32, set()).add((a + wb) // 4)
                wf += max(len(v) for v in banks.values())
                ideal += 1
    return wf, ideal, vb


def global_cost(lay: Layout, pos, elem_bytes: int, vcap: int, nwarps_check: int = 2):
    vb = vec_bits(lay, pos, vcap)
    heads = [r for r in range(1 << lay.e)
             if all(((r >> i) & 1) == 0 for i, b in enumerate(lay.regs) if pos(b) < vb)]
    sectors = lines = instr = partial = 0
    nw = min(nwarps_check, 1 << max(0, len(lay.thr) - 5))
    for w in range(nw):
        for r in heads:
            addrs = [a * elem_bytes for a in warp_addresses(lay, w, r, pos)]
            vbytes = elem_bytes << vb
            touched = {}
            for a in addrs:
                for b in range(vbytes):
                    touched.setdefault((a + b) // 32, set()).add((a + b) % 32)
            sectors += len(touched)
            lines += len({s // 4 for s in touched})
            partial += sum(1 for v in touched.values() if len(v) < 32)
            instr += 1
    return {"vec_bytes": elem_bytes << vb, "instr": instr, "sectors_per_instr": sectors / instr,
            "lines_per_instr": lines / instr, "partial_sectors_per_instr": partial / instr}


@dataclass
class Plan:
    name: str
    T: int
    layouts: List[Layout]
    bfly: List[Sequence[int]]      # butterfly tile bits per layout (register bits)
    shfl: List[Sequence[int]] = field(default_factory=list)  # shuffle bits per layout
    swz: Sequence[tuple] = ()
    in_pos: Optional[callable] = None
    out_pos: Optional[callable] = None
    io_bytes: int = 4
    word_bytes: int = 4
    need: Sequence[int] = ()       # tile bits that must be butterflied


def check(p: Plan, verbose=True):
    ident = lambda b: b  # noqa: E731
    inp = p.in_pos or ident
    outp = p.out_pos or ident
    done = []
    for i, (lay, bits) in enumerate(zip(p.layouts, p.bfly)):
        assert sorted(list(lay.regs) + list(lay.thr)) == list(range(p.T)), f"layout {i} not a bit partition"
        for b in bits:
            assert b in lay.regs, f"layout {i}: butterfly bit {b} not in registers"
        done += list(bits)
        if i < len(p.shfl):
            for b in p.shfl[i]:
                assert b in lay.thr[:5], f"layout {i}: shuffle bit {b} not a lane bit"
            done += list(p.shfl[i])
    assert sorted(done) == sorted(p.need), f"butterflies {sorted(done)} != needed {sorted(p.need)}"
    vcap_io = {8: 1, 4: 2, 2: 3}[p.io_bytes]
    vcap_w = {8: 1, 4: 2}[p.word_bytes]
    res = {"load": global_cost(p.layouts[0], inp, p.io_bytes, vcap_io),
           "store": global_cost(p.layouts[-1], outp, p.io_bytes, vcap_io)}
    sm = []
    for i in range(len(p.layouts) - 1):
        st = smem_cost(p.layouts[i], p.swz, p.word_bytes, vcap_w)
        ld = smem_cost(p.layouts[i + 1], p.swz, p.word_bytes, vcap_w)
        sm.append({"sts_wf/ideal": f"{st[0]}/{st[1]} (vec {st[2]})", "lds_wf/ideal": f"{ld[0]}/{ld[1]} (vec {ld[2]})"})
    res["smem"] = sm
    if verbose:
        print(f"== {p.name}")
        for k, v in res.items():
            print(f"   {k}: {v}")
    return res


def rev_pos(m):
    return lambda b: (m - 1 - b) if b < m else b


PLANS = [
    Plan("f32 m=12 (PlanF32M12)", 12,
         [Layout([0, 1, 8, 9, 10, 11], [2, 3, 4, 5, 6, 7]), Layout([2, 3, 4, 5, 6, 7], [0, 1, 9, 10, 11, 8])],
         [[0, 1, 8, 9, 10, 11], [2, 3, 4, 5, 6, 7]], swz=[(9, 2), (10, 3), (11, 4)],
         out_pos=rev_pos(12), need=range(12)),
    Plan("bf16 m=7 x32 rows (PlanBF16M7)", 12,
         [Layout([0, 1, 2, 6], [3, 4, 5, 7, 8, 9, 10, 11]), Layout([3, 4, 5, 6], [0, 1, 2, 7, 8, 9, 10, 11])],
         [[0, 1, 2, 6], [3, 4, 5]], swz=[(5, 2), (7, 3), (8, 4)], out_pos=rev_pos(7), io_bytes=2,
         need=range(7)),
    Plan("f32 m=16 K6 B tile (RowPipeF32M16 ItemB0)", 12,
         [Layout([0, 1, 5, 8, 9], [2, 3, 4, 6, 7, 10, 11]), Layout([4, 6, 7, 10, 11], [9, 8, 5, 0, 1, 2, 3])],
         [[5, 8, 9], [4, 6, 7, 10, 11]], swz=[(5, 2), (8, 3), (9, 4)],
         out_pos=lambda b: [13, 12, 15, 14, 7, 6, 5, 4, 3, 2, 1, 0][b], need=range(4, 12)),
]


if __name__ == "__main__":
    for p in PLANS:
        check(p)
