"""Test infrastructure: execute libsv's gate-circuit schedule (sv_plan_gates)
on numpy shards, to check the product's host-side planner (pass packing,
commuting reorders, qubit swaps, per-rank control decisions) on the CPU.  A
pass applies its gates, in the plan's order, as the tile kernel is specified
to: Fig. 3's 2x2 on the gate's PHYSICAL target slot, restricted to indices
whose control bits are set; a swap is the all-to-all of contiguous chunks."""
from __future__ import annotations

import numpy as np

from tests.circuits import matrix_of
from tests.plan_exec import alltoall_chunks


def phys(q: int, nl: int, g: int, swapped: bool) -> int:
    if not swapped:
        return q
    if q >= nl:
        return q - g
    if q >= nl - g:
        return q + g
    return q


def apply_local(x: np.ndarray, t: int, cmask: int, M: np.ndarray) -> None:
    """The 2x2 on slot t of shard x where (local index & cmask) == cmask."""
    idx = np.arange(x.size, dtype=np.int64)
    lo = idx[((idx >> t) & 1) == 0]
    lo = lo[(lo & cmask) == cmask]
    hi = lo | (1 << t)
    u, v = x[lo].copy(), x[hi].copy()
    x[lo] = M[0, 0] * u + M[0, 1] * v
    x[hi] = M[1, 0] * u + M[1, 1] * v


def execute(steps, order, gates, shards, n, exchange=alltoall_chunks, ranks=None):
    P = len(shards)
    g = P.bit_length() - 1
    nl = n - g
    ranks = list(range(P)) if ranks is None else ranks
    state = [s.copy() for s in shards]
    swapped = False
    for st in steps:
        if st["kind"] == 1:
            state = exchange(state)
            swapped = not swapped
            continue
        assert st["kind"] in (0, 2)
        for k in range(st["first"], st["first"] + st["count"]):
            gt = gates[int(order[k])]
            t = phys(int(gt["target"]), nl, g, swapped)
            assert t < nl and (st["proc_mask"] >> t) & 1, "gate target not a processed slot of its pass"
            M = matrix_of(gt)
            for r in ranks:
                cm, live = 0, True
                for q in range(n):
                    if (int(gt["controls"]) >> q) & 1:
                        pq = phys(q, nl, g, swapped)
                        if pq < nl:
                            cm |= 1 << pq
                        elif not (r >> (pq - nl)) & 1:
                            live = False
                if live:
                    apply_local(state[r], t, cm, M)
    assert not swapped, "plan must end in the natural layout"
    return state
