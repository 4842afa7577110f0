"""Test infrastructure: execute libsv's WHT schedule (sv_plan_wht) on numpy
shards, to check the product's host-side planner and its exchange semantics on
the CPU (no device).  Each pass does what the tile kernel is specified to do:
butterfly stages on the pass's processed slots, with the elementwise op (O or
F0) in between; a swap is the all-to-all of contiguous chunks."""
from __future__ import annotations

import numpy as np


def stages(x: np.ndarray, proc_mask: int) -> np.ndarray:
    """(u, v) -> (u + v, u - v) on every processed slot of a local shard."""
    N = x.size
    for s in range(N.bit_length() - 1):
        if (proc_mask >> s) & 1:
            y = x.reshape(-1, 2, 1 << s)
            u, v = y[:, 0, :].copy(), y[:, 1, :].copy()
            y[:, 0, :] = u + v
            y[:, 1, :] = u - v
    return x


def run_pass(x, step, rank, n, nl, marked_global):
    if step["pre"]:
        stages(x, step["proc_mask"])
    if step["mid"] == 1:  # oracle, natural layout
        lo, hi = rank << nl, (rank + 1) << nl
        loc = [int(m) - lo for m in marked_global if lo <= int(m) < hi]
        x[loc] = -x[loc]
    elif step["mid"] == 2:  # F0 with the 2^-n scale
        x *= -(2.0 ** -n)
        if rank == 0:
            x[0] = -x[0]
    if step["post"]:
        stages(x, step["proc_mask"])
    return x


def alltoall_chunks(shards):
    """recv[j] chunk r = send[r] chunk j (NCCL all-to-all semantics)."""
    P = len(shards)
    B = shards[0].size // P
    return [np.concatenate([shards[r][j * B:(j + 1) * B] for r in range(P)]) for j in range(P)]


def execute(plan, shards, n, marked_global, exchange=alltoall_chunks):
    P = len(shards)
    nl = n - (P.bit_length() - 1)
    state = [s.copy() for s in shards]
    recv = None
    for st in plan:
        if st["kind"] == 1:
            recv = exchange(state)
        elif st["kind"] == 0:
            src = recv if st["in_recv"] else state
            state = [run_pass(src[r].copy(), st, r, n, nl, marked_global) for r in range(P)]
        else:
            raise AssertionError("unexpected step kind in a sharded plan")
    return state
