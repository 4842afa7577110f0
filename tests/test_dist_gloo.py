"""Multi-process (world_size 2, gloo, CPU) tests of the N > 1 host path:
  * the torch.distributed plumbing the sharded bench/bootstrap uses
    (byte broadcast of the NCCL unique id, max-over-ranks timing);
  * libsv's sharded WHT schedule executed rank by rank with a REAL collective
    for the qubit-swap exchange (gloo all_to_all_single standing in for
    ncclAlltoAll, same chunk semantics), compared with the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, n, dtype, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD),
                      LOCAL_RANK=str(rank))
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_quant_ph_9804039_b200 as sv
        from paper_quant_ph_9804039_b200 import dist as svd
        from oracle import oracle as orc
        from tests.plan_exec import execute

        r, w, _ = svd.init_process_group("gloo")
        assert (r, w) == (rank, WORLD)
        # unique-id style broadcast and max-over-ranks
        payload = bytes(range(128)) if rank == 0 else None
        assert svd.broadcast_bytes(payload) == bytes(range(128))
        assert svd.max_over_ranks(float(rank + 1)) == float(WORLD)

        # sharded WHT schedule with a real collective for the exchange
        rng = np.random.default_rng(1234)  # same seed on both ranks -> same global state
        N = 1 << n
        a0 = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        a0 /= np.linalg.norm(a0)
        marked = orc.marked_from_seed(n, 7, 3)
        k = 2
        plan = sv.sv_plan_wht(n, WORLD, dtype, k, True)
        Nl = N // WORLD
        mine = a0[rank * Nl:(rank + 1) * Nl].copy()

        def exchange(states):
            # states holds only this rank's shard in slot `rank`; the others are placeholders
            send = torch.from_numpy(np.ascontiguousarray(states[rank]).view(np.float64).copy())
            recv = torch.empty_like(send)
            dist.all_to_all_single(recv, send)
            out = [None] * WORLD
            out[rank] = recv.numpy().view(np.complex128).copy()
            for j in range(WORLD):
                if out[j] is None:
                    out[j] = np.zeros(Nl, np.complex128)
            return out

        # execute(): every pass acts per shard; only our shard is real
        shards = [mine if j == rank else np.zeros(Nl, np.complex128) for j in range(WORLD)]
        got = execute(plan, shards, n, marked, exchange=exchange)[rank]
        ref = orc.iterate(a0.copy(), marked, k, orc.WHT)[rank * Nl:(rank + 1) * Nl]
        err = float(np.max(np.abs(got - ref)))
        result_q.put((rank, err, None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        result_q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("n,dtype", [(15, 0), (14, 1), (18, 0)])
def test_world2_sharded_schedule_with_gloo_alltoall(n, dtype):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, n, dtype, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, tb in res:
        assert tb is None, tb
        assert err <= 1e-12, (rank, err)


def _gate_worker(rank, port, n, dtype, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD),
                      LOCAL_RANK=str(rank))
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_quant_ph_9804039_b200 as sv
        from paper_quant_ph_9804039_b200 import dist as svd
        from oracle import oracle as orc
        from tests import circuits as C
        from tests.gate_exec import execute

        svd.init_process_group("gloo")
        rng = np.random.default_rng(77)  # same seed on both ranks -> same global state and circuit
        N = 1 << n
        a0 = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        a0 /= np.linalg.norm(a0)
        gates = C.random_circuit(n, 120, 5, max_controls=3)
        top = n - 1  # rank qubit: target and control
        gates = np.concatenate([gates, C.circuit([C.record(top, C.H), C.record(1, C.X, [top]),
                                                  C.record(top - 2, C.Y, [top])])])
        steps, order = sv.sv_plan_gates(n, WORLD, dtype, gates)
        assert any(s["kind"] == 1 for s in steps)
        Nl = N // WORLD

        def exchange(states):
            send = torch.from_numpy(np.ascontiguousarray(states[rank]).view(np.float64).copy())
            recv = torch.empty_like(send)
            dist.all_to_all_single(recv, send)
            out = [np.zeros(Nl, np.complex128) for _ in range(WORLD)]
            out[rank] = recv.numpy().view(np.complex128).copy()
            return out

        shards = [a0[j * Nl:(j + 1) * Nl].copy() if j == rank else np.zeros(Nl, np.complex128) for j in range(WORLD)]
        got = execute(steps, order, gates, shards, n, exchange=exchange, ranks=[rank])[rank]
        ref = orc.apply_gates(a0.copy(), gates)[rank * Nl:(rank + 1) * Nl]
        result_q.put((rank, float(np.max(np.abs(got - ref))), None))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        result_q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("n,dtype", [(15, 0), (14, 1)])
def test_world2_gate_plan_with_gloo_alltoall(n, dtype):
    """libsv's gate-circuit schedule (sv_plan_gates, NEXT-4) executed rank by
    rank with a real collective for its qubit swaps; controls on the rank
    qubit are decided per rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gate_worker, args=(r, port, n, dtype, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, tb in res:
        assert tb is None, tb
        assert err <= 1e-12, (rank, err)
