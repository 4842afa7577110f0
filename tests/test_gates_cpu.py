"""Host-side checks of the NEXT-4 gate engine (no device): libsv's planner
(sv_plan_gates) executed on numpy shards equals the oracle; structural
properties of the schedule; argument validation through the C ABI."""
import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests import circuits as C
from tests.gate_exec import execute

T = {sv.SV_C64: 13, sv.SV_C128: 12}
CARRY = {sv.SV_C64: 3, sv.SV_C128: 2}


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return a / np.linalg.norm(a)


def noncommuting(a, b):
    ta, tb = int(a["target"]), int(b["target"])
    return ta == tb or (int(a["controls"]) >> tb) & 1 or (int(b["controls"]) >> ta) & 1


@pytest.mark.parametrize("n,world,dtype,seed", [(14, 1, 0, 1), (15, 2, 0, 2), (16, 4, 0, 3), (16, 8, 0, 4),
                                                  (13, 1, 1, 5), (14, 2, 1, 6), (10, 1, 0, 7), (17, 8, 1, 8)])
def test_plan_executes_to_oracle(n, world, dtype, seed):
    gates = C.random_circuit(n, 150, seed, max_controls=3)
    steps, order = sv.sv_plan_gates(n, world, dtype, gates)
    a0 = rand_state(n, 50 + seed)
    ref = orc.apply_gates(a0.copy(), gates)
    Nl = (1 << n) // world
    got = np.concatenate(execute(steps, order, gates, [a0[r * Nl:(r + 1) * Nl] for r in range(world)], n))
    np.testing.assert_allclose(got, ref, atol=1e-12, rtol=0)


@pytest.mark.parametrize("n,world,dtype", [(20, 1, 0), (20, 4, 0), (18, 2, 1), (9, 1, 1)])
def test_plan_structure(n, world, dtype):
    gates = C.random_circuit(n, 400, n + world, max_controls=2)
    steps, order = sv.sv_plan_gates(n, world, dtype, gates)
    assert sorted(order.tolist()) == list(range(gates.size))  # every gate exactly once
    pos = np.empty(gates.size, int)
    pos[order.astype(int)] = np.arange(gates.size)
    for i in range(gates.size):  # non-commuting pairs keep their order
        for j in range(i + 1, min(gates.size, i + 40)):
            if noncommuting(gates[i], gates[j]):
                assert pos[i] < pos[j], (i, j)
    g = world.bit_length() - 1
    nl = n - g
    for st in steps:
        if st["kind"] == 2:
            assert world == 1 and n <= T[dtype] and len(steps) == 1
        if st["kind"] == 0:
            tm, pm = st["tile_mask"], st["proc_mask"]
            assert bin(tm).count("1") == T[dtype] and pm & ~tm == 0 and tm >> nl == 0
            assert tm & ((1 << CARRY[dtype]) - 1) == (1 << CARRY[dtype]) - 1  # >= 64-byte contiguous runs
            assert st["count"] > 0
    assert sum(1 for s in steps if s["kind"] == 1) % 2 == 0  # natural layout restored


def test_pass_packing_counts():
    n = 24
    # 10 target qubits (+ 3 carry slots) fit one c64 tile -> one pass for any number of gates on them
    gates = C.random_circuit(n, 300, 1, max_controls=3, qubits=range(10, 20))
    steps, _ = sv.sv_plan_gates(n, 1, sv.SV_C64, gates)
    assert [s["kind"] for s in steps] == [0]
    # a layer of H on every qubit: slots [0, 13), then 10 + 3 carry, then the last one -> 3 passes
    layer = C.circuit([C.record(q, C.H) for q in range(n)])
    steps, _ = sv.sv_plan_gates(n, 1, sv.SV_C64, layer)
    assert len(steps) == 3
    # non-commuting gates on far-apart qubits: slots {0, 23} + carry fit one tile -> one pass
    alt = C.circuit([C.record(0, C.H, [23]), C.record(23, C.H, [0])] * 3)
    steps, _ = sv.sv_plan_gates(n, 1, sv.SV_C64, alt)
    assert len(steps) == 1


def test_swaps_only_for_rank_targets():
    n, world = 18, 4  # rank bits = qubits 16, 17
    local = C.random_circuit(n, 100, 3, max_controls=3, qubits=range(16))  # controls may be rank bits
    steps, _ = sv.sv_plan_gates(n, world, sv.SV_C64, local)
    assert all(s["kind"] == 0 for s in steps)
    # X(2) controlled by 16 commutes with H(17): it runs before the swap
    glob = C.circuit([C.record(17, C.H), C.record(2, C.X, [16]), C.record(16, C.H)])
    steps, _ = sv.sv_plan_gates(n, world, sv.SV_C64, glob)
    assert [s["kind"] for s in steps] == [0, 1, 0, 1]
    # controlled by 17 it does not: swap first, then all three in one pass, restore
    glob = C.circuit([C.record(17, C.H), C.record(2, C.X, [17]), C.record(16, C.H)])
    steps, _ = sv.sv_plan_gates(n, world, sv.SV_C64, glob)
    assert [s["kind"] for s in steps] == [1, 0, 1]


@pytest.mark.parametrize("rec", [C.record(20, C.X), C.record(-1, C.X), C.record(3, C.X, [3]),
                                 C.record(0, C.X, [20])])
def test_invalid_gates_rejected(rec):
    gates = C.circuit([rec])
    with pytest.raises(sv.SvError) as e:
        sv.sv_plan_gates(20, 1, sv.SV_C64, gates)
    assert e.value.code == sv.SV_EINVAL


def test_reserved_field_must_be_zero():
    bad = C.circuit([C.record(1, C.X)])
    bad["reserved"] = 1
    with pytest.raises(sv.SvError) as e:
        sv.sv_plan_gates(20, 1, sv.SV_C64, bad)
    assert e.value.code == sv.SV_EINVAL


def test_empty_circuit():
    steps, order = sv.sv_plan_gates(20, 2, sv.SV_C64, C.circuit([]))
    assert steps == [] and order.size == 0


def test_relayout_counts_follow_the_plan():
    """sv_debug_gate_relayouts: one count per schedule step, 0 for swaps; a
    pass whose gates all target one register layout needs none; a pass
    touching all 13 tile qubits of complex64 with general gates needs the
    layouts A, B and C (>= 2 changes)."""
    n = 20
    one = C.circuit([C.record(12, C.H), C.record(11, C.H)])
    steps, _ = sv.sv_plan_gates(n, 1, sv.SV_C64, one)
    rel = sv.sv_debug_gate_relayouts(n, 1, sv.SV_C64, one)
    assert len(rel) == len(steps) == 1 and rel[0] <= 1
    layer = C.circuit([C.record(q, C.H) for q in range(13)] + [C.record(q, C.X) for q in range(13)])
    rel = sv.sv_debug_gate_relayouts(n, 1, sv.SV_C64, layer)
    assert rel[0] >= 2
    g = C.random_circuit(n, 60, 4, max_controls=1)
    for world in (1, 4):
        steps, _ = sv.sv_plan_gates(n, world, sv.SV_C64, g)
        rel = sv.sv_debug_gate_relayouts(n, world, sv.SV_C64, g)
        assert len(rel) == len(steps)
        for st, r in zip(steps, rel):
            if st["kind"] != 0:
                assert r == 0
            else:
                assert r <= st["ops"]


def test_gate_jit_sources_compile_with_nvrtc():
    """Every pass kernel the gate JIT generates for representative circuits
    compiles for sm_100a with NVRTC (host only, both program flavours)."""
    import numpy as np
    from tests import circuits as C
    n = 16
    for gates in (C.qft_circuit(n), C.random_circuit(n, 60, 3, max_controls=3),
                  C.circuit([C.record(q, C.random_unitary(np.random.default_rng(q))) for q in range(n)])):
        r = sv.sv_debug_gate_jit(n, sv.SV_C64, gates, True)
        steps, _ = sv.sv_plan_gates(n, 1, sv.SV_C64, gates)
        assert r["passes"] == sum(1 for s in steps if s["kind"] == 0) > 0
    with pytest.raises(sv.SvError):
        sv.sv_debug_gate_jit(n, sv.SV_C128, C.qft_circuit(n), True)


def test_strided_pass_takes_the_two_layout_family():
    """A complex64 pass of general unitaries on qubits 3..12 (tile slots 0-12,
    lowest target tile bit 3) runs on the two-layout family (gates.cu
    gate_pass_l2): targets 8-12 in layout A, 3-7 in layout B -> ONE relayout.
    The three-layout family would need two (A holds 9-12, B 3-4, C 5-8);
    complex128 keeps it (its tiles are 12 bits)."""
    import os
    if os.environ.get("SV_GATE_L2") == "0":
        pytest.skip("two-layout gate passes switched off in this process")
    rng = np.random.default_rng(5)
    g = C.circuit([C.record(q, C.random_unitary(rng)) for q in range(3, 13)])
    steps, _ = sv.sv_plan_gates(16, 1, sv.SV_C64, g)
    assert len(steps) == 1
    assert list(sv.sv_debug_gate_relayouts(16, 1, sv.SV_C64, g)) == [1]
    # a target on tile bit 2 keeps the three-layout family (16-B pairs, layout C)
    g2 = C.circuit([C.record(q, C.random_unitary(rng)) for q in range(2, 13)])
    assert list(sv.sv_debug_gate_relayouts(16, 1, sv.SV_C64, g2)) == [2]
