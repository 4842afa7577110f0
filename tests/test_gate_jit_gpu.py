"""Pass-specialised gate kernels (gate_jit.cu, NVRTC at run time) against the
op-program interpreter they replace -- bitwise, since every op is the same
device function in the same order -- and against the oracle (or_apply_gates),
on every op shape the planner emits: general / diagonal / phase / anti-diagonal
/ NOT 2x2s with register, thread and free-slot controls, diagonal gates on
thread bits (DIAGT), merged phase runs (QFT, phase-run circuits) in both
program flavours (constant bank / global memory), relayouts between all
three register layouts."""
import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests import circuits as C
from tests.test_gates_gpu import assert_close, phase_run_circuit, rand_state, run_gpu

pytestmark = pytest.mark.gpu


def circuits(n):
    return {
        "u_layer": C.circuit([C.record(q, C.random_unitary(np.random.default_rng(q))) for q in range(n)]),
        "qft": C.qft_circuit(n),
        "random": C.random_circuit(n, 160, 5, max_controls=3),
        "structured": C.structured_circuit(n, 160, 6, max_controls=2),
        "layered": C.layered_circuit(n, 2, 7),
        "phase_runs": phase_run_circuit(n, 11),
        "grover": C.grover_circuit(n, 5, 2),
    }


@pytest.mark.parametrize("name", ["u_layer", "qft", "random", "structured", "layered", "phase_runs", "grover"])
@pytest.mark.parametrize("n", [16, 20])
def test_jit_equals_interpreter_and_oracle(name, n, monkeypatch):
    gates = circuits(n)[name]
    a = rand_state(n, sv.SV_C64, 40 + n)
    monkeypatch.setenv("SV_GATE_JIT", "0")
    interp = run_gpu(a, sv.SV_C64, gates)
    monkeypatch.setenv("SV_GATE_JIT", "1")
    before = sv.sv_debug_gate_jit()["compiles"]
    jit = run_gpu(a, sv.SV_C64, gates)
    np.testing.assert_array_equal(jit, interp)
    steps, _ = sv.sv_plan_gates(n, 1, sv.SV_C64, gates)
    if any(s["kind"] == 0 for s in steps):  # tile passes ran specialised (compiled now or cached)
        assert sv.sv_debug_gate_jit()["compiles"] >= before
    assert_close(jit, orc.apply_gates(a.copy(), gates), sv.SV_C64, gates.size, f"jit {name} n={n}")


def test_jit_global_program_flavour(monkeypatch):
    """Merged phase runs read the program from global memory when it exceeds
    the parameter space (or SV_GATE_PARAM_OPS=0 in a fresh process): the
    specialised kernel then takes the same global flavour."""
    n = 18
    gates = np.concatenate([phase_run_circuit(n, 3)] * 6)  # long passes: > 256 records
    a = rand_state(n, sv.SV_C64, 9)
    monkeypatch.setenv("SV_GATE_JIT", "0")
    interp = run_gpu(a, sv.SV_C64, gates)
    monkeypatch.setenv("SV_GATE_JIT", "1")
    np.testing.assert_array_equal(run_gpu(a, sv.SV_C64, gates), interp)


def test_jit_automatic_at_large_states(monkeypatch):
    """Unset SV_GATE_JIT: passes of >= 2^11 tiles (n >= 24) run on the
    interpreter at a program's first call and on the specialised kernel, compiled
    then, from the second; both runs agree bitwise and with the oracle."""
    monkeypatch.delenv("SV_GATE_JIT", raising=False)
    n = 24
    gates = C.random_circuit(n, 40, 8, max_controls=2)
    before = sv.sv_debug_gate_jit()["compiles"]
    with sv.sv_init(n, 3, sv.SV_C64, sv.SV_INIT_GAUSSIAN) as c:
        a0 = sv.sv_get_amplitudes(c).astype(np.complex128)
        sv.sv_apply_gates(c, gates)  # first sight: interpreter, nothing compiled
        first = sv.sv_get_amplitudes(c)
        assert sv.sv_debug_gate_jit()["compiles"] == before
        sv.sv_set_amplitudes(c, a0)
        sv.sv_apply_gates(c, gates)  # second call: compiled, specialised kernels
        second = sv.sv_get_amplitudes(c)
    assert sv.sv_debug_gate_jit()["compiles"] > before
    np.testing.assert_array_equal(first, second)
    assert_close(second, orc.apply_gates(a0, gates), sv.SV_C64, gates.size, "auto jit n=24")
