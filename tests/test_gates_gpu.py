"""GPU parity of the NEXT-4 gate engine (sv_apply_gates): libsv's CUDA gate
tile passes vs the CPU oracle (or_apply_gates), element by element, through
the C ABI, on seeded random circuits (random targets, 0-3 controls, random
unitaries), the textbook QFT and Grover-as-gates; sharded schedules emulated
on one GPU with both exchange modes; full-size checks by properties that hold
at any size (QFT of a basis state: every amplitude in closed form, sampled;
circuit followed by its inverse = identity).

Tolerances: complex128 max-abs <= 1e-12 (north star).  complex64: max-abs
<= 1e-5 (north star) and <= gate64(G) x max|a_ref|, derived from the
arithmetic: one gate output w u + x v is 4 fp32 products and 3 adds of
unit-bounded terms (unitary m) plus the fp32 rounding of the 8 coefficients,
<= 8 x 2^-24 relative to the amplitude scale; G gates on one amplitude add at
most linearly -> 8 G 2^-24."""
import math

import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests import circuits as C

pytestmark = pytest.mark.gpu

TOL = {sv.SV_C128: 1e-12, sv.SV_C64: 1e-5}
DT = [sv.SV_C128, sv.SV_C64]
DT_IDS = ["c128", "c64"]


def gate64(G: int) -> float:
    return 8.0 * max(G, 1) * 2.0 ** -24


def assert_close(got, ref, dtype, G, what=""):
    got = np.asarray(got, dtype=np.complex128)
    err = float(np.max(np.abs(got - ref)))
    scale = float(np.max(np.abs(ref)))
    assert err <= TOL[dtype], f"{what}: max-abs {err:.3e} > {TOL[dtype]:.0e}"
    if dtype == sv.SV_C64:
        assert err <= gate64(G) * scale, f"{what}: max-abs {err:.3e} > {gate64(G):.2e} x {scale:.3e}"
    return err


def rand_state(n, dtype, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    a /= np.linalg.norm(a)
    return a.astype(sv.NP_DTYPE[dtype]).astype(np.complex128)  # the oracle starts from the dtype-rounded values


def run_gpu(a, dtype, gates, world=1, fused=None):
    n = a.size.bit_length() - 1
    with sv.sv_init(n, 0, dtype, sv.SV_INIT_ZERO_STATE, world=world) as c:
        if fused is not None:
            sv.sv_set_exchange(c, fused)
        sv.sv_set_amplitudes(c, a)
        sv.sv_apply_gates(c, gates)
        return sv.sv_get_amplitudes(c).astype(np.complex128)


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,count,seed", [(1, 5, 1), (5, 40, 2), (12, 120, 3), (13, 150, 4), (14, 150, 5),
                                          (17, 200, 6), (21, 120, 7)])
def test_random_circuit_matches_oracle(dtype, n, count, seed):
    gates = C.random_circuit(n, count, seed, max_controls=min(3, n - 1))
    a = rand_state(n, dtype, 100 + seed)
    ref = orc.apply_gates(a.copy(), gates)
    assert_close(run_gpu(a, dtype, gates), ref, dtype, count, f"n={n} G={count}")


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,count,seed", [(6, 80, 11), (13, 200, 12), (16, 300, 13), (22, 200, 14)])
def test_structured_gate_shapes_match_oracle(dtype, n, count, seed):
    # X / Y / Z / phase / diagonal / anti-diagonal / H / general, with controls
    gates = C.structured_circuit(n, count, seed, max_controls=3)
    a = rand_state(n, dtype, 200 + seed)
    ref = orc.apply_gates(a.copy(), gates)
    assert_close(run_gpu(a, dtype, gates), ref, dtype, count, f"structured n={n} G={count}")


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
def test_fusable_runs_match_oracle(dtype):
    # same-target same-control gates separated by commuting gates are fused
    # into one 2x2 on the host; separated by a non-commuting gate they are not
    n = 18
    rng = np.random.default_rng(3)
    recs = []
    for _ in range(6):
        for q in (0, 5, 11, 17):
            recs.append(C.record(q, C.random_unitary(rng), [3] if q != 3 else []))
        recs.append(C.record(9, C.phase(0.3), [0]))       # diagonal: blocks fusion on 0 and 9 only
        recs.append(C.record(5, C.X, [11]))               # non-diagonal on 5 controlled by 11
    gates = C.circuit(recs + [C.record(q, C.H) for q in range(n)] * 3)
    a = rand_state(n, dtype, 4)
    ref = orc.apply_gates(a.copy(), gates)
    assert_close(run_gpu(a, dtype, gates), ref, dtype, gates.size, "fusable runs")


def phase_run_circuit(n, seed):
    """Runs of phase gates diag(1, e^{i theta}) on one target with at most one
    control each (merged into one phase-polynomial op when >= 4 long), run
    lengths 1..12, controls anywhere (register, thread or free tile slots,
    none), interleaved with H / X on other qubits and a few 2-control phases."""
    rng = np.random.default_rng(seed)
    out = []
    for t in [0, 2, 5, 9, 12, n - 1, n // 2, 3, n - 2]:
        for _ in range(int(rng.integers(1, 13))):
            if rng.random() < 0.15:
                out.append(C.record(t, C.phase(float(rng.uniform(-3, 3)))))
            else:
                c = int(rng.choice([q for q in range(n) if q != t]))
                out.append(C.record(t, C.phase(float(rng.uniform(-3, 3))), [c]))
            if rng.random() < 0.3:  # commuting (other target, not a control of the run) or not
                q = int(rng.integers(0, n))
                if q != t:
                    out.append(C.record(q, C.H))
        out.append(C.record(t, C.H))
        cs = [q for q in range(n) if q != t][:2]
        out.append(C.record(t, C.phase(0.7), cs))
    return C.circuit(out)


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,world", [(16, 1), (21, 1), (19, 4)])
def test_phase_runs_match_oracle(dtype, n, world):
    gates = phase_run_circuit(n, n * 7 + world)
    a = rand_state(n, dtype, 300 + n)
    ref = orc.apply_gates(a.copy(), gates)
    assert_close(run_gpu(a, dtype, gates, world=world), ref, dtype, gates.size, f"phase runs n={n} P={world}")


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
def test_layered_circuit_matches_oracle(dtype):
    n = 20
    gates = C.layered_circuit(n, 4, 21)
    a = rand_state(n, dtype, 22)
    ref = orc.apply_gates(a.copy(), gates)
    assert_close(run_gpu(a, dtype, gates), ref, dtype, gates.size, "layered n=20")


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
def test_many_gates_on_few_qubits_one_pass(dtype):
    # 400 gates on 10 qubits: one tile pass with a long op program and relayouts
    n = 20
    gates = C.random_circuit(n, 400, 9, max_controls=3, qubits=[0, 1, 4, 5, 7, 9, 12, 15, 18, 19])
    steps, _ = sv.sv_plan_gates(n, 1, dtype, gates)
    assert len(steps) == 1
    a = rand_state(n, dtype, 10)
    ref = orc.apply_gates(a.copy(), gates)
    assert_close(run_gpu(a, dtype, gates), ref, dtype, 400, "one long pass")


# A pass's op program rides in the kernel's parameter space (constant bank)
# when it fits 24 KiB (256 records of 96 B: complex64 records carry the packed
# coefficient pairs, complex128 records the fp64 coefficients), else it is
# read from global memory: one pass on each side of the boundary.
PARAM_CAP = {sv.SV_C64: 256, sv.SV_C128: 256}


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("side", ["param", "global"])
def test_op_program_param_and_global_paths(dtype, side):
    n = 18
    count = PARAM_CAP[dtype] if side == "param" else 2 * PARAM_CAP[dtype]
    gates = C.random_circuit(n, count, 21, max_controls=2, qubits=[0, 2, 3, 6, 8, 11, 13, 16, 17])
    steps, _ = sv.sv_plan_gates(n, 1, dtype, gates)
    assert len(steps) == 1
    ops = steps[0]["ops"]
    assert (ops <= PARAM_CAP[dtype]) == (side == "param"), ops
    a = rand_state(n, dtype, 22)
    ref = orc.apply_gates(a.copy(), gates)
    assert_close(run_gpu(a, dtype, gates), ref, dtype, count, f"{side} op program ({ops} ops)")


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n", [4, 13, 16, 20])
def test_qft_equals_fft(dtype, n):
    a = rand_state(n, dtype, 30 + n)
    gates = C.qft_circuit(n)
    ref = np.fft.ifft(a) * math.sqrt(1 << n)
    assert_close(run_gpu(a, dtype, gates), ref, dtype, gates.size, f"QFT n={n}")


@pytest.mark.parametrize("n,k", [(10, 25), (16, 6)])
def test_grover_as_gates_equals_wht_engine(n, k):
    marked = int(orc.marked_from_seed(n, 1, 3)[0])
    with sv.sv_init(n, 0, sv.SV_C128, sv.SV_INIT_ZERO_STATE) as c:
        sv.sv_apply_gates(c, C.grover_circuit(n, marked, k))
        got = sv.sv_get_amplitudes(c)
    with sv.sv_init(n, 0, sv.SV_C128, sv.SV_INIT_UNIFORM) as c:
        sv.sv_set_marked(c, np.array([marked], np.uint64))
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        wht = sv.sv_get_amplitudes(c)
    # D_circuit = -(2|s><s| - I): a (-1)^k global phase
    assert float(np.max(np.abs(got - (-1) ** k * wht))) <= 1e-12


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,world", [(15, 2), (17, 4), (19, 8), (20, 4)])
@pytest.mark.parametrize("fused", [True, False], ids=["fused", "a2a"])
def test_emulated_sharding_matches_oracle(dtype, n, world, fused):
    gates = C.random_circuit(n, 160, n * world, max_controls=3)
    # make sure rank qubits are targets and controls
    top = n - 1
    gates = np.concatenate([gates, C.circuit([C.record(top, C.H), C.record(0, C.X, [top]),
                                              C.record(top - 1, C.Y, [2, top])])])
    a = rand_state(n, dtype, 7 * n + world)
    ref = orc.apply_gates(a.copy(), gates)
    assert_close(run_gpu(a, dtype, gates, world=world, fused=fused), ref, dtype, gates.size,
                 f"n={n} P={world} fused={fused}")


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
def test_many_asynchronous_calls(dtype):
    """Back-to-back sv_apply_gates calls without synchronisation (pinned,
    asynchronous program uploads; the device program buffer grows between
    calls) equal the oracle on the concatenated circuit."""
    n = 17
    chunks = [C.random_circuit(n, c, 40 + i, max_controls=2) for i, c in enumerate([3, 50, 7, 200, 1, 90, 30])]
    chunks.append(C.qft_circuit(n))
    a = rand_state(n, dtype, 41)
    ref = orc.apply_gates(a.copy(), np.concatenate(chunks))
    with sv.sv_init(n, 0, dtype, sv.SV_INIT_ZERO_STATE) as c:
        sv.sv_set_amplitudes(c, a)
        for g in chunks:
            sv.sv_apply_gates(c, g)
        got = sv.sv_get_amplitudes(c).astype(np.complex128)
    assert_close(got, ref, dtype, sum(g.size for g in chunks), "async chunks")


def test_empty_circuit_and_errors():
    a = rand_state(15, sv.SV_C64, 1)
    assert np.array_equal(run_gpu(a, sv.SV_C64, C.circuit([])), a)
    with sv.sv_init(15, 0, sv.SV_C64) as c:
        for rec in (C.record(15, C.X), C.record(2, C.X, [2]), C.record(0, C.X, [16])):
            with pytest.raises(sv.SvError) as e:
                sv.sv_apply_gates(c, C.circuit([rec]))
            assert e.value.code == sv.SV_EINVAL


@pytest.mark.parametrize("n", [28])
def test_full_size_qft_of_basis_state_closed_form(n):
    """QFT|x> = N^{-1/2} sum_y exp(2 pi i x y / N) |y>: every amplitude has a
    closed form; checked on a sample of indices at n = 28 (2 GiB c64)."""
    x = 0x5A5A5A5 & ((1 << n) - 1)
    prep = [C.record(q, C.X) for q in range(n) if (x >> q) & 1]
    gates = np.concatenate([C.circuit(prep), C.qft_circuit(n)])
    with sv.sv_init(n, 0, sv.SV_C64, sv.SV_INIT_ZERO_STATE) as c:
        sv.sv_apply_gates(c, gates)
        rng = np.random.default_rng(5)
        idx = np.unique(np.concatenate([[0, 1, (1 << n) - 1], rng.integers(0, 1 << n, 4000)]))
        got = np.array([sv.sv_get_amplitudes(c, int(i), 1)[0] for i in idx[:300]], np.complex128)
    N = 1 << n
    ref = np.exp(2j * np.pi * ((x * idx[:300].astype(np.int64)) % N) / N) / math.sqrt(N)
    assert_close(got, ref, sv.SV_C64, gates.size, "QFT n=28 sampled")


def test_full_size_circuit_then_inverse_is_identity():
    n = 30
    gates = C.random_circuit(n, 120, 77, max_controls=2)
    inv = gates[::-1].copy()
    for i in range(inv.size):
        M = C.matrix_of(inv[i]).conj().T
        inv[i] = C.record(int(inv[i]["target"]), M, [q for q in range(n) if (int(inv[i]["controls"]) >> q) & 1])
    with sv.sv_init(n, 4, sv.SV_C64, sv.SV_INIT_GAUSSIAN) as c:
        a0 = sv.sv_get_amplitudes(c, 0, 1 << 16).astype(np.complex128)
        tail0 = sv.sv_get_amplitudes(c, (1 << n) - (1 << 12), 1 << 12).astype(np.complex128)
        sv.sv_apply_gates(c, gates)
        sv.sv_apply_gates(c, inv)
        a1 = sv.sv_get_amplitudes(c, 0, 1 << 16).astype(np.complex128)
        tail1 = sv.sv_get_amplitudes(c, (1 << n) - (1 << 12), 1 << 12).astype(np.complex128)
    scale = float(np.max(np.abs(a0)))
    for u, v in ((a0, a1), (tail0, tail1)):
        assert float(np.max(np.abs(u - v))) <= gate64(2 * gates.size) * scale


def test_phase_runs_global_program_path():
    """The merged-phase-run op on the global-memory program path:
    the library reads SV_GATE_PARAM_OPS once per process, so the phase-run and
    program-path tests rerun in a subprocess with the parameter-space programs
    switched off (every pass then walks its program from global memory with
    the lane-parallel factor tree)."""
    import os
    import subprocess
    import sys
    if os.environ.get("SV_GATE_PARAM_OPS") == "0":
        pytest.skip("this is the subprocess")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SV_GATE_PARAM_OPS="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gates_gpu.py", "-k",
                        "test_phase_runs_match_oracle or test_op_program_param_and_global_paths or qft"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("n", [16, 22])
def test_two_layout_strided_passes_match_oracle(n):
    """Complex64 passes whose lowest non-diagonal target is tile bit 3 or 4 run
    on the two-layout family (gates.cu gate_pass_l2): unitaries, controlled
    gates (register / thread / tile-slot controls) and phase runs on qubits
    >= 3, against the oracle; n = 22 puts the targets in strided tiles."""
    rng = np.random.default_rng(n)
    recs = []
    for q in range(3, n):
        recs.append(C.record(q, C.random_unitary(rng)))
    for _ in range(60):
        t, c1, c2 = (int(v) for v in rng.choice(np.arange(3, n), 3, replace=False))
        recs.append(C.record(t, C.random_unitary(rng), controls=(c1,) if rng.random() < 0.5 else (c1, c2)))
    for q in range(4, n):
        recs.append(C.record(q, C.phase(0.1 * q), controls=(3,)))
    gates = C.circuit(recs)
    a = rand_state(n, sv.SV_C64, 17)
    ref = orc.apply_gates(a.copy(), gates)
    got = run_gpu(a, sv.SV_C64, gates)
    assert_close(got, ref, sv.SV_C64, len(recs), f"two-layout n={n}")


def test_three_layout_family_still_matches_oracle():
    """SV_GATE_L2=0 (read once per process): the oracle tests of strided
    circuits rerun in a subprocess on the three-layout family."""
    import os
    import subprocess
    import sys
    if os.environ.get("SV_GATE_L2") == "0":
        pytest.skip("this is the subprocess")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SV_GATE_L2="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gates_gpu.py", "-k",
                        "random_circuit or structured or two_layout or qft or emulated_sharding"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:]
