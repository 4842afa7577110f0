"""Error behaviour of the C ABI as include/sv.h states it, called through
the raw entry points (ctypes, no Python-side checks in between).

CPU part: every context entry point rejects a NULL context with SV_EINVAL
and a message, before touching the device; the host-only planners and
generators reject invalid arguments.  GPU part (-m gpu): on a live context
every documented invalid argument returns its code, sv_last_error() says why,
and a rejected call leaves the state and the marked set unchanged."""
import ctypes

import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv

lib = sv.lib
NULL = None


def last():
    return lib.sv_last_error().decode()


def gates_arr(rows):
    g = np.zeros(len(rows), dtype=sv.GATE_DTYPE)
    for i, (t, ctl, res) in enumerate(rows):
        g[i]["target"], g[i]["controls"], g[i]["reserved"] = t, ctl, res
        g[i]["m"] = [0, 0, 1, 0, 1, 0, 0, 0]  # NOT
    return g


NULL_CTX_CALLS = {
    "sv_reset": lambda: lib.sv_reset(NULL, 0, 0),
    "sv_set_marked": lambda: lib.sv_set_marked(NULL, NULL, 0),
    "sv_apply_oracle": lambda: lib.sv_apply_oracle(NULL, NULL, 0),
    "sv_diffuse": lambda: lib.sv_diffuse(NULL, 0),
    "sv_iterate": lambda: lib.sv_iterate(NULL, 1, 0),
    "sv_iterate_noisy": lambda: lib.sv_iterate_noisy(NULL, 1, 0.01, 0, 0),
    "sv_iterate_decoherent": lambda: lib.sv_iterate_decoherent(NULL, 1, 0.0, 0.1, 0, 0, NULL),
    "sv_probabilities": lambda: lib.sv_probabilities(NULL, NULL, 0, 0),
    "sv_sample": lambda: lib.sv_sample(NULL, 0, 0, NULL, 0),
    "sv_measure_marked_mass": lambda: lib.sv_measure_marked_mass(NULL, ctypes.byref(ctypes.c_double())),
    "sv_get_amplitudes": lambda: lib.sv_get_amplitudes(NULL, NULL, 0, 0),
    "sv_set_amplitudes": lambda: lib.sv_set_amplitudes(NULL, NULL, 0, 0),
    "sv_info": lambda: lib.sv_info(NULL, None, None, None, None, None),
    "sv_set_exchange": lambda: lib.sv_set_exchange(NULL, 0),
    "sv_get_exchange": lambda: lib.sv_get_exchange(NULL, ctypes.byref(ctypes.c_int())),
    "sv_synchronize": lambda: lib.sv_synchronize(NULL),
    "sv_comm_info": lambda: lib.sv_comm_info(NULL, None, None),
    "sv_norm2": lambda: lib.sv_norm2(NULL, ctypes.byref(ctypes.c_double())),
    "sv_attach": lambda: lib.sv_attach(NULL, NULL, 0),
    "sv_snapshot": lambda: lib.sv_snapshot(NULL, b"/tmp/x", None),
    "sv_apply_gates": lambda: lib.sv_apply_gates(NULL, NULL, 0),
    "sv_profile": lambda: lib.sv_profile(NULL, 1),
    "sv_profile_read": lambda: lib.sv_profile_read(NULL, 0, None, None),
    "sv_profile_timeline": lambda: lib.sv_profile_timeline(NULL, None, None, 0, None),
}


@pytest.mark.parametrize("name", sorted(NULL_CTX_CALLS))
def test_null_context_is_einval(name):
    assert NULL_CTX_CALLS[name]() == sv.SV_EINVAL
    assert "ctx is NULL" in last()


def test_every_context_entry_point_is_covered():
    from tests.test_abi_cpu import declared_functions
    ctx_free = {"sv_init", "sv_marked_from_seed", "sv_nccl_unique_id", "sv_plan_wht", "sv_plan_gates", "sv_free",
                "sv_debug_gate_relayouts", "sv_debug_wht_variants", "sv_debug_gate_jit",
                "sv_last_error", "sv_debug_tile_layout", "sv_debug_tile_owner"}
    assert set(declared_functions()) - ctx_free == set(NULL_CTX_CALLS)


def test_free_null_and_success_clears_message():
    lib.sv_free(NULL)  # NULL-safe
    assert lib.sv_reset(NULL, 0, 0) == sv.SV_EINVAL and last()
    out = np.zeros(1, np.uint64)
    assert lib.sv_marked_from_seed(4, 1, 0, out.ctypes.data) == sv.SV_OK
    assert last() == ""


def test_init_rejects_before_device():
    p = ctypes.c_void_p()
    assert lib.sv_init(None, 12, 0, sv.SV_C64, 0, None) == sv.SV_EINVAL
    for n, dt in ((0, sv.SV_C64), (41, sv.SV_C64), (12, 2), (12, -1)):
        assert lib.sv_init(ctypes.byref(p), n, 0, dt, 0, None) == sv.SV_EINVAL, (n, dt)
        assert p.value is None
    for world in (0, 3, 6, -2):
        d = sv.sv_dist(0, world, None, 0, None)
        assert lib.sv_init(ctypes.byref(p), 20, 0, sv.SV_C64, 0, ctypes.byref(d)) == sv.SV_EINVAL
    d = sv.sv_dist(0, 4, None, 0, None)
    assert lib.sv_init(ctypes.byref(p), 1, 0, sv.SV_C64, 0, ctypes.byref(d)) == sv.SV_EINVAL  # 2^g > 2^n


def test_host_planners_reject_invalid_arguments():
    out = (sv.sv_plan_step * 4)()
    ns = ctypes.c_int()
    assert lib.sv_plan_wht(20, 3, sv.SV_C64, 1, 1, out, 4, ctypes.byref(ns)) == sv.SV_EINVAL
    assert lib.sv_plan_wht(20, 1, sv.SV_C64, -1, 1, out, 4, ctypes.byref(ns)) == sv.SV_EINVAL
    assert lib.sv_plan_wht(20, 1, 5, 1, 1, out, 4, ctypes.byref(ns)) == sv.SV_EINVAL
    assert lib.sv_plan_wht(41, 1, sv.SV_C64, 1, 1, out, 4, ctypes.byref(ns)) == sv.SV_EINVAL
    gout = (sv.sv_gate_plan_step * 4)()
    for rows, why in (([(20, 0, 0)], "target"), ([(-1, 0, 0)], "target"), ([(3, 1 << 3, 0)], "control"),
                      ([(3, 1 << 20, 0)], "control"), ([(3, 0, 1)], "reserved")):
        g = gates_arr(rows)
        rc = lib.sv_plan_gates(20, 1, sv.SV_C64, g.ctypes.data, len(g), gout, 4, ctypes.byref(ns), None)
        assert rc == sv.SV_EINVAL, why
    assert lib.sv_plan_gates(20, 1, sv.SV_C64, None, 3, gout, 4, ctypes.byref(ns), None) == sv.SV_EINVAL
    assert lib.sv_plan_gates(20, 1, sv.SV_C64, None, 0, gout, 4, ctypes.byref(ns), None) == sv.SV_OK
    assert ns.value == 0
    assert lib.sv_nccl_unique_id(None, 128) == sv.SV_EINVAL
    buf = ctypes.create_string_buffer(64)
    assert lib.sv_nccl_unique_id(buf, 64) == sv.SV_EINVAL
    assert lib.sv_marked_from_seed(4, 2, 0, None) == sv.SV_EINVAL
    assert lib.sv_marked_from_seed(4, 0, 0, None) == sv.SV_OK


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [sv.SV_C64, sv.SV_C128])
def test_rejected_calls_leave_the_context_unchanged(dtype):
    n = 14
    with sv.sv_init(n, 3, dtype, sv.SV_INIT_GAUSSIAN) as c:
        cp = c.ptr
        assert lib.sv_iterate(cp, 1, 0) == sv.SV_ESTATE and "marked" in last()
        assert lib.sv_iterate_noisy(cp, 1, 0.01, 0, 0) == sv.SV_ESTATE
        assert lib.sv_iterate_decoherent(cp, 1, 0.0, 0.1, 0, 0, None) == sv.SV_ESTATE
        assert lib.sv_measure_marked_mass(cp, ctypes.byref(ctypes.c_double())) == sv.SV_ESTATE
        mk = np.array([5, 77, 4000], np.uint64)
        sv.sv_set_marked(c, mk)
        before = sv.sv_get_amplitudes(c)
        mass = sv.sv_measure_marked_mass(c)
        N = 1 << n
        bad_sets = ([np.array([3, 3], np.uint64), "strictly increasing"], [np.array([9, 2], np.uint64), "increasing"],
                    [np.array([N], np.uint64), ">= 2^n"])
        for arr, msg in bad_sets:
            assert lib.sv_set_marked(cp, arr.ctypes.data, len(arr)) == sv.SV_EINVAL and msg in last()
            assert lib.sv_apply_oracle(cp, arr.ctypes.data, len(arr)) == sv.SV_EINVAL
        assert lib.sv_set_marked(cp, None, 2) == sv.SV_EINVAL
        assert lib.sv_set_marked(cp, mk.ctypes.data, N + 1) == sv.SV_EINVAL
        calls = [
            lambda: lib.sv_reset(cp, 0, 7),
            lambda: lib.sv_diffuse(cp, 2),
            lambda: lib.sv_iterate(cp, -1, 0),
            lambda: lib.sv_iterate(cp, 1, -1),
            lambda: lib.sv_iterate_noisy(cp, -1, 0.0, 0, 0),
            lambda: lib.sv_iterate_noisy(cp, 1, -0.1, 0, 0),
            lambda: lib.sv_iterate_noisy(cp, 1, 10.0, 0, 0),
            lambda: lib.sv_iterate_noisy(cp, 1, float("nan"), 0, 0),
            lambda: lib.sv_iterate_decoherent(cp, 1, 0.0, 1.0, 0, 0, None),
            lambda: lib.sv_iterate_decoherent(cp, 1, 0.0, -0.5, 0, 0, None),
            lambda: lib.sv_iterate_decoherent(cp, 1, -1.0, 0.1, 0, 0, None),
            lambda: lib.sv_iterate_decoherent(cp, -2, 0.0, 0.1, 0, 0, None),
            lambda: lib.sv_probabilities(cp, None, N, 0),
            lambda: lib.sv_probabilities(cp, np.zeros(N - 1).ctypes.data, N - 1, 0),
            lambda: lib.sv_sample(cp, 4, 0, None, 0),
            lambda: lib.sv_measure_marked_mass(cp, None),
            lambda: lib.sv_get_amplitudes(cp, np.zeros(4, np.complex128).ctypes.data, N - 1, 2),
            lambda: lib.sv_get_amplitudes(cp, None, 0, 1),
            lambda: lib.sv_set_amplitudes(cp, np.zeros(4, np.complex128).ctypes.data, N, 1),
            lambda: lib.sv_set_amplitudes(cp, None, 0, 1),
            lambda: lib.sv_get_exchange(cp, None),
            lambda: lib.sv_profile_read(cp, sv.SV_K_COUNT, None, None),
            lambda: lib.sv_profile_read(cp, -1, None, None),
            lambda: lib.sv_apply_gates(cp, None, 2),
        ]
        for i, call in enumerate(calls):
            assert call() == sv.SV_EINVAL, i
            assert last(), i
        for rows in ([(n, 0, 0)], [(2, 1 << 2, 0)], [(2, 1 << n, 0)], [(2, 0, 5)], [(0, 0, 0), (n + 3, 0, 0)]):
            g = gates_arr(rows)
            assert lib.sv_apply_gates(cp, g.ctypes.data, len(g)) == sv.SV_EINVAL, rows
        assert lib.sv_set_exchange(cp, 1) == sv.SV_ESTATE  # one rank: no fused exchange
        assert lib.sv_set_exchange(cp, 0) == sv.SV_OK
        # nothing above touched the state or the marked set
        np.testing.assert_array_equal(sv.sv_get_amplitudes(c), before)
        assert sv.sv_measure_marked_mass(c) == mass
        # the degenerate-but-valid forms are no-ops
        assert lib.sv_get_amplitudes(cp, None, N, 0) == sv.SV_OK
        assert lib.sv_set_amplitudes(cp, None, 0, 0) == sv.SV_OK
        assert lib.sv_sample(cp, 0, 0, None, 0) == sv.SV_OK
        assert lib.sv_apply_gates(cp, None, 0) == sv.SV_OK
        assert lib.sv_iterate_noisy(cp, 0, 0.5, 0, 0) == sv.SV_OK
        assert lib.sv_iterate_decoherent(cp, 0, 0.5, 0.5, 0, 0, None) == sv.SV_OK
        np.testing.assert_array_equal(sv.sv_get_amplitudes(c), before)
