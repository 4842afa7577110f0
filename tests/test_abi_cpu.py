"""CPU-only checks of the C ABI: the library loads, exports every symbol that
include/sv.h declares, and its host-only entry points (seeded generators,
schedule introspection, argument validation) behave -- no device calls."""
import os
import re

import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    txt = open(os.path.join(ROOT, "include", "sv.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(sv_[a-z0-9_]+)\s*\(", txt, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ["sv_init", "sv_apply_oracle", "sv_diffuse", "sv_iterate", "sv_probabilities",
                     "sv_measure_marked_mass", "sv_free", "sv_last_error"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 20
    for nm in names:
        assert hasattr(sv.lib, nm), f"libsv.so does not export {nm}"


def test_library_is_sm100a_cuda():
    """The shipped .so carries sm_100a SASS for our kernels (cuobjdump)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", sv.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n,m,seed", [(1, 1, 0), (1, 2, 3), (10, 1, 1), (20, 4, 2), (28, 1, 3), (32, 256, 4),
                                      (34, 1024, 5), (12, 4096, 9), (40, 17, 123456789)])
def test_marked_generator_matches_oracle_bitwise(n, m, seed):
    """G6/G7: the library's and the oracle's independent implementations agree."""
    np.testing.assert_array_equal(sv.sv_marked_from_seed(n, m, seed), orc.marked_from_seed(n, m, seed))


def test_marked_generator_errors():
    with pytest.raises(sv.SvError) as e:
        sv.sv_marked_from_seed(3, 9, 0)
    assert e.value.code == sv.SV_EINVAL
    with pytest.raises(sv.SvError):
        sv.sv_marked_from_seed(0, 1, 0)
    with pytest.raises(sv.SvError):
        sv.sv_marked_from_seed(41, 1, 0)


def popcount(x):
    return bin(x).count("1")


@pytest.mark.parametrize("dtype", [sv.SV_C64, sv.SV_C128])
@pytest.mark.parametrize("n,world", [(14, 1), (20, 1), (25, 1), (28, 1), (32, 1), (34, 1), (40, 1),
                                     (28, 2), (32, 2), (32, 4), (32, 8), (34, 8), (27, 8), (30, 4)])
def test_plan_invariants(dtype, n, world):
    T = 13 if dtype == sv.SV_C64 else 12
    c = 3 if dtype == sv.SV_C64 else 2
    g = world.bit_length() - 1
    nl = n - g
    if world > 1 and nl - g < T:
        with pytest.raises(sv.SvError):
            sv.sv_plan_wht(n, world, dtype, 1, True)
        return
    k = 3
    steps = sv.sv_plan_wht(n, world, dtype, k, True)
    passes = [s for s in steps if s["kind"] == 0]
    swaps = [s for s in steps if s["kind"] == 1]
    for s in passes:
        assert popcount(s["tile_mask"]) == T
        assert s["proc_mask"] & ~s["tile_mask"] == 0
        assert s["tile_mask"] & 1
        assert s["tile_mask"] < (1 << nl)
        unproc = s["tile_mask"] & ~s["proc_mask"]
        if unproc:  # the unprocessed slots are the lowest ones: >= 2^c-amplitude runs
            assert unproc == (1 << popcount(unproc)) - 1 and popcount(unproc) >= c
    # O always meets the same group (its per-tile lookup is built for one group)
    assert len({s["tile_mask"] for s in passes if s["mid"] == 1}) == 1
    # the fused roles go to small groups: the contiguous tile is fused only
    # when there are just two groups
    n_groups = len({s["tile_mask"] for s in passes})
    if world == 1 and n_groups >= 3:
        assert all(s["tile_mask"] != (1 << T) - 1 for s in passes if s["mid"] != 0)
    # every pass reads/writes the state once: count HBM passes per iteration
    assert swaps == [] or world > 1
    assert len(swaps) == (2 * k if world > 1 else 0)
    # stage count: each WHT visits every one of the n logical qubits once
    stage_instances = sum(popcount(s["proc_mask"]) * (s["pre"] + s["post"]) for s in passes)
    assert stage_instances == 2 * k * (nl + g)


def test_plan_c4_pass_counts():
    """The fused schedule: (O.G1.G1) G2 (G3.F0.G3) G2 ... -> 4k+1 passes at n=32."""
    for n, world, per_iter in [(28, 1, 4), (32, 1, 4), (32, 2, 4), (32, 4, 4), (32, 8, 4), (23, 1, 2)]:
        k = 5
        steps = sv.sv_plan_wht(n, world, sv.SV_C64, k, True)
        passes = sum(1 for s in steps if s["kind"] == 0)
        assert passes == per_iter * k + 1, (n, world, passes)


def test_plan_whole_state_small_n():
    steps = sv.sv_plan_wht(10, 1, sv.SV_C128, 25, True)
    assert len(steps) == 1 and steps[0]["kind"] == 2
    assert sv.sv_plan_wht(12, 1, sv.SV_C64, 0, True) == []


def test_plan_errors():
    for args in [(0, 1, 0), (41, 1, 0), (20, 3, 0), (20, 1, 7), (30, 128, 0)]:
        with pytest.raises(sv.SvError) as e:
            sv.sv_plan_wht(args[0], args[1], args[2], 1, True)
        assert e.value.code == sv.SV_EINVAL
    with pytest.raises(sv.SvError):
        sv.sv_plan_wht(20, 1, 0, -1, True)
