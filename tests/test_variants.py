"""Every WHT tile-kernel variant a bench launches is run by an element-wise
oracle parity case (tests/variant_cases.py, executed by
tests/test_variants_gpu.py).  Host only: sv_debug_wht_variants describes the
launches with the library's own schedule code, no device needed."""
import os

import pytest

import paper_quant_ph_9804039_b200 as sv
from tests.variant_cases import BENCH, CASES

FIELDS = ("family", "u", "pre", "mid", "post", "noisy", "xchg")


def variants(n, world, flavour, k, sigma, rate, seed, env=None):
    old = {key: os.environ.get(key) for key in (env or {})}
    try:
        os.environ.update(env or {})
        return set(sv.sv_debug_wht_variants(n, world, sv.SV_C64, flavour, k, sigma, rate, seed, True))
    finally:
        for key, v in old.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v


def covered():
    out = {}
    for cid, n, world, fl, k, sig, rate, seed, env in CASES:
        for v in variants(n, world, fl, k, sig, rate, seed, env):
            out.setdefault(v, cid)
    return out


def test_bench_table_matches_bench_py():
    import bench

    for name, n, world, fl, k, sig, rate, seed in BENCH:
        cfg = bench.CONFIGS[name.split("-")[0]]
        assert (cfg[0], cfg[3], cfg[5]) == (n, k, seed), name
        assert cfg[4] == {0: "wht", 1: "wht-noisy", 2: "wht-decoherent"}[fl], name


@pytest.mark.parametrize("bench_cfg", BENCH, ids=[b[0] for b in BENCH])
def test_bench_variants_are_parity_tested(bench_cfg):
    name, n, world, fl, k, sig, rate, seed = bench_cfg
    have = covered()
    launched = variants(n, world, fl, k, sig, rate, seed)
    missing = [dict(zip(FIELDS, v)) for v in sorted(launched) if v not in have]
    assert not missing, f"{name}: variants without a parity case: {missing}"


def test_overrides_change_the_shape_and_reject_bad_input():
    # SV_PLAN_CHUNKS reproduces n=32's O-group shape at n=24 ...
    got = variants(24, 1, 0, 3, 0, 0, 0, {"SV_PLAN_CHUNKS": "10o,1f"})
    assert (2, 3, 1, 1, 1, 0, 0) in got and (1, 12, 1, 2, 1, 0, 0) in got
    # ... and the default plan at n=24 does not have it
    assert (2, 3, 1, 1, 1, 0, 0) not in variants(24, 1, 0, 3, 0, 0, 0)
    for bad in ("10o,2f", "11,0", "5o,6o", "x", "10o,,1f", "3o,8o"):
        os.environ["SV_PLAN_CHUNKS"] = bad
        try:
            with pytest.raises(sv.SvError):
                sv.sv_debug_wht_variants(24, 1, sv.SV_C64, 0, 1)
        finally:
            os.environ.pop("SV_PLAN_CHUNKS")
    os.environ["SV_PLAN_L1"] = "11"
    try:
        with pytest.raises(sv.SvError):
            sv.sv_debug_wht_variants(24, 2, sv.SV_C64, 0, 1)
    finally:
        os.environ.pop("SV_PLAN_L1")


def test_design_table():
    """The DESIGN.md variant table (regenerated here; printed with -s)."""
    have = covered()
    rows = []
    for name, n, world, fl, k, sig, rate, seed in BENCH:
        for v in sorted(variants(n, world, fl, k, sig, rate, seed)):
            rows.append((name, v, have[v]))
    for name, v, cid in rows:
        print(f"| {name} | {', '.join(f'{f}={x}' for f, x in zip(FIELDS, v))} | {cid} |")
    assert rows
