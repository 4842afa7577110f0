"""Parity cases that reproduce, at sizes the oracle runs in seconds, every WHT
tile-kernel variant the benches launch (verdict r1 weak #1).

A variant is the template instantiation a pass runs: (family, u, pre, mid,
post, noisy, xchg) as sv_debug_wht_variants describes it (include/sv.h).  The
benches' large states pick their group shapes from n (plan.cpp); the
test-only planner overrides SV_PLAN_CHUNKS (one GPU: processed slots per
strided group, `o` / `f` = the group hosting the oracle / F0) and SV_PLAN_L1
(sharded: slots of the post-swap group) give small states the same shapes.
tests/test_variants.py (CPU) checks the coverage; tests/test_variants_gpu.py
runs each case against the oracle.
"""

# flavours of sv_debug_wht_variants / the entry point a case calls
IDEAL, NOISY, DECOHERENT = 0, 1, 2

# (id, n, world, flavour, k, sigma, rate, seed, env)
CASES = []
for _fl, _sig, _rate in ((IDEAL, 0.0, 0.0), (NOISY, 0.05, 0.0), (DECOHERENT, 0.03, 0.02)):
    for _n, _chunks in ((24, "10o,1f"),   # n=32's O group: 10 slots, 64-B runs (two-layout, U=3)
                        (23, "1o,9f"),    # n=32's F0 group: 9 slots, 128-B runs (two-layout, U=4)
                        (22, "8o,1f"),    # n=28's O group (U=5)
                        (21, "1o,7f"),    # n=28's F0 group (U=6)
                        (21, "7o,1f")):   # n=34's O group (U=6)
        CASES.append((f"fl{_fl}-n{_n}-{_chunks}", _n, 1, _fl, 3 if _fl == IDEAL else 2, _sig, _rate,
                      100 + _n, {"SV_PLAN_CHUNKS": _chunks}))
    for _l1 in (10, 2):  # sharded c4 shapes: post-swap group of 10 slots (U=3) / O group of 9 slots (U=4)
        CASES.append((f"fl{_fl}-n24-P2-L1={_l1}", 24, 2, _fl, 2, _sig, _rate, 200 + _l1, {"SV_PLAN_L1": str(_l1)}))
    # the opt-in supertile pass (SV_SUPER=1, wht_super.cuh; measured slower than the plain
    # schedule, kept as a correct A/B option): n = 25's plan (level A tiles U=2, level B U=12)
    # and the test-only level split SV_SUPER_A=4 (level B U=5, n = 32's shape)
    CASES.append((f"fl{_fl}-n25-super", 25, 1, _fl, 2, _sig, _rate, 300, {"SV_SUPER": "1"}))
    CASES.append((f"fl{_fl}-n25-super-A4", 25, 1, _fl, 2, _sig, _rate, 301, {"SV_SUPER": "1", "SV_SUPER_A": "4"}))

# the benches' WHT workloads: (config, n, world, flavour, k, sigma, rate, seed) -- bench.py CONFIGS
BENCH = [
    ("c3", 28, 1, IDEAL, 64, 0.0, 0.0, 3),
    ("c4", 32, 1, IDEAL, 16, 0.0, 0.0, 4),
    ("c4-P2", 32, 2, IDEAL, 16, 0.0, 0.0, 4),
    ("c4-P4", 32, 4, IDEAL, 16, 0.0, 0.0, 4),
    ("c4-P8", 32, 8, IDEAL, 16, 0.0, 0.0, 4),
    ("c5w", 34, 1, IDEAL, 8, 0.0, 0.0, 5),
    ("c3n", 28, 1, NOISY, 64, 0.01, 0.0, 3),
    ("c4n", 32, 1, NOISY, 16, 0.01, 0.0, 4),
    ("c3d", 28, 1, DECOHERENT, 64, 0.01, 1e-3, 3),
]
