"""Randomised soak of the WHT tile passes against the oracle on one B200:
random strided-group splits (the test-only SV_PLAN_CHUNKS override, any
split is a valid schedule, G18), random marked sets, Gaussian start states,
ideal / angle-error / decoherent flavours, both dtypes:
python tools/soak_wht_gpu.py [cases] [seed].  Prints one line per failure and
a summary; exit code 1 on any failure.  Test infrastructure (imports oracle/)."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_quant_ph_9804039_b200 as sv  # noqa: E402
from oracle import oracle as orc  # noqa: E402

TOL = {sv.SV_C128: 1e-12, sv.SV_C64: 1e-5}


def random_split(rng, nstrided):
    """1-3 groups adding up to nstrided, O and F0 tagged on different groups (or untagged)."""
    ng = int(rng.integers(1, min(3, nstrided) + 1))
    cuts = sorted(rng.choice(np.arange(1, nstrided), size=ng - 1, replace=False).tolist()) if ng > 1 else []
    lens = [b - a for a, b in zip([0] + cuts, cuts + [nstrided])]
    tags = [""] * ng
    if ng > 1 and rng.random() < 0.7:
        o, f = rng.choice(ng, size=2, replace=False)
        tags[int(o)], tags[int(f)] = "o", "f"
    return ",".join(f"{v}{t}" for v, t in zip(lens, tags))


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    fails = skipped = 0
    worst = {}
    for i in range(cases):
        dt = sv.SV_C64 if rng.random() < 0.7 else sv.SV_C128
        fl = ["ideal", "noisy", "decoherent"][int(rng.integers(0, 3))]
        n = int(rng.integers(17, 24 if fl == "ideal" else 23))
        tile = 13 if dt == sv.SV_C64 else 12  # sv_internal.h tile_bits
        split = random_split(rng, n - tile)
        k = int(rng.integers(1, 4))
        M = int(rng.choice([1, 2, 37, 256]))
        seed = int(rng.integers(1, 1 << 30))
        sigma, rate = float(rng.choice([0.0, 0.01, 0.2])), float(rng.choice([1e-3, 0.05]))
        N = 1 << n
        a = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        a /= np.linalg.norm(a)
        a = a.astype(sv.NP_DTYPE[dt]).astype(np.complex128)
        marked = orc.marked_from_seed(n, M, seed)
        tag = f"case {i}: n={n} {'c64' if dt == sv.SV_C64 else 'c128'} {fl} k={k} M={M} split={split}"
        os.environ["SV_PLAN_CHUNKS"] = split
        try:
            try:  # host-only: a split the planner rejects (a group larger than the tile's processed slots)
                sv.sv_plan_wht(n, 1, dt, k, True)
            except sv.SvError as e:
                skipped += 1
                print(f"skip {tag}: {e}", flush=True)
                continue
            with sv.sv_init(n, 0, dt, sv.SV_INIT_ZERO_STATE) as c:
                sv.sv_set_amplitudes(c, a)
                sv.sv_set_marked(c, marked)
                if fl == "ideal":
                    sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
                    ref = orc.iterate(a.copy(), marked, k, orc.WHT)
                elif fl == "noisy":
                    sv.sv_iterate_noisy(c, k, sigma, seed, 0)
                    ref = orc.iterate_noisy(a.copy(), marked, k, sigma, seed, 0)
                else:
                    sv.sv_iterate_decoherent(c, k, sigma, rate, seed, 0)
                    ref, _ = orc.iterate_decoherent(a.copy(), marked, k, sigma, rate, seed, 0)
                got = np.asarray(sv.sv_get_amplitudes(c), dtype=np.complex128)
        finally:
            os.environ.pop("SV_PLAN_CHUNKS", None)
        err, scale = float(np.max(np.abs(got - ref))), float(np.max(np.abs(ref)))
        bound = TOL[dt]
        if dt == sv.SV_C64:  # tests/test_parity_gpu.py rel64: 2 n 2^-24 sqrt(k) of the amplitude scale
            bound = min(bound, 2.0 * n * 2.0 ** -24 * math.sqrt(k) * scale)
        key = f"{fl}/{'c64' if dt == sv.SV_C64 else 'c128'}"
        worst[key] = max(worst.get(key, 0.0), err / scale)
        if not err <= bound:
            fails += 1
            print(f"FAIL {tag}: max-abs {err:.3e} > {bound:.3e}", flush=True)
    print({k: f"{v:.2e}" for k, v in sorted(worst.items())}, f"(max-abs / max|ref|) {cases} cases, {skipped} skipped, {fails} failures")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
