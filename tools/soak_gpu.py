"""Randomised soak of the round-2 kernels against the oracle on one B200
(register-resident mean diffusion at every NPT shape, two-layout gate passes):
python tools/soak_gpu.py [cases] [seed].  Prints one line per failure and a
summary; exit code 1 on any failure.  Test infrastructure (imports oracle/)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_quant_ph_9804039_b200 as sv  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from tests import circuits as C  # noqa: E402

TOL = {sv.SV_C128: 1e-12, sv.SV_C64: 1e-5}


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    fails = 0
    worst = {}
    for i in range(cases):
        dt = sv.SV_C64 if rng.random() < 0.5 else sv.SV_C128
        kind = "gates" if rng.random() < 0.3 else "mean"
        n = int(rng.integers(14, 22 if dt == sv.SV_C64 else 21)) if kind == "mean" else int(rng.integers(14, 21))
        N = 1 << n
        a0 = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        a0 /= np.linalg.norm(a0)
        a0 = a0.astype(sv.NP_DTYPE[dt]).astype(np.complex128)
        with sv.sv_init(n, 0, dt, sv.SV_INIT_ZERO_STATE) as c:
            sv.sv_set_amplitudes(c, a0)
            if kind == "mean":
                m = int(rng.choice([0, 1, 4, 64, 1000, N // 3]))
                k = int(rng.integers(1, 40))
                marked = orc.marked_from_seed(n, m, int(rng.integers(1 << 30))) if m else np.zeros(0, np.uint64)
                sv.sv_set_marked(c, marked)
                sv.sv_iterate(c, k, sv.SV_DIFFUSE_MEAN)
                ref = orc.iterate(a0.copy(), marked, k, orc.MEAN)
                tol = TOL[dt] * (1 + k / 8)
                what = f"mean n={n} m={m} k={k}"
            else:
                g = C.random_circuit(n, int(rng.integers(20, 200)), int(rng.integers(1 << 30)), max_controls=2)
                sv.sv_apply_gates(c, g)
                ref = orc.apply_gates(a0.copy(), g)
                tol = TOL[dt]
                what = f"gates n={n} G={len(g)}"
            got = sv.sv_get_amplitudes(c).astype(np.complex128)
        err = float(np.max(np.abs(got - ref)))
        key = (kind, "c64" if dt == sv.SV_C64 else "c128")
        worst[key] = max(worst.get(key, 0.0), err)
        if not err <= tol:
            fails += 1
            print(f"FAIL {what} {key[1]}: max-abs {err:.3e} > {tol:.1e}", flush=True)
    print({f"{k[0]}/{k[1]}": f"{v:.2e}" for k, v in worst.items()}, f"{cases} cases, {fails} failures", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
