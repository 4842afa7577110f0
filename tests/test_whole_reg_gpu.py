"""Every warp split of the register-resident one-CTA kernel (wht.cu
whole_reg_kernel<E, LOGR, LOGW, GEN>: n = LOGR + 5 + LOGW, transforms
alternating between layouts A and B) against the oracle: ideal WHT and mean
iterations, angle-error (GEN) and decoherent iterations.  SV_WHOLE_W is read
once per process, so each split runs in its own subprocess, which writes its
input state and the device results; the oracle runs here."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests.test_parity_gpu import TOL, assert_close

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# instantiated (dtype, n) per LOGW (wht.cu launch_whole_state)
SPLITS = {
    2: [("c64", n) for n in (9, 10, 11, 12, 13)] + [("c128", n) for n in (9, 10, 11)],
    3: [("c64", n) for n in (10, 11, 12, 13)] + [("c128", n) for n in (10, 11, 12)],
    4: [("c64", n) for n in (11, 12, 13)] + [("c128", n) for n in (10, 11, 12)],
    5: [("c64", 10), ("c128", 10)],
}
DTS = {"c64": sv.SV_C64, "c128": sv.SV_C128}
K, M, SIGMA, RATE = 3, 3, 0.07, 0.02

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_quant_ph_9804039_b200 as sv
from tests.test_parity_gpu import rand_state
from oracle import oracle as orc
cases = json.loads(sys.argv[2]); out = {}
for name, n in cases:
    dt = {"c64": sv.SV_C64, "c128": sv.SV_C128}[name]
    a = rand_state(n, dt)
    marked = orc.marked_from_seed(n, %(M)d, n)
    res = {"a": [a.real.tolist(), a.imag.tolist()]}
    for mode in ("wht", "mean", "noisy", "deco"):
        c = sv.sv_init(n, 0, dt)
        sv.sv_set_amplitudes(c, a)
        sv.sv_set_marked(c, marked)
        if mode == "wht": sv.sv_iterate(c, %(K)d, sv.SV_DIFFUSE_WHT)
        elif mode == "mean": sv.sv_iterate(c, %(K)d, sv.SV_DIFFUSE_MEAN)
        elif mode == "noisy": sv.sv_iterate_noisy(c, %(K)d, %(SIGMA)r, 11 + n, 2)
        else: res["surv"] = sv.sv_iterate_decoherent(c, %(K)d, %(SIGMA)r, %(RATE)r, 5 + n, 1).tolist()
        g = sv.sv_get_amplitudes(c).astype(np.complex128)
        res[mode] = [g.real.tolist(), g.imag.tolist()]
        sv.sv_free(c)
    out[name + str(n)] = res
print(json.dumps(out))
""" % dict(M=M, K=K, SIGMA=SIGMA, RATE=RATE)


@pytest.mark.parametrize("logw", sorted(SPLITS))
def test_whole_reg_split_matches_oracle(logw):
    env = dict(os.environ, SV_WHOLE_W=str(logw))
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, json.dumps(SPLITS[logw])], env=env, capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    for name, n in SPLITS[logw]:
        dt = DTS[name]
        marked = orc.marked_from_seed(n, M, n)
        res = got[name + str(n)]
        dev = {k: np.array(v[0]) + 1j * np.array(v[1]) for k, v in res.items() if k != "surv"}
        a = dev["a"]  # the child's (dtype-rounded) input state
        what = f"W={logw} {name} n={n}"
        assert_close(dev["wht"], orc.iterate(a.copy(), marked, K, orc.WHT), dt, what + " wht", n=n, k=K)
        assert_close(dev["mean"], orc.iterate(a.copy(), marked, K, orc.MEAN), dt, what + " mean", n=n, k=K)
        assert_close(dev["noisy"], orc.iterate_noisy(a.copy(), marked, K, SIGMA, 11 + n, 2), dt, what + " noisy",
                     n=n, k=K)
        ref, surv = orc.iterate_decoherent(a.copy(), marked, K, SIGMA, RATE, 5 + n, 1)
        assert_close(dev["deco"], ref, dt, what + " decoherent", n=n, k=K)
        assert np.max(np.abs(np.array(res["surv"]) - surv)) <= 100 * TOL[dt]
