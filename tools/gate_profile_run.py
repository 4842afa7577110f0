"""One gate circuit (n=28, c64) through the gate engine, for ncu captures of its tile passes:
    ncu --set full -k regex:gate_tile -s 5 -c 2 python tools/gate_profile_run.py [qft|u_layer|layered]
(the first sv_apply_gates call is the warm-up; -s skips its launches)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_9804039_b200 as sv  # noqa: E402
from tests import circuits as C  # noqa: E402

n = 28
which = sys.argv[1] if len(sys.argv) > 1 else "qft"
if which == "qft":
    g = C.qft_circuit(n)
elif which == "u_layer":
    g = C.circuit([C.record(q, C.random_unitary(np.random.default_rng(q))) for q in range(n)])
else:
    g = C.layered_circuit(n, 4, 1)
with sv.sv_init(n, 1, sv.SV_C64, sv.SV_INIT_GAUSSIAN) as c:
    steps, _ = sv.sv_plan_gates(n, 1, sv.SV_C64, g)
    print(which, "passes", len(steps))
    sv.sv_apply_gates(c, g)  # warm-up
    sv.sv_apply_gates(c, g)
    sv.sv_synchronize(c)
print("ok")
