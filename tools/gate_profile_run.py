"""One QFT (n=28, c64) through the gate engine, for ncu captures of its tile passes:
    ncu --set full -k regex:gate_tile -s 5 -c 2 python tools/gate_profile_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_9804039_b200 as sv  # noqa: E402
from tests import circuits as C  # noqa: E402

n = 28
g = C.qft_circuit(n)
with sv.sv_init(n, 1, sv.SV_C64, sv.SV_INIT_GAUSSIAN) as c:
    sv.sv_apply_gates(c, g)  # warm-up: launches 0-4
    sv.sv_apply_gates(c, g)
    sv.sv_synchronize(c)
print("ok")
