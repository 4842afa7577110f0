"""Resident mean kernels (mean_resident.cu): device microseconds per iteration
vs state size.  At n = 14 a block holds ~110 amplitudes, so the time is the
per-iteration reduction + grid barrier alone: the latency floor of the design.
The kernel variant comes from the environment (SV_MEAN_RESIDENT=smem: the
shared-memory kernel; SV_RESREG_G / SV_RESREG_NEG / SV_RESREG_NT512: A/B
variants of the register-resident one), read once per process.

python tools/mean_resident_scan.py [k] [n,dtype ...]     e.g. 402 14,c128 20,c128
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_9804039_b200 as sv  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 402
cases = [(int(a.split(",")[0]), a.split(",")[1]) for a in sys.argv[2:]] or \
    [(n, "c128") for n in range(14, 21)] + [(n, "c64") for n in range(14, 22)]
variant = {e: os.environ[e] for e in ("SV_MEAN_RESIDENT", "SV_RESREG_G", "SV_RESREG_NEG", "SV_RESREG_NT512")
           if e in os.environ}
for n, dts in cases:
    dt = sv.SV_C128 if dts == "c128" else sv.SV_C64
    with sv.sv_init(n, 1, dt) as c:
        sv.sv_set_marked(c, sv.sv_marked_from_seed(n, 4, 1))
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_MEAN)
        sv.sv_synchronize(c)
        sv.sv_profile(c, True)
        for _ in range(5):
            sv.sv_iterate(c, k, sv.SV_DIFFUSE_MEAN)
        launches, ms = sv.sv_profile_read(c, sv.SV_K_MEAN)
        print(json.dumps({"variant": variant, "dtype": dts, "n": n, "launches": launches,
                          "us_per_iteration": round(ms / launches / k * 1e3, 3)}), flush=True)
