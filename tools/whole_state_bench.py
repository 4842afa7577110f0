"""One-CTA WHT kernel timing (n <= T): device microseconds per 25 iterations.

python tools/whole_state_bench.py            # the default warp split per size
SV_WHOLE_W=3 python tools/whole_state_bench.py   # force 2^3 warps where instantiated
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_9804039_b200 as sv  # noqa: E402

for n, dt in ((9, sv.SV_C128), (10, sv.SV_C128), (11, sv.SV_C128), (12, sv.SV_C128), (9, sv.SV_C64), (10, sv.SV_C64),
              (11, sv.SV_C64), (12, sv.SV_C64), (13, sv.SV_C64)):
    with sv.sv_init(n, 1, dt) as c:
        sv.sv_set_marked(c, sv.sv_marked_from_seed(n, 1, 1))
        sv.sv_iterate(c, 25)
        sv.sv_synchronize(c)
        sv.sv_profile(c, True)
        for _ in range(5):
            sv.sv_iterate(c, 25)
        l, ms = sv.sv_profile_read(c, sv.SV_K_WHT_WHOLE)
        print(n, "c128" if dt == sv.SV_C128 else "c64", "W=" + os.environ.get("SV_WHOLE_W", "default"), l,
              round(ms / l * 1e3, 2), "us per 25 iterations", flush=True)
