"""One-CTA WHT kernel timing (n <= T): device microseconds per 25 iterations."""
import sys, time
sys.path.insert(0, '.')
import paper_quant_ph_9804039_b200 as sv
for n, dt in ((9, sv.SV_C128), (10, sv.SV_C128), (11, sv.SV_C128), (12, sv.SV_C128), (10, sv.SV_C64), (11, sv.SV_C64),
              (12, sv.SV_C64), (13, sv.SV_C64)):
    with sv.sv_init(n, 1, dt) as c:
        sv.sv_set_marked(c, sv.sv_marked_from_seed(n, 1, 1))
        sv.sv_iterate(c, 25)
        sv.sv_synchronize(c)
        sv.sv_profile(c, True)
        for _ in range(5):
            sv.sv_iterate(c, 25)
        l, ms = sv.sv_profile_read(c, sv.SV_K_WHT_WHOLE)
        print(n, dt, l, ms / l * 1e3, "us per 25 iterations")
