#!/usr/bin/env python
"""Supertile-pass wait statistics (measurement build: build.py -DSV_SUPER_STATS=1 --out=PATH, SV_LIB=PATH).

    SV_LIB=/tmp/libsv_stats.so python tools/super_stats.py --n 28
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_9804039_b200 as sv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=28)
a = ap.parse_args()
st = (ctypes.c_ulonglong * 8)()
with sv.sv_init(a.n, 0, sv.SV_C64) as c:
    sv.sv_set_marked(c, [3])
    sv.sv_iterate(c, 1, sv.SV_DIFFUSE_WHT)
    sv.sv_synchronize(c)
    sv.lib.sv_debug_super_stats(st)
    sv.sv_iterate(c, 1, sv.SV_DIFFUSE_WHT)
    sv.sv_synchronize(c)
    sv.lib.sv_debug_super_stats(st)
items, waited, wait_cyc, _, item_cyc = st[0], st[1], st[2], st[3], st[4]
print(f"n={a.n} items={items} waited={waited} ({100.0 * waited / max(items, 1):.1f}%) "
      f"mean wait {wait_cyc / max(items, 1):.0f} cyc, mean item {item_cyc / max(items, 1):.0f} cyc")
