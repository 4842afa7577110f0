#!/usr/bin/env python
"""Per-pass device time of sv_iterate(k, WHT), attributed to the plan steps.

    python tools/pass_breakdown.py --n 32 --k 2 [--m 256] [--dtype c64]

Prints one JSON object: for every distinct pass type (group tile/proc masks,
pre/mid/post) its launch count, mean ms and achieved GB/s (2 x state bytes
per pass), from CUDA events the library records around each launch.
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_quant_ph_9804039_b200 as sv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--m", type=int, default=256)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--world", type=int, default=1, help="emulated shards on one GPU")
    ap.add_argument("--sigma", type=float, default=0.0, help="> 0: sv_iterate_noisy (NEXT-1 angle errors), same schedule")
    a = ap.parse_args()
    dt = sv.SV_C64 if a.dtype == "c64" else sv.SV_C128
    eb = 8 if dt == sv.SV_C64 else 16
    ctx = sv.sv_init(a.n, 0, dt, sv.SV_INIT_UNIFORM, world=a.world)
    sv.sv_set_marked(ctx, sv.sv_marked_from_seed(a.n, a.m, 1))
    def run(k):
        if a.sigma > 0:
            sv.sv_iterate_noisy(ctx, k, a.sigma, 7, 0)
        else:
            sv.sv_iterate(ctx, k, sv.SV_DIFFUSE_WHT)
    run(1)  # warm-up
    sv.sv_profile(ctx, True)
    run(a.k)
    tl = sv.sv_profile_timeline(ctx)
    plan = sv.sv_plan_wht(a.n, a.world, dt, a.k, True)
    agg = collections.OrderedDict()
    it = iter(tl)
    fused = a.world > 1 and sv.sv_get_exchange(ctx)
    for st in plan:
        if st["kind"] == 1 and fused:
            continue  # emulated fused exchange: the swap is inside the preceding pass
        kind, ms = next(it)
        if st["kind"] == 0:
            key = "tile=%#x proc=%#x pre=%d mid=%d post=%d" % (st["tile_mask"], st["proc_mask"], st["pre"], st["mid"],
                                                             st["post"])
        else:
            key = "kind=%d" % st["kind"]
        agg.setdefault(key, []).append(ms)
    bytes_pass = 2 * (1 << a.n) * eb
    out = {k: {"launches": len(v), "mean_ms": sum(v) / len(v), "GBps": bytes_pass / (sum(v) / len(v) / 1e3) / 1e9}
           for k, v in agg.items()}
    print(json.dumps({"n": a.n, "k": a.k, "world": a.world, "sigma": a.sigma, "passes": out, "total_ms": sum(ms for _, ms in tl)},
                     indent=1))


if __name__ == "__main__":
    main()
