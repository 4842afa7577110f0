#!/usr/bin/env python
"""Device time of sv_sample (NEXT-3) on a c4-sized state.

    python tools/sample_bench.py [--n 32] [--shots 1048576] [--reps 3]

Prints one JSON object: the chunk-prefix launch (an HBM read of the state:
GB/s against the measured copy peak) and the draw launch (shots/s), from the
CUDA events libsv records around each launch.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_quant_ph_9804039_b200 as sv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--shots", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    ctx = sv.sv_init(a.n, 4, sv.SV_C64, sv.SV_INIT_UNIFORM)
    sv.sv_set_marked(ctx, sv.sv_marked_from_seed(a.n, 256, 4))
    sv.sv_iterate(ctx, 16, sv.SV_DIFFUSE_WHT)
    sv.sv_sample(ctx, a.shots, 0)  # warm-up (allocations)
    sv.sv_profile(ctx, True)
    for r in range(a.reps):
        out = sv.sv_sample(ctx, a.shots, r)
    tl = sv.sv_profile_timeline(ctx)
    prefix = [ms for i, (k, ms) in enumerate(tl) if i % 2 == 0]
    draw = [ms for i, (k, ms) in enumerate(tl) if i % 2 == 1]
    state_bytes = (1 << a.n) * 8
    pm = sum(prefix) / len(prefix)
    dm = sum(draw) / len(draw)
    marked = set(sv.sv_marked_from_seed(a.n, 256, 4).tolist())
    hit = sum(1 for v in out.tolist() if v in marked) / a.shots
    print(json.dumps({"n": a.n, "shots": a.shots, "prefix_ms": pm, "prefix_GBps": state_bytes / (pm / 1e3) / 1e9,
                      "draw_ms": dm, "shots_per_s": a.shots / (dm / 1e3), "marked_hit_fraction": hit}))


if __name__ == "__main__":
    main()
