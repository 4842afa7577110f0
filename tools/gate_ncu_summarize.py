"""Summarise ncu --set full captures of gate tile passes (tools/gate_profile_run.py):
key metrics (ncu_summarize.KEYS + issue activity) and the executed-instruction
mix per warp-tile from the SASS source page.

    python tools/gate_ncu_summarize.py OUT.json NAME=REP.ncu-rep [NAME=REP ...]
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summarize import KEYS  # noqa: E402

EXTRA = ["smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum", "launch__grid_size"]


def raw(rep):
    rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                      capture_output=True, text=True).stdout)))
    hdr, data = rows[0], rows[2:]
    return [{k: r[hdr.index(k)] for k in KEYS + EXTRA if k in hdr} for r in data]


def mix(rep, launch):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(launch), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    op = collections.Counter()
    for r in rows[2:]:
        if r and r[0] == "Address":
            break  # one copy of the listing
        if len(r) != len(hdr) or not r[iE].isdigit():
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
        if m:
            op[m.group(2)] += int(r[iE])
    return op


def main():
    out = {"_note": "ncu --set full of gate_tile passes at n = 28 c64 (tools/gate_profile_run.py); "
                    "inst_mix = executed warp instructions per warp-tile by opcode (top 12)"}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        caps = raw(rep)
        for i, c in enumerate(caps):
            op = mix(rep, i)
            warps = int(c["launch__grid_size"].replace(",", "")) * 8
            c["inst_mix_per_warp_tile"] = {k: round(v / warps, 1) for k, v in op.most_common(12)}
            c["inst_per_warp_tile"] = round(sum(op.values()) / warps, 1)
        out[name] = caps
    json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
