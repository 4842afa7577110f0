"""Summarise ncu outputs of tools/measure_round.sh into profiles/ (run here, no GPU).

python tools/ncu_summarize.py gpurun_out/r1b profiles r1

Writes <prefix>_c4_ncu_launch_summary.txt (per-kernel launch counts, mean /
total device time and share of the step from the gpu__time_duration launch
list), <prefix>_c4_ncu_full_wht_tile.json (key metrics of each fully captured
tile-pass launch) and updates ncu_traffic.json (mean DRAM read + write bytes
per WHT tile launch, read by bench.py as roofline.traffic).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "idc__requests.sum"]


def launch_summary(path: str, cmd: str) -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] not in ("ID",) and r[0].isdigit()]
    agg = collections.OrderedDict()
    for r in rows:
        name, ns = r[4], float(r[-1].replace(",", ""))
        a = agg.setdefault(name.split("(")[0].strip(), [0, 0.0])
        a[0] += 1
        a[1] += ns / 1e6
    tot = sum(v[1] for v in agg.values())
    out = [f"# ncu launch list of `{cmd}` (c4: n=32 c64, 16 WHT iterations per step)",
           "# gpu__time_duration.sum, --clock-control none, cold-cache serialised launches: compare SHARES, not absolutes",
           "# kernel, launches, mean_ms, total_ms, share"]
    for k, (n, ms) in agg.items():
        out.append(f"{k}, {n}, {ms / n:.3f}, {ms:.2f}, {ms / tot:.4f}")
    return "\n".join(out) + "\n"


def full_capture(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    return [{k: r[hdr.index(k)] for k in KEYS if k in hdr} for r in data]


def main():
    src, dst, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
    cmd = "python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
    open(os.path.join(dst, f"{prefix}_c4_ncu_launch_summary.txt"), "w").write(
        launch_summary(os.path.join(src, "launches.csv"), cmd))
    caps = full_capture(os.path.join(src, "c4_full.ncu-rep"))
    json.dump(caps, open(os.path.join(dst, f"{prefix}_c4_ncu_full_wht_tile.json"), "w"), indent=1)
    tr = [float(c["dram__bytes_read.sum"]) + float(c["dram__bytes_write.sum"]) for c in caps]
    # ncu reports these in GB (1e9 B) for this metric set
    per_launch = sum(tr) / len(tr) * 1e9
    p = os.path.join(dst, "ncu_traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per wht_tile launch (bytes), mean of the launches in "
                  f"profiles/{prefix}_c4_ncu_full_wht_tile.json (ncu --set full, bench.py c4, P=1); "
                  "algorithmic = 2 x 2^32 x 8 B = 6.872e10")
    d["c4_P1"] = per_launch
    json.dump(d, open(p, "w"), indent=1)
    print(open(os.path.join(dst, f"{prefix}_c4_ncu_launch_summary.txt")).read())
    for c in caps:
        print(c["Kernel Name"][:70], c["gpu__time_duration.sum"], c["dram__bytes_read.sum"], c["dram__bytes_write.sum"],
              c.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"))


if __name__ == "__main__":
    main()
