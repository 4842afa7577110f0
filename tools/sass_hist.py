#!/usr/bin/env python
"""SASS instruction histograms of the kernels the c4 / c3m benches launch
(evidence for DESIGN.md: packed FADD2 / FFMA2 butterflies, 128-bit global and
shared accesses, no local-memory spills, no tensor-core or TMA instructions on
this memory-bound path).  Host only: cuobjdump of the built objects.

    python tools/sass_hist.py > profiles/r2_sass_hist.json
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_quant_ph_9804039_b200", "build")

# (object, demangled-name regex, label): the c4 bench's four tile-pass kinds
# (plan of n = 32: contiguous pre-only, two-layout O-fused U=3 / post-only /
# pre-only, two-layout F0-fused U=4) and the mean kernels of c3m / c5m
KERNELS = [
    ("wht.cu.o", r"wht_tile_kernel<float2, 13, 5, true, false, 0, 0, false>", "contiguous pass (U=0, pre)"),
    ("wht.cu.o", r"wht_tile2_kernel<13, 5, true, true, 3, 0, false>", "O-fused strided pass (two-layout, U=3)"),
    ("wht.cu.o", r"wht_tile2_kernel<13, 5, true, true, 4, 0, false>", "F0-fused strided pass (two-layout, U=4)"),
    ("wht.cu.o", r"wht_tile_kernel<float2, 13, 5, true, true, 5, 0, false>", "fused strided pass (U=5, c3)"),
    ("mean.cu.o", r"mean_kernel<float2, true>", "fused flip + invert-about-mean (complex64)"),
    ("mean_resident.cu.o", r"mean_resident_kernel<double2>", "shared-memory-resident mean (A/B, SV_MEAN_RESIDENT=smem)"),
    ("mean_resident.cu.o", r"mean_resreg_kernel<double2, 16, 512>", "register-resident mean (c2)"),
    ("gates.cu.o", r"gate_tile_kernel_p<float2, 13, 5, false, false, true>", "gate interpreter, two-layout family"),
]
CLASSES = {
    "FADD2": r"^FADD2\b", "FFMA2": r"^FFMA2\b", "FMUL2": r"^FMUL2\b", "FADD": r"^FADD\b", "FFMA": r"^FFMA\b",
    "DADD": r"^DADD\b", "DFMA": r"^DFMA\b",
    "LDG.128": r"^LDG\.E\.(?:.*\.)?128\b", "LDG.64": r"^LDG\.E\.(?:.*\.)?64\b", "LDG(other)": r"^LDG\b",
    "STG.128": r"^STG\.E\.(?:.*\.)?128\b", "STG.64": r"^STG\.E\.(?:.*\.)?64\b", "STG(other)": r"^STG\b",
    "LDS.128": r"^LDS\.128\b", "LDS(other)": r"^LDS\b", "STS.128": r"^STS\.128\b", "STS(other)": r"^STS\b",
    "LDL": r"^LDL\b", "STL": r"^STL\b", "BAR": r"^BAR\b", "SHFL": r"^SHFL\b",
    "tensor (UTC*MMA/HMMA)": r"^(UTC\w*MMA|HMMA)\b", "TMA (UTMALDG/UTMASTG/UBLKCP)": r"^(UTMALDG|UTMASTG|UBLKCP)\b",
}


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
    funcs, cur, body = {}, None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                funcs[cur] = body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)(.*?);", line)
        if m and cur:
            body.append(m.group(1))
    if cur:
        funcs[cur] = body
    return funcs


def main():
    res = []
    cache = {}
    for obj, pat, label in KERNELS:
        if obj not in cache:
            f = functions(obj)
            cache[obj] = dict(zip(demangle(list(f)), f.values()))
        hit = [(n, b) for n, b in cache[obj].items() if re.search(re.escape(pat).replace("\\ ", " "), n.replace("(int)", "").replace("(bool)", ""))]
        if not hit:
            res.append({"kernel": label, "pattern": pat, "error": "not found"})
            continue
        name, body = hit[0]
        ops = collections.Counter(body)
        cls = {}
        for c, rx in CLASSES.items():
            cls[c] = 0
        for op, cnt in ops.items():
            for c, rx in CLASSES.items():
                if re.match(rx, op):
                    cls[c] += cnt
                    break
        res.append({"kernel": label, "symbol": name, "instructions": len(body), "classes": cls,
                    "top_opcodes": ops.most_common(12)})
    json.dump({"what": "static SASS instruction counts per kernel (cuobjdump -sass of the sm_100a objects)",
               "kernels": res}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
