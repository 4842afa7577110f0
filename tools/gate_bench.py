"""Measure the NEXT-4 gate engine (sv_apply_gates) on one B200.

python tools/gate_bench.py [--n 30] [--reps 3] [--out gpurun_out/gate_bench.json]

Workloads (complex64, seeded; tests/circuits.py): a layer of H on every qubit
x4, the textbook QFT, hardware-efficient layers (random 1-qubit unitaries +
CZ chain) x4, 300 random gates with <= 2 controls, 300 structured gates.
Per workload: plan (passes, swaps), device time (CUDA events on the
context's stream, sv_profile), per-pass GB/s = 2 x state bytes / pass time
(one HBM read + write per pass), gate-amplitude-updates/s = 2^n x G / t.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_quant_ph_9804039_b200 as sv  # noqa: E402
from tests import circuits as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "gate_bench.json"))
    args = ap.parse_args()
    n = args.n
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    work = {
        "u_layer": C.circuit([C.record(q, C.random_unitary(np.random.default_rng(q))) for q in range(n)]),
        "h_layers_x4": C.circuit([C.record(q, C.H) for q in range(n)] * 4),  # H^4 fuses to an exact diagonal
        "qft": C.qft_circuit(n),
        "layered_x4": C.layered_circuit(n, 4, 1),
        "random_300": C.random_circuit(n, 300, 2, max_controls=2),
        "structured_300": C.structured_circuit(n, 300, 3, max_controls=2),
    }
    S = (1 << n) * 8
    res = {"n": n, "dtype": "c64", "state_bytes": S, "peak_gbs": peak, "workloads": {}}
    with sv.sv_init(n, 1, sv.SV_C64, sv.SV_INIT_GAUSSIAN) as c:
        for name, gates in work.items():
            steps, _ = sv.sv_plan_gates(n, 1, sv.SV_C64, gates)
            for _ in range(2):  # warm-up: first call on the interpreter, the second compiles (gate_jit.cu)
                sv.sv_apply_gates(c, gates)
            sv.sv_synchronize(c)
            best = None
            for _ in range(args.reps):
                sv.sv_profile(c, True)
                sv.sv_apply_gates(c, gates)
                tl = [ms for k, ms in sv.sv_profile_timeline(c) if k == sv.SV_K_GATE_TILE]
                sv.sv_profile(c, False)
                if best is None or sum(tl) < sum(best):
                    best = tl
            t = sum(best) / 1e3
            passes = [{"gates": int(s["count"]), "proc_bits": bin(s["proc_mask"]).count("1"), "ms": ms,
                       "gbs": 2 * S / (ms / 1e3) / 1e9} for s, ms in zip([s for s in steps if s["kind"] == 0], best)]
            # ALU side of the roofline: a general complex 2x2 on one pair = 16 FMA = 32 FLOP
            # (diagonal / merged ops counted the same: an upper bound on the useful work)
            ops = sum(int(s["ops"]) for s in steps if s["kind"] == 0)
            flop = ops * (1 << (n - 1)) * 32.0
            fp32_peak = 148 * 128 * 2 * 1.965e9  # non-tensor FP32 FMA peak, B200 (148 SMs x 128 lanes)
            res["workloads"][name] = {
                "gates": int(gates.size), "ops_after_host_merging": ops, "passes": len(best), "ms": 1e3 * t,
                "fp32_tflops_upper": flop / t / 1e12, "fp32_frac_upper": flop / t / fp32_peak,
                "gate_amp_updates_per_s": (1 << n) * gates.size / t,
                "avg_pass_gbs": 2 * S * len(best) / t / 1e9,
                "avg_pass_frac": 2 * S * len(best) / t / 1e9 / peak,
                "per_pass": passes}
            print(name, json.dumps({k: v for k, v in res["workloads"][name].items() if k != "per_pass"}), flush=True)
    res["gate_jit"] = {"mode": os.environ.get("SV_GATE_JIT", "auto"), **sv.sv_debug_gate_jit()}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
