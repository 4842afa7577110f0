#!/usr/bin/env python
"""Table 3 analog: reorganisation (qubit-swap) counts the library's planners
choose for the benchmark circuits at 1..3 parallel bits (2 / 4 / 8 GPUs).

The paper's Table 3 counts the reorganisation operations its
simulator performs for the factoring circuits at 1..11 parallel bits; those
circuits are not given, so the analog runs the gate
bench's circuits (tools/gate_bench.py) through sv_plan_gates and the Grover
iteration through sv_plan_wht, host only.

    python tools/reorg_table.py [--n 30] > profiles/r2_reorg_table.json
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


def workloads(n):
    return {
        "u_layer": C.circuit([C.record(q, C.random_unitary(np.random.default_rng(q))) for q in range(n)]),
        "h_layers_x4": C.circuit([C.record(q, C.H) for q in range(n)] * 4),
        "qft": C.qft_circuit(n),
        "layered_x4": C.layered_circuit(n, 4, 1),
        "random_300": C.random_circuit(n, 300, 2, max_controls=2),
        "structured_300": C.structured_circuit(n, 300, 3, max_controls=2),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    a = ap.parse_args()
    n = a.n
    rows = {}
    for name, gates in workloads(n).items():
        row = {"gates": int(gates.size)}
        for g in range(0, 4):
            steps, _ = sv.sv_plan_gates(n, 1 << g, sv.SV_C64, gates)
            row[f"parallel_bits_{g}"] = {"reorganisations": sum(1 for s in steps if s["kind"] == 1),
                                         "passes": sum(1 for s in steps if s["kind"] == 0)}
        rows[name] = row
    k = 16
    wht = {"iterations": k}
    for g in range(0, 4):
        plan = sv.sv_plan_wht(32, 1 << g, sv.SV_C64, k, True)
        wht[f"parallel_bits_{g}"] = {"reorganisations": sum(1 for s in plan if s["kind"] == 1),
                                     "passes": sum(1 for s in plan if s["kind"] == 0)}
    out = {"what": ("qubit swaps (the paper's reorganisation operations, Fig. 8) planned per circuit; "
                    "parallel_bits_g = 2^g GPUs sharded by the top g qubits"),
           "n": n, "circuits": rows, "grover_c4_n32_k16": wht,
           "paper_table3_context": {"Mult2": [6, 7, 22, 46], "f15_9bits": [4, 8, 21, 71, 161, 363, 582],
                                    "source": "PAPER.md:4884-4973 (1, 2, 3, ... parallel bits)"}}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
