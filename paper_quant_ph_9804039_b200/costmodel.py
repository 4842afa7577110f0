"""Analytical execution-time model: the paper's
Eqs. 2-9 and their B200 refit for this library's schedules.

Section 3.5 (symbols in Table 4, constants of the
T3E / SP2 in Fig. 9) models a simulation as computation steps separated by
reorganisations:

  Eq. 4  T_comp(l, n_b, n_l) = l (s^n_l t_t + s^(n_b - 1) t_op)      per step
  Eq. 2  T_reorg(n_l, n_b, n_c) = (s^n_l - s^(n_l - n_c)) (t_lat + t_b q s^(n_b - n_l) + t_lr)
  Eq. 7  T_par = sum_steps [T_comp(l, n_b - n_p, n_l) + T_reorg(n_l, n_b, n_c)]
  Eq. 3/8/9  decoherence: T_dec = 2 l t_lat, T_pardec = 3 T_par + T_dec, T_seqdec = 3 T_seq
  (Eq. 5 flat: n_l = 0; Eq. 6 sequential: n_p = 0, n_c = 0.)

B200 refit: a "laser operation" sweeping all pairs
becomes an HBM tile PASS that applies many of them on-chip, so

  t_op  -> the time per amplitude pair per pass: 2 amplitudes read + written
           = 4 q / BW_pass (BW_pass calibrated per pass class: contiguous,
           strided run length, fused or not), or, for compute-bound gate
           passes, ops_in_pass x t_gate (per pair per gate, calibrated);
  t_t   -> 0 (flat dense store: no link structure to traverse);
  t_b   -> 1 / NVLink bandwidth (all-to-all of (1 - 1/P) S_l per swap);
  t_lat -> one NCCL collective latency per swap / allreduce (the P - 1
           messages of a swap are concurrent, not P - 1 serial latencies);
  t_lr  -> 0 (the exchange is fused into the pass's stores).

Predictions are driven by the library's own host-side schedules
(sv_plan_wht / sv_plan_gates: no device needed); tools/costmodel_validate.py
measures the Table 5/6 analog on the GPU.
"""
from __future__ import annotations

import dataclasses
import math

# --------------------------------------------------------------------------- #
# The paper's model (Eqs. 2-9)                                                 #
# --------------------------------------------------------------------------- #


@dataclasses.dataclass(frozen=True)
class MachineParams:
    """Table 4 symbols; seconds (t_b: seconds per byte; q: bytes per state)."""
    t_op2: float
    t_op3: float
    t_t: float
    t_lat: float
    t_b: float
    t_lr: float
    q: int = 16   # not given by the paper (G24): double complex

    def t_op(self, s: int) -> float:
        return self.t_op2 if s == 2 else self.t_op3


# Fig. 9: measured on the Cray T3E (a) and IBM SP2 (b)
T3E = MachineParams(t_op2=1.5e-6, t_op3=900e-9, t_t=450e-9, t_lat=6e-6, t_b=1e-9, t_lr=80e-6)
SP2 = MachineParams(t_op2=2.3e-6, t_op3=1.28e-6, t_t=1e-6, t_lat=20e-6, t_b=20e-9, t_lr=500e-6)


@dataclasses.dataclass(frozen=True)
class Step:
    """One computation step of Eqs. 6/7: l laser operations on a vector of
    n_b bits with n_l link bits, entered by a reorganisation of n_c bits."""
    l: int
    n_b: int
    n_l: int
    n_c: int = 0


def eq2_reorg(n_l: int, n_b: int, n_c: int, s: int, mp: MachineParams) -> float:
    blocks = s ** n_l - s ** (n_l - n_c)
    return blocks * (mp.t_lat + mp.t_b * mp.q * s ** (n_b - n_l) + mp.t_lr)


def eq3_dec(l_total: int, mp: MachineParams) -> float:
    return 2.0 * l_total * mp.t_lat


def eq4_comp(l: int, n_b: int, n_l: int, s: int, mp: MachineParams) -> float:
    return l * (s ** n_l * mp.t_t + s ** (n_b - 1) * mp.t_op(s))


def eq5_seqflat(l_total: int, n_b_total: int, s: int, mp: MachineParams) -> float:
    return eq4_comp(l_total, n_b_total, 0, s, mp)


def eq6_seqdyn(steps, s: int, mp: MachineParams) -> float:
    return sum(eq4_comp(st.l, st.n_b, st.n_l, s, mp) for st in steps)


def eq7_par(steps, n_p: int, s: int, mp: MachineParams) -> float:
    return sum(eq4_comp(st.l, st.n_b - n_p, st.n_l, s, mp) + eq2_reorg(st.n_l, st.n_b, st.n_c, s, mp)
               for st in steps)


def eq8_pardec(steps, n_p: int, s: int, mp: MachineParams) -> float:
    return 3.0 * eq7_par(steps, n_p, s, mp) + eq3_dec(sum(st.l for st in steps), mp)


def eq9_seqdec(steps, s: int, mp: MachineParams) -> float:
    return 3.0 * eq6_seqdyn(steps, s, mp)


# --------------------------------------------------------------------------- #
# B200 refit                                                                   #
# --------------------------------------------------------------------------- #

ELEM_BYTES = {0: 8, 1: 16}  # SV_C64, SV_C128
TILE_BITS = {0: 13, 1: 12}


def pass_class(tile_mask: int, fused: bool) -> str:
    """Bandwidth class of a tile pass: the contiguous run length of its tile
    (low consecutive slots), whether its first strided slot is >= 18 ("far":
    a >= 2 MiB stride between the 64-128-B runs, which the DRAM serves at ~2/3
    of the near-stride rate, profiles/r1_strided_rw_probe.txt) and whether two
    stage sets are fused around an elementwise op (twice the on-chip work)."""
    run = 0
    while (tile_mask >> run) & 1:
        run += 1
    rest, s = tile_mask >> run, run
    while rest and not rest & 1:
        rest >>= 1
        s += 1
    far = "_far" if rest and s >= 18 else ""
    return f"run{run}{far}{'_fused' if fused else ''}"


@dataclasses.dataclass
class B200Params:
    """Calibrated on the GPU by tools/costmodel_validate.py (defaults: the
    round-1 measurements, profiles/r1_costmodel_b200.json)."""
    # achieved HBM bytes/s (2 S_l per pass) per pass class; "default" covers
    # classes not calibrated
    bw_pass: dict = dataclasses.field(default_factory=lambda: dict({'run4': 6377000000000.0, 'run13': 7010000000000.0, 'run5_far_fused': 6405000000000.0, 'run4_fused': 6337000000000.0, 'run3_far': 3020000000000.0, 'run3_fused': 5104000000000.0, 'run3_far_fused': 3016000000000.0, 'default': 4905000000000.0}))
    bw_mean: float = 5.823e+12        # fused flip + invert-about-mean pass (2 S_l)
    bw_reduce: float = 4.289e+12      # read-only sum pass (S_l)
    t_gate: float = 4.934e-13          # seconds per amplitude pair per general 2x2 op (compute term)
    t_diag: float = 1.008e-13          # ... per diagonal op (phase / controlled phase)
    t_lin: float = 1.076e-12          # ... per merged phase-polynomial op (a run of >= 4 single-control phases)
    t_rel: float = 2.196e-13               # ... per amplitude per shared-memory relayout of a gate pass
    rho: float = 0                  # gate passes: fraction of min(memory, compute) hidden by overlap
    bw_nvlink: float = 900e9       # per direction, NVLink 5 (nominal)
    bw_copy: float = 6.342e+12        # device-local copy (emulated exchange), bytes moved / s
    t_lat: float = 15e-6           # one NCCL collective
    t_launch: float = 2e-6         # per kernel launch gap

    def bw(self, cls: str) -> float:
        """Calibrated bandwidth of a class, else of the same run length and
        stride bucket with the other fusion flag, else of the calibrated class
        with the same flags and the nearest run length, else the default."""
        if cls in self.bw_pass:
            return self.bw_pass[cls]
        fused = cls.endswith("_fused")
        far = "_far" in cls
        run = int(cls[3:].split("_")[0])
        other = f"run{run}{'_far' if far else ''}{'' if fused else '_fused'}"
        if other in self.bw_pass:
            return self.bw_pass[other]
        best = None
        for c, v in self.bw_pass.items():
            if not c.startswith("run") or c.endswith("_fused") != fused:
                continue
            d = 2 * abs(int(c[3:].split("_")[0]) - run) + (("_far" in c) != far)
            if best is None or d < best[0]:
                best = (d, v)
        return best[1] if best else self.bw_pass.get("default", 5.6e12)

    def as_machine_params(self, dtype: int = 0, cls: str = "default") -> MachineParams:
        """The refit in the paper's terms (per pair per pass t_op = 4q/BW)."""
        q = ELEM_BYTES[dtype]
        t_op = 4.0 * q / self.bw(cls)
        return MachineParams(t_op2=t_op, t_op3=t_op, t_t=0.0, t_lat=self.t_lat, t_b=1.0 / self.bw_nvlink,
                             t_lr=0.0, q=q)


def _swap_time(S_l: float, P: int, prm: B200Params, emulated: bool) -> float:
    moved = (1.0 - 1.0 / P) * S_l
    if emulated:  # device-local copies of the whole emulated buffer S_l (read + write)
        return 2.0 * S_l / prm.bw_copy
    return moved / prm.bw_nvlink + prm.t_lat


def predict_wht(n: int, world: int, dtype: int, k: int, prm: B200Params, emulated: bool = False,
                fused_exchange: bool = True) -> dict:
    """sv_iterate(k, SV_DIFFUSE_WHT): sum over the planned passes and swaps."""
    from . import _sv as sv

    plan = sv.sv_plan_wht(n, world, dtype, k, True)
    eb = ELEM_BYTES[dtype]
    S_l = (1 << n) * eb / (1 if emulated else world)
    t_pass = t_swap = 0.0
    npass = nswap = 0
    for st in plan:
        if st["kind"] == 0:
            cls = pass_class(st["tile_mask"], bool(st["pre"] and st["post"]))
            t_pass += 2.0 * S_l / prm.bw(cls) + prm.t_launch
            npass += 1
        elif st["kind"] == 1:
            nswap += 1
            if fused_exchange and not emulated:
                # the pass before the swap stores to the peers: NVLink-bound if slower than HBM
                t_swap += max(0.0, (1.0 - 1.0 / world) * S_l / prm.bw_nvlink - 2.0 * S_l / prm.bw("default")) + prm.t_lat
            elif not fused_exchange:
                t_swap += _swap_time(S_l, world, prm, emulated)
        elif st["kind"] == 2:
            t_pass += prm.t_launch  # one-CTA kernel (tiny states)
    return {"t": t_pass + t_swap, "t_pass": t_pass, "t_swap": t_swap, "passes": npass, "swaps": nswap}


def predict_mean(n: int, world: int, dtype: int, k: int, prm: B200Params, emulated: bool = False) -> dict:
    """sv_iterate(k, SV_DIFFUSE_MEAN): one read-only sum pass, k fused passes,
    an allreduce per iteration when sharded (Eq. 3's two messages become one
    NCCL allreduce)."""
    eb = ELEM_BYTES[dtype]
    S_l = (1 << n) * eb / (1 if emulated else world)
    t = S_l / prm.bw_reduce + k * 2.0 * S_l / prm.bw_mean + (k + 1) * prm.t_launch
    if world > 1 and not emulated:
        t += k * prm.t_lat
    return {"t": t, "passes": k + 1}


def _is_diag(g) -> bool:
    m = g["m"]
    return m[2] == 0.0 and m[3] == 0.0 and m[4] == 0.0 and m[5] == 0.0


def _is_phase1(g) -> bool:
    m = g["m"]
    return _is_diag(g) and m[0] == 1.0 and m[1] == 0.0 and bin(int(g["controls"])).count("1") <= 1


def gate_op_mix(st: dict, order, gates) -> dict:
    """A gate pass's ops split into merged phase runs, diagonal and general
    ops (the diagonal share taken over the pass's gates that are not
    single-control phases, as the host merges them)."""
    idx = order[st["first"]:st["first"] + st["count"]]
    rest = [gates[int(j)] for j in idx if not _is_phase1(gates[int(j)])] or [gates[int(j)] for j in idx]
    fd = sum(1 for g in rest if _is_diag(g)) / len(rest) if rest else 0.0
    lin = st.get("lin_ops", 0)
    other = st["ops"] - lin
    return {"lin": lin, "diag": other * fd, "gen": other * (1.0 - fd)}


def gate_pass_time(t_mem: float, t_ops: float, rho: float) -> float:
    return t_mem + t_ops - rho * min(t_mem, t_ops)


def predict_gates(n: int, world: int, dtype: int, gates, prm: B200Params, emulated: bool = False) -> dict:
    """sv_apply_gates: each pass costs its HBM round trip t_mem plus its
    on-chip work t_ops = ops x pairs x t_op(kind) -- Eq. 4's l s^(n_b - 1) t_op
    next to the memory term -- plus its shared-memory relayouts (count from
    sv_debug_gate_relayouts) x amplitudes x t_rel, less the part the two
    co-resident CTAs per SM overlap: t_mem + t_ops - rho min(t_mem, t_ops)
    (rho = 0 as calibrated); swaps as in predict_wht (unfused all-to-all)."""
    from . import _sv as sv

    steps, order = sv.sv_plan_gates(n, world, dtype, gates)
    rel = sv.sv_debug_gate_relayouts(n, world, dtype, gates)
    eb = ELEM_BYTES[dtype]
    N_l = (1 << n) / (1 if emulated else world)
    S_l = N_l * eb
    t_pass = t_swap = 0.0
    npass = nswap = 0
    for i, st in enumerate(steps):
        if st["kind"] == 1:
            t_swap += _swap_time(S_l, world, prm, emulated)
            nswap += 1
            continue
        f = gate_op_mix(st, order, gates)
        t_ops = (f["lin"] * prm.t_lin + f["diag"] * prm.t_diag + f["gen"] * prm.t_gate) * (N_l / 2.0)
        t_ops += float(rel[i]) * N_l * prm.t_rel
        if st["kind"] == 0:
            t_mem = 2.0 * S_l / prm.bw(pass_class(st["tile_mask"], False))
            t_pass += gate_pass_time(t_mem, t_ops, prm.rho) + prm.t_launch
            npass += 1
        else:
            t_pass += t_ops + prm.t_launch
    return {"t": t_pass + t_swap, "t_pass": t_pass, "t_swap": t_swap, "passes": npass, "swaps": nswap}


def scaling_efficiency(t1: float, tP: float, P: int) -> float:
    """t_1 / (P t_P), as SURVEY 8(d) reports it."""
    return t1 / (P * tP) if tP > 0 else math.nan
