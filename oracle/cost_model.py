"""The paper's analytical execution-time model, Eqs. 2-9, written out literally.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): used by tests/ to check
paper_quant_ph_9804039_b200/costmodel.py.  Shares no code with the product.

Section 3.5 of the paper (P:5222-5318 for Eqs. 2-7, P:5830-5838 for Eqs. 8-9;
Table 4, defines the symbols; Fig. 9, gives the
measured T3E / SP2 constants).  The PostScript equations are garbled in
PAPER.md (their glyphs are listed one per line); the forms below are the
readings of DESIGN.md G24 (they match SPEC's restatement):

  Eq. 2  T_reorg(n_l, n_b, n_c) = (s^n_l - s^(n_l - n_c)) (t_lat + t_b q s^(n_b - n_l) + t_lr)
  Eq. 3  T_dec = 2 l_total t_lat
  Eq. 4  T_comp(l, n_b, n_l) = l (s^n_l t_t + s^(n_b - 1) t_op)
  Eq. 5  T_seqflat = T_comp(l_total, n_b_total, 0)
  Eq. 6  T_seqdyn = sum_steps T_comp(l_step, n_b_step, n_l_step)
  Eq. 7  T_par = sum_steps [T_comp(l_step, n_b_step - n_p, n_l_step) + T_reorg(n_l_step, n_b_step, n_c_step)]
  Eq. 8  T_pardec = 3 T_par + T_dec
  Eq. 9  T_seqdec = 3 T_seq

Eq. 7 writes T_reorg(n_b, n_l, n_c) while Eq. 2 defines T_reorg(n_l, n_b,
n_c); the arguments are bound by name (G16).  q (bytes per state) is not
given by the paper: 16 (double complex), SPEC's choice.
"""
from __future__ import annotations

# Fig. 9 (a) T3E and (b) SP2, "Measured time values"
T3E = dict(t_op2=1.5e-6, t_op3=900e-9, t_t=450e-9, t_lat=6e-6, t_b=1e-9, t_lr=80e-6, q=16)
SP2 = dict(t_op2=2.3e-6, t_op3=1.28e-6, t_t=1e-6, t_lat=20e-6, t_b=20e-9, t_lr=500e-6, q=16)


def t_op(mp: dict, s: int) -> float:
    return mp["t_op2"] if s == 2 else mp["t_op3"]


def t_reorg(n_l: int, n_b: int, n_c: int, s: int, mp: dict) -> float:
    """Eq. 2."""
    return (s ** n_l - s ** (n_l - n_c)) * (mp["t_lat"] + mp["t_b"] * mp["q"] * s ** (n_b - n_l) + mp["t_lr"])


def t_dec(l_total: int, mp: dict) -> float:
    """Eq. 3."""
    return 2 * l_total * mp["t_lat"]


def t_comp(l: int, n_b: int, n_l: int, s: int, mp: dict) -> float:
    """Eq. 4."""
    return l * (s ** n_l * mp["t_t"] + s ** (n_b - 1) * t_op(mp, s))


def t_seqflat(l_total: int, n_b_total: int, s: int, mp: dict) -> float:
    """Eq. 5."""
    return t_comp(l_total, n_b_total, 0, s, mp)


def t_seqdyn(steps: list, s: int, mp: dict) -> float:
    """Eq. 6; steps = [(l_step, n_b_step, n_l_step, n_c_step), ...]."""
    return sum(t_comp(l, n_b, n_l, s, mp) for (l, n_b, n_l, _n_c) in steps)


def t_par(steps: list, n_p: int, s: int, mp: dict) -> float:
    """Eq. 7."""
    return sum(t_comp(l, n_b - n_p, n_l, s, mp) + t_reorg(n_l, n_b, n_c, s, mp) for (l, n_b, n_l, n_c) in steps)


def t_pardec(steps: list, n_p: int, s: int, mp: dict) -> float:
    """Eq. 8."""
    return 3 * t_par(steps, n_p, s, mp) + t_dec(sum(l for (l, _, _, _) in steps), mp)


def t_seqdec(steps: list, s: int, mp: dict) -> float:
    """Eq. 9."""
    return 3 * t_seqdyn(steps, s, mp)
