"""Exhaustive checks of the WHT tile kernel's register / shared-memory layouts
(read from libsv.so's own constexpr layout functions via sv_debug_*):
bijectivity, one owner layout per tile bit, bank-conflict-free shared-memory
wavefronts, and fully coalesced 128-bit global accesses in layout A."""
import ctypes

import pytest

import paper_quant_ph_9804039_b200 as sv

CFG = {sv.SV_C64: dict(T=13, R=5, eb=8), sv.SV_C128: dict(T=12, R=4, eb=16)}


def layout(dtype, phase):
    T, R = CFG[dtype]["T"], CFG[dtype]["R"]
    nt, nr = 1 << (T - R), 1 << R
    e, s = ctypes.c_int(), ctypes.c_int()
    tab = {}
    for t in range(nt):
        for j in range(nr):
            assert sv.lib.sv_debug_tile_layout(dtype, phase, t, j, ctypes.byref(e), ctypes.byref(s)) == 0
            tab[(t, j)] = (e.value, s.value)
    return tab


@pytest.mark.parametrize("dtype", [sv.SV_C64, sv.SV_C128])
def test_layouts_are_bijections_with_single_owner(dtype):
    T = CFG[dtype]["T"]
    for ph in range(3):
        tab = layout(dtype, ph)
        assert sorted(v[0] for v in tab.values()) == list(range(1 << T))
        assert sorted(v[1] for v in tab.values()) == list(range(1 << T))
    for b in range(T):
        assert sum(sv.lib.sv_debug_tile_owner(dtype, ph, b) for ph in range(3)) == 1


@pytest.mark.parametrize("dtype", [sv.SV_C64, sv.SV_C128])
def test_shared_memory_bank_conflict_free(dtype):
    """Each shared-memory wavefront (128 B: 16 lanes x 8 B, or 8 lanes x 16 B)
    touches every 4-byte bank at most once."""
    T, R, eb = CFG[dtype]["T"], CFG[dtype]["R"], CFG[dtype]["eb"]
    nt, nr = 1 << (T - R), 1 << R
    for ph in range(3):
        tab = layout(dtype, ph)
        vec16 = True  # c64 moves 16-B pairs (e, e|1) in every layout; c128 amplitudes are 16 B
        lanes_per_wave = 8 if vec16 else 16
        regs = range(0, nr, 2) if dtype == sv.SV_C64 else range(nr)
        for w in range(nt // 32):
            for j in regs:
                for q in range(0, 32, lanes_per_wave):
                    banks = []
                    for l in range(q, q + lanes_per_wave):
                        byte = tab[(32 * w + l, j)][1] * eb
                        width = 16 if vec16 else eb
                        banks += [((byte + o) // 4) % 32 for o in range(0, width, 4)]
                    assert len(banks) == len(set(banks)), (ph, w, j, q)


@pytest.mark.parametrize("dtype", [sv.SV_C64, sv.SV_C128])
def test_layout_a_is_coalesced(dtype):
    """Layout A: for each register vector, a warp's 32 lanes cover 512
    consecutive bytes of a contiguous tile."""
    T, R, eb = CFG[dtype]["T"], CFG[dtype]["R"], CFG[dtype]["eb"]
    tab = layout(dtype, 0)
    step = 2 if dtype == sv.SV_C64 else 1
    for w in range((1 << (T - R)) // 32):
        for j in range(0, 1 << R, step):
            addr = sorted(tab[(32 * w + l, j)][0] * eb for l in range(32))
            assert addr[-1] - addr[0] == 31 * 16 and len(set(addr)) == 32


def test_strided_two_layout_family():
    """Strided complex64 tiles (processed bits [U, 13), U >= 3): two layouts
    of 8-byte amplitudes -- bijective, each processed bit owned once, carry
    bits 0..2 never register bits, conflict-free half-warp wavefronts, and
    layout A's warp loads cover whole 64-byte carry runs."""
    T, R, eb, D = 13, 5, 8, 2
    nt, nr = 1 << (T - R), 1 << R
    e, s = ctypes.c_int(), ctypes.c_int()
    tabs = []
    for ph in range(2):
        tab = {}
        for t in range(nt):
            for j in range(nr):
                assert sv.lib.sv_debug_tile_layout(D, ph, t, j, ctypes.byref(e), ctypes.byref(s)) == 0
                tab[(t, j)] = (e.value, s.value)
        assert sorted(v[0] for v in tab.values()) == list(range(1 << T))
        assert sorted(v[1] for v in tab.values()) == list(range(1 << T))
        for w in range(nt // 32):
            for j in range(nr):
                for q in (0, 16):
                    banks = []
                    for l in range(q, q + 16):
                        byte = tab[(32 * w + l, j)][1] * eb
                        banks += [(byte // 4) % 32, (byte // 4 + 1) % 32]
                    assert len(banks) == len(set(banks)), (ph, w, j, q)
        tabs.append(tab)
    for b in range(T):
        owners = sum(sv.lib.sv_debug_tile_owner(D, ph, b) for ph in range(2))
        assert owners == (1 if b >= 3 else 0)
    for w in range(nt // 32):  # layout A: lanes 0..7 of a warp = one 64-B run
        for j in range(nr):
            elems = sorted(tabs[0][(32 * w + l, j)][0] for l in range(8))
            assert elems == list(range(elems[0], elems[0] + 8)) and elems[0] % 8 == 0
