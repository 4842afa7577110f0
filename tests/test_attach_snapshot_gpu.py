"""sv_attach (compute in a caller-owned torch buffer, SURVEY 8(b) phase-2
option) and sv_snapshot (SPEC's text snapshot) through the C ABI,
against the oracle."""
import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests.test_parity_gpu import assert_close, rand_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [sv.SV_C64, sv.SV_C128], ids=["c64", "c128"])
@pytest.mark.parametrize("n", [12, 18])
def test_attach_torch_buffer_iterates_in_place(dtype, n):
    import torch
    a = rand_state(n, dtype)
    tdt = torch.complex64 if dtype == sv.SV_C64 else torch.complex128
    t = torch.from_numpy(a.astype(sv.NP_DTYPE[dtype])).to("cuda")
    marked = orc.marked_from_seed(n, 5, n)
    c = sv.sv_init(n, 0, dtype, sv.SV_INIT_ZERO_STATE)
    sv.sv_attach(c, t.data_ptr(), t.numel() * t.element_size())
    sv.sv_set_marked(c, marked)
    sv.sv_iterate(c, 3, sv.SV_DIFFUSE_WHT)
    sv.sv_synchronize(c)
    via_api = sv.sv_get_amplitudes(c)
    sv.sv_free(c)  # must not free the caller's buffer
    got = t.cpu().numpy()
    ref = orc.iterate(a.copy(), marked, 3, orc.WHT)
    assert_close(got, ref, dtype, f"attach n={n}", n=n, k=3)
    np.testing.assert_array_equal(via_api, got)
    t.add_(0)  # still a live allocation
    torch.cuda.synchronize()
    assert t.dtype == tdt


def test_attach_rejects_bad_buffers():
    import torch
    n = 14
    with sv.sv_init(n, 0, sv.SV_C64) as c:
        good = torch.zeros(1 << n, dtype=torch.complex64, device="cuda")
        for ptr, nb in ((good.data_ptr(), good.numel() * 8 - 8),     # size
                        (good.data_ptr() + 8, good.numel() * 8),     # alignment
                        (0, good.numel() * 8)):                      # NULL
            with pytest.raises(sv.SvError) as e:
                sv.sv_attach(c, ptr, nb)
            assert e.value.code == sv.SV_EINVAL
        host = np.zeros(1 << n, np.complex64)
        with pytest.raises(sv.SvError):
            sv.sv_attach(c, host.ctypes.data, host.nbytes)
        # the context still works on its own buffer
        sv.sv_set_marked(c, [3])
        sv.sv_iterate(c, 2)
        assert sv.sv_measure_marked_mass(c) > 0


@pytest.mark.parametrize("dtype", [sv.SV_C64, sv.SV_C128], ids=["c64", "c128"])
def test_snapshot_matches_oracle_snapshot(dtype, tmp_path):
    n, k = 11, 4
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, 3, 2)
    from tests.test_parity_gpu import ctx_with
    with ctx_with(a, dtype) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        lines = sv.sv_snapshot(c, str(tmp_path / "gpu.txt"))
        got = sv.sv_get_amplitudes(c)
    ref = orc.iterate(a.copy(), marked, k, orc.WHT)
    assert orc.write_snapshot(ref, str(tmp_path / "oracle.txt")) == lines == (1 << n)
    s_g, m_g, amps_g = orc.read_snapshot(str(tmp_path / "gpu.txt"))
    s_o, m_o, amps_o = orc.read_snapshot(str(tmp_path / "oracle.txt"))
    assert (s_g, m_g) == (s_o, m_o) == (2, n)
    assert sorted(amps_g) == sorted(amps_o) == list(range(1 << n))
    # the file holds the stored values exactly (17 significant digits round-trip)
    np.testing.assert_array_equal(np.array([amps_g[i] for i in range(1 << n)]), got.astype(np.complex128))
    assert_close(np.array([amps_g[i] for i in range(1 << n)]), np.array([amps_o[i] for i in range(1 << n)]),
                 dtype, "snapshot", n=n, k=k)


def test_snapshot_sparse_states_and_guard(tmp_path):
    with sv.sv_init(5, 0, sv.SV_C128, sv.SV_INIT_ZERO_STATE) as c:  # |0...0>: one line
        assert sv.sv_snapshot(c, str(tmp_path / "z.txt")) == 1
        assert open(tmp_path / "z.txt").read() == "s=2 M=5\n0 1 0\n"
    with sv.sv_init(1, 0, sv.SV_C128, sv.SV_INIT_UNIFORM) as c:  # Fig. 1(b): both 2^-1/2
        sv.sv_snapshot(c, str(tmp_path / "u.txt"))
        assert open(tmp_path / "u.txt").read() == "s=2 M=1\n0 0.70710678118654757 0\n1 0.70710678118654757 0\n"
    with sv.sv_init(27, 0, sv.SV_C64) as c:
        with pytest.raises(sv.SvError) as e:
            sv.sv_snapshot(c, str(tmp_path / "big.txt"))
        assert e.value.code == sv.SV_ETOOBIG
    with sv.sv_init(4, 0, sv.SV_C64) as c:
        with pytest.raises(sv.SvError) as e:
            sv.sv_snapshot(c, "/nonexistent-dir/x.txt")
        assert e.value.code == sv.SV_EINVAL
