"""The NCCL plumbing on one GPU: a one-rank communicator (sv_init with world =
1 and an ncclUniqueId) runs every collective the schedule issues through NCCL
-- ncclCommInitRank, the Gaussian init's norm allreduce, the mean diffusion's
2-double allreduce per iteration (Eq. 3's accumulate and redistribute,
P:5248-5251), the decoherence step's global sum, the marked-mass allreduce,
the sampler's allgather / allreduce -- and the host waits through the polling
sync_ctx (ncclCommGetAsyncError).  Results must equal the communicator-free
path bitwise (a one-rank sum is the identity) and the oracle."""
import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests.test_parity_gpu import assert_close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [sv.SV_C64, sv.SV_C128], ids=["c64", "c128"])
def test_one_rank_communicator_runs_the_collectives(dtype, monkeypatch):
    # the launched mean path on both sides (a communicator always takes it)
    monkeypatch.setenv("SV_MEAN_RESIDENT", "0")
    n, m, k, seed = 20, 7, 5, 3
    marked = sv.sv_marked_from_seed(n, m, seed)
    nid = sv.sv_nccl_unique_id()
    out = {}
    for tag, kw in (("nccl", dict(world=1, nccl_id=nid)), ("plain", {})):
        with sv.sv_init(n, seed, dtype, sv.SV_INIT_GAUSSIAN, **kw) as c:
            if tag == "nccl":
                assert sv.sv_comm_info(c) == {"nranks": 1, "rank": 0}
            else:
                assert sv.sv_comm_info(c) == {"nranks": 0, "rank": -1}
            a0 = sv.sv_get_amplitudes(c).astype(np.complex128)
            sv.sv_set_marked(c, marked)
            sv.sv_iterate(c, k, sv.SV_DIFFUSE_MEAN)    # launched path: allreduce per iteration
            sv.sv_iterate(c, 2, sv.SV_DIFFUSE_WHT)
            mass = sv.sv_measure_marked_mass(c)
            surv = sv.sv_iterate_decoherent(c, 2, 0.02, 0.01, 9, 0)
            shots = sv.sv_sample(c, 1000, 11)
            out[tag] = (a0, sv.sv_get_amplitudes(c), mass, surv, shots, sv.sv_norm2(c))
    for x, y in zip(out["nccl"], out["plain"]):
        np.testing.assert_array_equal(x, y)
    a0 = out["plain"][0]
    ref = orc.iterate(orc.iterate(a0.copy(), marked, k, orc.MEAN), marked, 2, orc.WHT)
    assert abs(out["nccl"][2] - orc.marked_mass(ref, marked)) <= 1e-5
    ref, _ = orc.iterate_decoherent(ref, marked, 2, 0.02, 0.01, 9, 0)
    assert_close(out["nccl"][1], ref, dtype, "one-rank NCCL", n=n, k=k + 4)
    assert abs(out["nccl"][5] - orc.norm_sq(ref)) <= (1e-12 if dtype == sv.SV_C128 else 1e-5)
