"""bench.py host logic without a GPU: the NVLink attribution of a sharded run
(nvlink_report) on a synthetic per-launch timeline laid out like the
library's schedule, and the CLI contract (configs, defaults)."""
import types

import pytest

import bench
import paper_quant_ph_9804039_b200 as sv


def shim(fused):
    m = types.SimpleNamespace(**{k: getattr(sv, k) for k in dir(sv) if k.startswith("SV_")})
    m.sv_plan_wht = sv.sv_plan_wht
    m.sv_get_exchange = lambda ctx: fused
    return m


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("fused", [True, False])
def test_nvlink_report_attribution(world, fused):
    n, k, steps = 32, 4, 3
    plan = [st["kind"] for st in sv.sv_plan_wht(n, world, sv.SV_C64, k, True) if st["kind"] in (0, 1)]
    pre = {i for i in range(len(plan) - 1) if plan[i] == 0 and plan[i + 1] == 1}
    tl = []
    for _ in range(steps):
        tl.append((sv.SV_K_INIT, 1.0))  # sv_reset's launch: ignored
        for i, kind in enumerate(plan):
            if kind == 1:
                tl.append((sv.SV_K_EXCHANGE, 3.0))
            else:
                tl.append((sv.SV_K_WHT_TILE, 9.0 if i in pre else 5.0))
    r = bench.nvlink_report(shim(fused), None, n, world, sv.SV_C64, k, tl)
    S_l = (1 << n) // world * 8
    moved = (1 - 1 / world) * S_l
    assert r["swaps_per_step"] == 2 * k
    assert r["preswap_pass_ms"] == 9.0 and r["other_pass_ms"] == 5.0 and r["swap_step_ms"] == 3.0
    t = 9.0 if fused else 3.0
    assert r["achieved"] == pytest.approx(moved / (t / 1e3) / 1e9)
    assert r["frac"] == pytest.approx(r["achieved"] / 900.0)


def test_configs_and_defaults():
    assert bench.CONFIGS["c4"][:5] == (32, "c64", 256, 16, "wht")  # BASELINE.json configs[3]
    import sys
    argv, sys.argv = sys.argv, ["bench.py"]
    try:
        args = bench.parse()
    finally:
        sys.argv = argv
    assert (args.gpus, args.config, args.impl) == (1, "c4", "ours") and args.warmup >= 3


@pytest.mark.parametrize("cfg", sorted(bench.CONFIGS))
def test_cpu_sample_shape_is_bounded_and_valid(cfg):
    """The oracle's bounded sample of every config: at most the sample size,
    a marked set the generator accepts (1 <= m <= 2^n), k >= 1; configs smaller
    than the sample run whole."""
    n, _, M, k = bench.CONFIGS[cfg][:4]
    for n_s, k_s in ((26, 2), (24, 1)):
        ns, ms, ks = bench.sample_shape(n, M, k, n_s, k_s)
        assert 1 <= ns <= max(n_s, n) and 1 <= ms <= (1 << ns) and ks >= 1
        if n <= n_s:
            assert (ns, ms) == (n, M) and ks <= k
        else:
            assert (ns, ks) == (n_s, k_s)


@pytest.mark.parametrize("gpus", [1, 2])
def test_self_spawned_ranks_dry_run(gpus):
    """`bench.py --gpus N` with no torchrun environment relaunches itself under
    torch.distributed.run (127.0.0.1 rendezvous); the CPU dry run starts the
    ranks on gloo, describes the sharded schedule and rank 0 prints one line
    naming every rank that joined (verdict r1: the first multi-GPU run must
    start first time)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(gpus), "--dry-run"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == gpus and sorted(d["ranks_joined"]) == list(range(gpus))
    assert d["swaps"] == (2 * 16 if gpus > 1 else 0)  # c4: one qubit swap per transform
