"""bench.py's command line (host logic, CPU): `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks on 127.0.0.1 (one process per GPU), and `--mode auto` resolves to
the tensor-parallel arm for N > 1 and the single-GPU step for N = 1."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_gpus_n_spawns_torchrun(monkeypatch):
    calls = []
    import subprocess
    monkeypatch.setattr(subprocess, "call", lambda cmd, env=None: calls.append((cmd, env)) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7", "--warmup", "3"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    (cmd, env), = calls
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "7", "--warmup", "3"]
    assert env["NCCL_DEBUG"] == "INFO"


@pytest.mark.parametrize("world,mode", [("1", "replicas"), ("2", "tp"), ("8", "tp")])
def test_mode_auto(monkeypatch, world, mode):
    seen = {}
    monkeypatch.setenv("WORLD_SIZE", world)
    monkeypatch.setattr(bench, "main_arm", lambda a: seen.setdefault("mode", "replicas"))
    monkeypatch.setattr(bench, "tp_arm", lambda a: seen.setdefault("mode", "tp"))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", world])
    bench.main()
    assert seen["mode"] == mode


def test_reference_arm_is_not_spawned(monkeypatch):
    """--impl reference with --gpus N (no torchrun) runs once, as rank 0, on the host cores."""
    seen = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench, "reference_arm", lambda a: seen.append(a.gpus))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "8"])
    bench.main()
    assert seen == [8]


PK = {"bf16_tflops": 1644.7, "bf16_tflops_sustained": 1397.9, "source": "measured"}


@pytest.mark.parametrize("timed_ms,clk,kind", [
    # a short region whose median clock stayed at max takes the burst peak even if sw_power_cap showed up
    (200.0, {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": ["sw_power_cap"]}, "burst"),
    (200.0, {"sm_mhz": 1882, "sm_max_mhz": 1965, "reasons": []}, "burst"),
    # the clock held > 10 % below max: sustained
    (200.0, {"sm_mhz": 1700, "sm_max_mhz": 1965, "reasons": ["sw_power_cap"]}, "sustained"),
    # thermal / hw slowdown: sustained
    (200.0, {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": ["hw_thermal_slowdown"]}, "sustained"),
    # a long region: sustained
    (1500.0, {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": []}, "sustained"),
    # no clock samples but a power cap reported: sustained
    (200.0, {"reasons": ["sw_power_cap"]}, "sustained"),
])
def test_roofline_peak_choice(timed_ms, clk, kind):
    """roofline.frac's denominator: the measured burst bf16 peak unless the clocks
    were actually held down or the region is long; both fractions always reported."""
    r = bench._roofline(1300.0, PK, timed_ms, clk, 3, "k")
    assert r["peak_kind"].startswith(kind), r
    assert r["peak"] == (PK["bf16_tflops"] if kind == "burst" else PK["bf16_tflops_sustained"])
    assert abs(r["frac"] - 1300.0 / r["peak"]) < 1e-12
    assert abs(r["frac_of_burst"] - 1300.0 / 1644.7) < 1e-12
    assert abs(r["frac_of_sustained"] - 1300.0 / 1397.9) < 1e-12
