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
