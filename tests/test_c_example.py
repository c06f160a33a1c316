"""The C ABI is usable from plain C: examples/mux_example.c compiles and links
against libmux.so with gcc (CPU), and runs on a B200 (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "mux_example")


def _build():
    from paper_2603_02885_b200 import build as mbuild
    mbuild.build()
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    lib_dir = os.path.join(ROOT, "paper_2603_02885_b200")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "mux_example.c"), "-L", lib_dir, "-l:libmux.so",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}", "-o", EXE]
    subprocess.check_call(cmd)


def test_c_example_compiles_and_links():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_c_example_runs():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    _build()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ok" in out.stdout and "status 1" in out.stdout, out.stdout
    assert "rows 192 (valid 184)" in out.stdout, out.stdout
    assert "sliced: slice 0 == plain Y: yes" in out.stdout, out.stdout
