"""C-ABI checks that need no GPU: libmux.so loads, exports every function
include/mux.h declares, and its host-side validation rejects bad arguments
before touching the device (SURVEY.md §8(b) conventions)."""
import ctypes
import os
import re

import pytest

from paper_2603_02885_b200 import build as mbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mux():
    mbuild.build()
    from paper_2603_02885_b200 import mux as m
    return m


def _declared():
    src = open(os.path.join(ROOT, "include", "mux.h")).read()
    return sorted(set(re.findall(r"MUX_API\s+[\w\s\*]+?\b(mux_\w+)\s*\(", src)))


def test_header_declares_expected(mux):
    assert _declared() == sorted(mux.EXPORTS)


def test_exports_every_declared_symbol(mux):
    L = mux.lib()
    for name in _declared():
        assert hasattr(L, name), name


def test_sm100a_code_in_library():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump -lelf {mbuild.LIB} 2>&1").read()
    assert "sm_100a" in out, out


def test_version_and_bounds(mux):
    assert "sm_100a" in mux.version()
    assert mux.pack_bound_rows(100, 2, 64) == 228
    assert mux.pack_bound_rows(-1, 2, 64) == -1
    assert mux.linear_workspace_size(4, 1024, 4096, 4096, 16) > 1024 * 16 * 2


def _adapters(n, rank=16, ldb=0, scale=2.0):
    tab = (mux_mod()._Adapter * n)()
    for i in range(n):
        tab[i].A = 0x1000 if rank else None
        tab[i].B = 0x2000 if rank else None
        tab[i].rank = rank
        tab[i].ldb = ldb
        tab[i].scale = scale
    return tab


def mux_mod():
    from paper_2603_02885_b200 import mux as m
    return m


def _fwd(mux, **kw):
    args = dict(S=1, seg_off=0x3000, seg_task=(ctypes.c_int32 * 1)(0), na=1, ads=_adapters(1),
                max_rows=128, K=256, N=256, r_cap=16, X=0x4000, W=0x5000, Y=0x6000, Hs=0x7000,
                ws=0x8000, wsb=1 << 30)
    args.update(kw)
    L = mux.lib()
    st = L.mux_linear_fwd(args["S"], args["seg_off"], args["seg_task"], args["na"], args["ads"],
                          args["max_rows"], args["K"], args["N"], args["r_cap"], args["X"], args["W"],
                          args["Y"], args["Hs"], args["ws"], args["wsb"], None)
    return st, L.mux_last_error().decode()


@pytest.mark.parametrize("kw,frag", [
    (dict(S=0), "num_segs"),
    (dict(S=65), "num_segs"),
    (dict(K=100), "multiples of 8"),
    (dict(N=0), "multiples of 8"),
    (dict(r_cap=24), "r_cap"),
    (dict(max_rows=0), "max_rows"),
    (dict(seg_task=(ctypes.c_int32 * 1)(3)), "seg_task"),
    (dict(ads=_adapters(1, rank=65)), "rank"),
    (dict(ads=_adapters(1, rank=32), r_cap=16), "r_cap"),
    (dict(ads=_adapters(1, rank=4)), "ldb"),
    (dict(ads=_adapters(1, scale=float("nan"))), "scale"),
    (dict(X=0x4001), "aligned"),
    (dict(wsb=16), "workspace"),
])
def test_linear_validation(mux, kw, frag):
    st, msg = _fwd(mux, **kw)
    assert st in (1, 3), (st, msg)
    assert frag in msg, msg


def test_pack_validation(mux):
    L = mux.lib()
    off = (ctypes.c_int32 * 2)(0, 1)
    z = ctypes.c_void_p(0x1000)
    st = L.mux_pack_chunks(1, 1, z, z, None, 0, 32, 64, 4, z, z, z, z, z, z, z, z, z, 1 << 20, None)
    assert st == 1 and "chunk_min" in L.mux_last_error().decode()
    st = L.mux_pack_chunks(1, 1, z, z, None, 96, 64, 64, 4, z, z, z, z, z, z, z, z, z, 1 << 20, None)
    assert st == 1 and "chunk_size" in L.mux_last_error().decode()
    st = L.mux_pack_chunks(0, 1, z, z, None, 0, 64, 64, 4, z, z, z, z, z, z, z, z, z, 1 << 20, None)
    assert st == 1
    st = L.mux_pack_chunks(1, 1, z, z, None, 0, 64, 64, 4, z, z, z, z, z, z, z, z, z, 4, None)
    assert st == 3
    del off


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    import importlib
    m = mux_mod()
    monkeypatch.setattr(m, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(m, "_lib", None)
    with pytest.raises(RuntimeError, match="libmux.so not found"):
        m.lib()
    importlib.reload(m)
