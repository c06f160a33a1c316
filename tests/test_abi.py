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
    (dict(max_rows=524288 + 256), "max_rows"),   # MUX_MAX_ROWS: the workspace's fixed flag region
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


# ---------------------------------------------------------------- decoder-block ops: host validation
A16 = 0x10000  # a 16-byte aligned fake device address (never dereferenced: validation fails first)


def _attn_fwd(mux, R=128, H=4, Hkv=4, d=128, ldq=512, ldk=512, ldv=512, ldo=512, q=A16, scale=0.1):
    L = mux.lib()
    return L.mux_attn_fwd(R, H, Hkv, d, q, ldq, A16, ldk, A16, ldv, A16, scale, A16, ldo, A16, None), \
        L.mux_last_error().decode()


@pytest.mark.parametrize("kw,status,frag", [
    (dict(d=64), 2, "head_dim"),
    (dict(H=6, Hkv=4), 1, "heads"),
    (dict(ldq=256), 1, "strides"),
    (dict(ldk=508), 1, "strides"),
    (dict(q=A16 + 8), 1, "aligned"),
    (dict(scale=float("inf")), 1, "scale"),
])
def test_attn_fwd_rejects(mux, kw, status, frag):
    st, msg = _attn_fwd(mux, **kw)
    assert st == status and frag in msg, (st, msg)


def test_attn_fwd_zero_rows_is_noop(mux):
    st, _ = _attn_fwd(mux, R=0)
    assert st == 0


def test_attn_bwd_workspace_checked(mux):
    L = mux.lib()
    need = mux.attn_workspace_size(128, 4)
    assert need >= 128 * 4 * 4
    st = L.mux_attn_bwd(128, 4, 2, 128, A16, 512, A16, 512, A16, 256, A16, 256, A16, 512, A16, A16, 0.1,
                        A16, 512, A16, 256, A16, 256, A16, need - 1, None)
    assert st == 3 and "workspace" in L.mux_last_error().decode()


def test_elementwise_ops_reject(mux):
    L = mux.lib()
    assert L.mux_rope(16, 2, 10, A16, 64, A16, 10000.0, 0, None) == 1            # head_dim % 16
    assert L.mux_rope(16, 2, 64, A16, 64, A16, 10000.0, 0, None) == 1            # ld < heads * head_dim
    assert L.mux_rope(16, 2, 64, A16, 128, A16, 1.0, 0, None) == 1               # base <= 1
    assert L.mux_rmsnorm_fwd(4, 12, A16, 16, None, 0, None, 0, A16, 1e-5, A16, 16, None) == 1      # dim % 8
    assert L.mux_rmsnorm_fwd(4, 16, A16, 16, None, 0, None, 0, A16, -1.0, A16, 16, None) == 1      # eps < 0
    assert L.mux_rmsnorm_fwd(4, 16, A16, 16, None, 0, A16, 16, A16, 1e-5, A16, 16, None) == 1      # xsum w/o res
    assert L.mux_rmsnorm_fwd(4, 16, A16, 16, A16 + 4, 16, A16, 16, A16, 1e-5, A16, 16, None) == 1  # res misaligned
    assert L.mux_rmsnorm_bwd(4, 16, A16, 16, None, 0, None, 0, A16, 8, A16, 1e-5, None, 0, A16, 16,
                             None) == 1                                                           # ldx < dim
    assert L.mux_rmsnorm_bwd(4, 16, A16, 16, None, 0, A16, 16, A16, 16, A16, 1e-5, None, 0, A16, 16,
                             None) == 1                                                           # dy3 w/o dy2
    assert L.mux_swiglu_fwd(4, 16, A16 + 2, 16, A16, 16, A16, 16, None) == 1    # misaligned
    assert L.mux_swiglu_bwd(4, 16, A16, 16, A16, 16, A16, 16, A16, 16, A16, 12, None) == 1
    assert L.mux_pack_row_start(-1, A16, A16, 16, A16, None) == 1
    assert L.mux_swiglu_fwd(0, 16, A16, 16, A16, 16, A16, 16, None) == 0        # empty: no-op


def test_fwd_hs_and_shrink_validation(mux):
    """mux_linear_fwd_hs needs its input Hs; mux_linear_shrink needs an output Hs and a row range
    that starts on a 256-row pair block (host-side checks, nothing launched)."""
    L = mux.lib()
    ads = _adapters(1)
    st = (ctypes.c_int32 * 1)(0)
    r = L.mux_linear_fwd_hs(1, 0x3000, st, 1, ads, 128, 256, 256, 16, 0x4000, 0x5000, 0x6000, None, 0x8000,
                            1 << 30, None)
    assert r == 1 and "Hs" in L.mux_last_error().decode()
    r = L.mux_linear_shrink(1, 0x3000, st, 1, ads, 512, 256, 256, 16, 0x4000, 100, 512, 0x7000, 0x8000,
                            1 << 30, None)
    assert r == 1 and "row range" in L.mux_last_error().decode()
    r = L.mux_linear_shrink(1, 0x3000, st, 1, ads, 512, 256, 256, 16, 0x4000, 0, 512, None, 0x8000, 1 << 30, None)
    assert r == 1 and "Hs" in L.mux_last_error().decode()


def test_linear_args_layout_matches_header(mux, tmp_path):
    """The ctypes mirror of mux_linear_args / mux_slices has the C layout (compiled from mux.h)."""
    src = tmp_path / "chk.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "mux.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(mux_linear_args), '
                   'sizeof(mux_slices), offsetof(mux_linear_args, slices), offsetof(mux_linear_args, X), '
                   'offsetof(mux_linear_args, row_begin), offsetof(mux_linear_args, stream));return 0;}\n')
    exe = tmp_path / "chk"
    rc = os.system(f"gcc -I {ROOT}/include -I /usr/local/cuda/include {src} -o {exe}")
    assert rc == 0
    got = [int(x) for x in os.popen(str(exe)).read().split()]
    L = mux._LinearArgs
    assert got == [ctypes.sizeof(L), ctypes.sizeof(mux._Slices), L.slices.offset, L.X.offset,
                   L.row_begin.offset, L.stream.offset]


def _generic(mux, op=1, S=2, col_off=(0, 128, 256), n_tasks=1, ranks=None, **kw):
    m = mux
    sl = m._Slices()
    sl.num_slices = S
    for i, c in enumerate(col_off[:mux.MAX_SLICES + 1]):
        sl.col_off[i] = c
    slots = n_tasks * max(S, 1)
    tab = _adapters(max(slots, 1))
    if ranks is not None:
        for i, r in enumerate(ranks):
            tab[i].rank = r
    st_arr = (ctypes.c_int32 * 1)(0)
    a = m._LinearArgs()
    a.op, a.num_segs, a.seg_off, a.seg_task = op, 1, 0x3000, ctypes.addressof(st_arr)
    a.num_adapters, a.adapters, a.slices = n_tasks, ctypes.addressof(tab), ctypes.addressof(sl)
    a.max_rows, a.K, a.N, a.r_cap = 128, 256, 256, 16
    a.X, a.W, a.Y, a.Hs, a.dY, a.dX = 0x4000, 0x5000, 0x6000, 0x7000, 0x9000, 0xA000
    a.workspace, a.workspace_bytes = 0x8000, 1 << 30
    for k, v in kw.items():
        setattr(a, k, v)
    st = m.lib().mux_linear(ctypes.byref(a))
    return st, m.lib().mux_last_error().decode()


@pytest.mark.parametrize("kw,frag", [
    (dict(op=9), "unknown op"),
    (dict(S=0, col_off=(0, 256)), "num_slices"),
    (dict(S=5, col_off=(0, 64, 128, 192, 224, 256)), "num_slices"),
    (dict(col_off=(0, 128, 248)), "end at N"),
    (dict(col_off=(8, 128, 256)), "start at 0"),
    (dict(col_off=(0, 100, 256)), "multiples of 8"),
    (dict(col_off=(0, 256, 256)), "non-empty"),
    (dict(n_tasks=49), "adapter slots"),
    (dict(op=2, Hs=None), "Hs"),
])
def test_generic_linear_validation(mux, kw, frag):
    st, msg = _generic(mux, **kw)
    assert st == 1, (st, msg)
    assert frag in msg, msg


def test_workspace_counts_every_slice(mux):
    """Hs/Gs scratch is [rows, S * r_cap]: a sliced call needs the workspace of S * r_cap."""
    st, msg = _generic(mux, workspace_bytes=mux.linear_workspace_size(1, 128, 256, 256, 16))
    assert st == 3 and "workspace" in msg, msg


def test_workspace_flag_region_is_fixed(mux):
    """The row-block flags sit in a fixed-size region at a fixed offset, so calls with different
    max_rows (or r_cap) can share one workspace: the size grows only by the Gs / Hs scratch
    (2 bytes per row and r_cap column, twice), never by a max_rows-sized flag array."""
    a = mux.linear_workspace_size(4, 1024, 4096, 4096, 16)
    b = mux.linear_workspace_size(4, 1024 + 256 * 64, 4096, 4096, 16)
    assert b - a == 2 * (256 * 64) * 16 * 2
    assert a >= 256 + (524288 // 256) * 8 + 2 * 1024 * 16 * 2
