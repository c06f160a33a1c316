"""Thin Python binding of libmux (include/mux.h) — argument marshalling only.

torch is used for device memory and the current stream; every step of the
path runs in libmux's CUDA kernels.  There is no fallback: if libmux.so is
missing or the GPU path fails, these functions raise.

Names follow mux.h: pack_chunks, pack_apply, linear_fwd, linear_bwd.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# MUX_LIB_FILE selects an experiment build under this directory (A/B only, e.g. libmux_direct.so)
LIB_PATH = os.path.join(_HERE, os.environ.get("MUX_LIB_FILE", "libmux.so"))

MUX_OK = 0
STATUS = {0: "MUX_OK", 1: "MUX_ERR_INVALID_ARGUMENT", 2: "MUX_ERR_UNSUPPORTED",
          3: "MUX_ERR_INSUFFICIENT_BUFFER", 4: "MUX_ERR_CUDA"}
MAX_SEGMENTS = 64
MAX_ADAPTERS = 64
MAX_SLICES = 4
MAX_ADAPTER_SLOTS = 96

BWD_DX, BWD_GRADS = 1, 2

EXPORTS = ("mux_last_error", "mux_version", "mux_pack_bound_rows", "mux_pack_workspace_size",
           "mux_pack_chunks", "mux_pack_apply", "mux_linear_workspace_size", "mux_linear_fwd",
           "mux_linear_bwd", "mux_linear_bwd_part", "mux_pack_row_start", "mux_attn_fwd", "mux_attn_workspace_size", "mux_attn_bwd",
           "mux_rope", "mux_rmsnorm_fwd", "mux_rmsnorm_bwd", "mux_swiglu_fwd", "mux_swiglu_bwd", "mux_add", "mux_rs_flags_elems", "mux_linear_fwd_rs",
           "mux_linear_bwd_dx_rs", "mux_rs_reduce", "mux_ag_push", "mux_ag_release", "mux_linear_fwd_ag",
           "mux_linear_bwd_ag", "mux_linear_fwd_hs", "mux_linear_shrink", "mux_nvls_flags_elems",
           "mux_nvls_reduce_scatter", "mux_nvls_all_gather", "mux_nvls_release", "mux_linear")


class MuxError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class PackInfo(ctypes.Structure):
    _fields_ = [("chunk_size", ctypes.c_int32), ("num_chunks", ctypes.c_int32),
                ("num_packs", ctypes.c_int32), ("total_rows", ctypes.c_int32),
                ("valid_rows", ctypes.c_int32), ("zero_pad_rows", ctypes.c_int32),
                ("overflow", ctypes.c_int32)]


PACK_INFO_FIELDS = [f[0] for f in PackInfo._fields_]


class _Adapter(ctypes.Structure):
    _fields_ = [("A", ctypes.c_void_p), ("B", ctypes.c_void_p), ("dA", ctypes.c_void_p),
                ("dB", ctypes.c_void_p), ("rank", ctypes.c_int32), ("ldb", ctypes.c_int32),
                ("scale", ctypes.c_float)]


_lib = None


def lib():
    """Load libmux.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libmux.so not found at {LIB_PATH}: run __graft_entry__.build() "
                               "(python -m paper_2603_02885_b200.build)")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        L.mux_last_error.restype = ctypes.c_char_p
        L.mux_version.restype = ctypes.c_char_p
        L.mux_pack_bound_rows.restype = I64
        L.mux_pack_bound_rows.argtypes = [I64, I32, I32]
        L.mux_pack_workspace_size.restype = SZ
        L.mux_pack_workspace_size.argtypes = [I32, I32]
        L.mux_pack_chunks.restype = ctypes.c_int
        L.mux_pack_chunks.argtypes = [I32, I32, P, P, P, I32, I32, I32, I32, P, P, P, P, P, P, P, P, P, SZ, P]
        L.mux_pack_apply.restype = ctypes.c_int
        L.mux_pack_apply.argtypes = [I32, I32, I32, P, P, P, P]
        L.mux_linear_workspace_size.restype = SZ
        L.mux_linear_workspace_size.argtypes = [I32, I32, I32, I32, I32]
        L.mux_linear_fwd.restype = ctypes.c_int
        L.mux_linear_fwd.argtypes = [I32, P, P, I32, P, I32, I32, I32, I32, P, P, P, P, P, SZ, P]
        L.mux_linear_fwd_hs.restype = ctypes.c_int
        L.mux_linear_fwd_hs.argtypes = [I32, P, P, I32, P, I32, I32, I32, I32, P, P, P, P, P, SZ, P]
        L.mux_linear_shrink.restype = ctypes.c_int
        L.mux_linear_shrink.argtypes = [I32, P, P, I32, P, I32, I32, I32, I32, P, I32, I32, P, P, SZ, P]
        L.mux_linear_bwd.restype = ctypes.c_int
        L.mux_linear_bwd.argtypes = [I32, P, P, I32, P, I32, I32, I32, I32, P, P, P, P, P, P, SZ, P]
        L.mux_linear_bwd_part.restype = ctypes.c_int
        L.mux_linear_bwd_part.argtypes = [I32, I32, P, P, I32, P, I32, I32, I32, I32, P, P, P, P, P, P, SZ, P]
        F = ctypes.c_float
        L.mux_pack_row_start.restype = ctypes.c_int
        L.mux_pack_row_start.argtypes = [I32, P, P, I32, P, P]
        L.mux_attn_fwd.restype = ctypes.c_int
        L.mux_attn_fwd.argtypes = [I32, I32, I32, I32, P, I64, P, I64, P, I64, P, F, P, I64, P, P]
        L.mux_attn_workspace_size.restype = SZ
        L.mux_attn_workspace_size.argtypes = [I32, I32]
        L.mux_attn_bwd.restype = ctypes.c_int
        L.mux_attn_bwd.argtypes = [I32, I32, I32, I32, P, I64, P, I64, P, I64, P, I64, P, I64, P, P, F,
                                   P, I64, P, I64, P, I64, P, SZ, P]
        L.mux_rope.restype = ctypes.c_int
        L.mux_rope.argtypes = [I32, I32, I32, P, I64, P, F, I32, P]
        L.mux_rmsnorm_fwd.restype = ctypes.c_int
        L.mux_rmsnorm_fwd.argtypes = [I32, I32, P, I64, P, I64, P, I64, P, F, P, I64, P]
        L.mux_rmsnorm_bwd.restype = ctypes.c_int
        L.mux_rmsnorm_bwd.argtypes = [I32, I32, P, I64, P, I64, P, I64, P, I64, P, F, P, I64, P, I64, P]
        L.mux_swiglu_fwd.restype = ctypes.c_int
        L.mux_swiglu_fwd.argtypes = [I32, I32, P, I64, P, I64, P, I64, P]
        L.mux_swiglu_bwd.restype = ctypes.c_int
        L.mux_swiglu_bwd.argtypes = [I32, I32, P, I64, P, I64, P, I64, P, I64, P, I64, P]
        L.mux_add.restype = ctypes.c_int
        L.mux_add.argtypes = [I32, I32, P, I64, P, I64, P, I64, P]
        L.mux_rs_flags_elems.restype = SZ
        L.mux_rs_flags_elems.argtypes = [I32]
        L.mux_linear_fwd_rs.restype = ctypes.c_int
        L.mux_linear_fwd_rs.argtypes = [I32, P, P, I32, P, I32, I32, I32, I32, P, P, P, P, P, SZ, P]
        L.mux_linear_bwd_dx_rs.restype = ctypes.c_int
        L.mux_linear_bwd_dx_rs.argtypes = [I32, P, P, I32, P, I32, I32, I32, I32, P, P, P, P, P, P, SZ, P]
        L.mux_rs_reduce.restype = ctypes.c_int
        L.mux_rs_reduce.argtypes = [P, I32, P, I64, P]
        L.mux_ag_push.restype = ctypes.c_int
        L.mux_ag_push.argtypes = [P, P, I64, I32, P]
        L.mux_ag_release.restype = ctypes.c_int
        L.mux_ag_release.argtypes = [P, P]
        L.mux_linear_fwd_ag.restype = ctypes.c_int
        L.mux_linear_fwd_ag.argtypes = [I32, P, P, I32, P, I32, I32, I32, I32, P, P, P, P, P, SZ, P]
        L.mux_linear_bwd_ag.restype = ctypes.c_int
        L.mux_linear_bwd_ag.argtypes = [I32, P, P, I32, P, I32, I32, I32, I32, P, P, P, P, P, P, SZ, P]
        L.mux_nvls_flags_elems.restype = SZ
        L.mux_nvls_flags_elems.argtypes = []
        L.mux_nvls_reduce_scatter.restype = ctypes.c_int
        L.mux_nvls_reduce_scatter.argtypes = [P, I32, P, I64, I32, P]
        L.mux_nvls_all_gather.restype = ctypes.c_int
        L.mux_nvls_all_gather.argtypes = [P, P, I64, I32, I32, P]
        L.mux_nvls_release.restype = ctypes.c_int
        L.mux_nvls_release.argtypes = [P, P]
        L.mux_linear.restype = ctypes.c_int
        L.mux_linear.argtypes = [P]
        _lib = L
    return _lib


def version() -> str:
    return lib().mux_version().decode()


def _check(status: int):
    if status != MUX_OK:
        raise MuxError(status, lib().mux_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dev_i32(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        assert x.dtype == torch.int32 and x.is_contiguous()
        return x.to(device)
    return torch.as_tensor(list(x), dtype=torch.int32, device=device)


# ---------------------------------------------------------------- host-side argument checks
def _need(cond: bool, msg: str):
    if not cond:
        raise ValueError(msg)


def _check_mat(name: str, t: Optional[torch.Tensor], shape, dtype=torch.bfloat16, device=None, dense=True):
    """t must be a `dtype` tensor of `shape` on `device` whose rows are contiguous (and, with
    dense=True, packed back to back: the ABI takes no leading dimension for it)."""
    if t is None:
        return
    _need(isinstance(t, torch.Tensor), f"{name} must be a torch.Tensor")
    _need(t.dtype == dtype, f"{name}: dtype {t.dtype}, expected {dtype}")
    _need(tuple(t.shape) == tuple(shape), f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    _need(t.is_cuda, f"{name} must be a CUDA tensor")
    if device is not None:
        _need(t.device == device, f"{name} is on {t.device}, expected {device}")
    if t.dim() == 2 and t.numel() > 0:
        _need(t.stride(1) == 1, f"{name}: rows must be contiguous")
        if dense:
            _need(t.stride(0) == t.shape[1], f"{name}: must be contiguous (row stride {t.stride(0)})")


def _check_linear(seg_off, seg_task, adapters, X, W, r_cap, K=None, N=None, *, Y=None, Hs=None, dY=None,
                  dX=None, rows=None, grads=False):
    """Everything the C side cannot check through raw pointers: dtypes, shapes, contiguity, device.
    A mismatch raises ValueError before any launch (the C side then validates sizes/alignment)."""
    if X is not None:
        _need(X.dim() == 2, "X must be 2-D [rows, K]")
        rows, K = X.shape if rows is None else (rows, X.shape[1])
    _need(K is not None and rows is not None, "K and rows are required")
    _need(W is not None or N is not None, "W [N, K] (or N) is required")
    if W is not None:
        _need(W.dim() == 2, "W must be 2-D [N, K]")
        N = W.shape[0] if N is None else N
    dev = W.device if W is not None else X.device
    _check_mat("X", X, (rows, K), device=dev)
    _check_mat("W", W, (N, K), device=dev)
    _check_mat("Y", Y, (rows, N), device=dev)
    _check_mat("Hs", Hs, (rows, r_cap), device=dev)
    _check_mat("dY", dY, (rows, N), device=dev)
    _check_mat("dX", dX, (rows, K), device=dev)
    _need(isinstance(seg_off, torch.Tensor) and seg_off.dtype == torch.int32 and seg_off.is_cuda
          and seg_off.is_contiguous() and seg_off.numel() == len(seg_task) + 1,
          f"seg_off must be a contiguous int32 CUDA tensor of len(seg_task)+1 = {len(seg_task) + 1} entries")
    for i, a in enumerate(adapters):
        if a.rank == 0:
            continue
        # memoised per adapter object on the tensors it holds (a call with 64 adapters would
        # otherwise spend more host time here than the GPU spends on a short GEMM)
        key = (K, N, dev, grads, id(a.A), id(a.B), id(a.dA), id(a.dB),
               a.A.data_ptr() if a.A is not None else 0, a.B.data_ptr() if a.B is not None else 0)
        if getattr(a, "_checked", None) == key:
            continue
        _check_mat(f"adapters[{i}].A", a.A, (a.rank, K), device=dev)
        _check_mat(f"adapters[{i}].B", a.B, (N, a.rank), device=dev, dense=False)
        if grads:
            _check_mat(f"adapters[{i}].dA", a.dA, (a.rank, K), torch.float32, dev)
            _check_mat(f"adapters[{i}].dB", a.dB, (N, a.rank), torch.float32, dev)
        a._checked = key


# ---------------------------------------------------------------- packing
def pack_bound_rows(total_tokens: int, num_seqs: int, chunk_size_or_max: int) -> int:
    return int(lib().mux_pack_bound_rows(total_tokens, num_seqs, chunk_size_or_max))


def pack_chunks(task_seq_off, seq_len, pack_capacity=None, chunk_size: int = 0, chunk_min: int = 64,
                max_rows: int = None, max_chunks: int = None, device="cuda", stream=None, out=None):
    """mux_pack_chunks.  task_seq_off/seq_len/pack_capacity: int32 device tensors
    (or host sequences, copied).  Returns a dict of device tensors; info is a
    device int32 tensor of PACK_INFO_FIELDS (read it with read_info())."""
    tso = _dev_i32(task_seq_off, device)
    sl = _dev_i32(seq_len, device)
    pc = None if pack_capacity is None else _dev_i32(pack_capacity, device)
    M = tso.numel() - 1
    S = sl.numel()
    if max_rows is None or max_chunks is None:
        raise ValueError("max_rows and max_chunks are required (host never reads device data)")
    if out is None:
        out = alloc_pack_outputs(M, S, max_rows, max_chunks, device)
    o = out
    _check(lib().mux_pack_chunks(M, S, _ptr(tso), _ptr(sl), _ptr(pc), chunk_size, chunk_min, max_rows,
                                 max_chunks, _ptr(o["seg_off"]), _ptr(o["seq_row"]), _ptr(o["chunk_task"]),
                                 _ptr(o["chunk_pack"]), _ptr(o["chunk_valid"]), _ptr(o["chunk_dep"]),
                                 _ptr(o["row_src"]), _ptr(o["info"]), _ptr(o["workspace"]),
                                 o["workspace"].numel(), _stream(stream)))
    return o


def alloc_pack_outputs(M: int, S: int, max_rows: int, max_chunks: int, device="cuda"):
    i32 = dict(dtype=torch.int32, device=device)
    ws = int(lib().mux_pack_workspace_size(M, S))
    return {"seg_off": torch.empty(M + 1, **i32), "seq_row": torch.empty(max(S, 1), **i32),
            "chunk_task": torch.empty(max(max_chunks, 1), **i32),
            "chunk_pack": torch.empty(max(max_chunks, 1), **i32),
            "chunk_valid": torch.empty(max(max_chunks, 1), **i32),
            "chunk_dep": torch.empty(max(max_chunks, 1), **i32),
            "row_src": torch.empty(max(max_rows, 1), **i32),
            "info": torch.empty(len(PACK_INFO_FIELDS), **i32),
            "workspace": torch.empty(ws, dtype=torch.uint8, device=device)}


def read_info(info: torch.Tensor) -> dict:
    v = info.cpu().tolist()
    return dict(zip(PACK_INFO_FIELDS, v))


def pack_apply(row_src: torch.Tensor, src: torch.Tensor, max_rows: int, out: torch.Tensor = None,
               stream=None) -> torch.Tensor:
    """mux_pack_apply: packed[r] = src[row_src[r]] or 0."""
    assert src.dtype == torch.bfloat16 and src.is_contiguous() and src.dim() == 2
    cols = src.shape[1]
    if out is None:
        out = torch.empty(max_rows, cols, dtype=torch.bfloat16, device=src.device)
    _check(lib().mux_pack_apply(max_rows, cols, src.shape[0], _ptr(row_src), _ptr(src), _ptr(out),
                                _stream(stream)))
    return out


# ---------------------------------------------------------------- linear
@dataclass
class Adapter:
    """One task's LoRA adapter on one linear layer.  B is stored with a leading
    dimension that is a multiple of 8 (TMA needs 16-byte rows): `B` is the
    [N, rank] view of that padded storage, so no copy happens per call."""
    A: Optional[torch.Tensor]          # [rank, K] bf16
    B: Optional[torch.Tensor]          # [N, rank] bf16 view, row stride ldb
    rank: int
    scale: float
    dA: Optional[torch.Tensor] = None  # [rank, K] fp32
    dB: Optional[torch.Tensor] = None  # [N, rank] fp32

    @property
    def ldb(self) -> int:
        if self.B is None or self.rank == 0:
            return 0
        return int(self.B.stride(0))


def make_B_storage(N: int, rank: int, device="cuda") -> torch.Tensor:
    """Zeroed [N, rank] bf16 view over [N, round_up(rank, 8)] storage."""
    ld = max(8, -(-rank // 8) * 8)
    return torch.zeros(N, ld, dtype=torch.bfloat16, device=device)[:, :rank]


def _adapter_table(adapters: Sequence[Adapter], want_grads: bool):
    tab = (_Adapter * len(adapters))()
    for i, a in enumerate(adapters):
        tab[i].A = a.A.data_ptr() if (a.A is not None and a.rank > 0) else None
        tab[i].B = a.B.data_ptr() if (a.B is not None and a.rank > 0) else None
        tab[i].dA = a.dA.data_ptr() if (want_grads and a.dA is not None) else None
        tab[i].dB = a.dB.data_ptr() if (want_grads and a.dB is not None) else None
        tab[i].rank = a.rank
        tab[i].ldb = a.ldb
        tab[i].scale = float(a.scale)
    return tab


def linear_workspace_size(num_segs: int, max_rows: int, K: int, N: int, r_cap: int) -> int:
    return int(lib().mux_linear_workspace_size(num_segs, max_rows, K, N, r_cap))


def _i32_host(seq_task):
    arr = (ctypes.c_int32 * len(seq_task))(*[int(x) for x in seq_task])
    return arr


def linear_fwd(seg_off: torch.Tensor, seg_task: Sequence[int], adapters: Sequence[Adapter],
               X: torch.Tensor, W: torch.Tensor, r_cap: int, Y: torch.Tensor = None,
               Hs: torch.Tensor = None, workspace: torch.Tensor = None, want_hs: bool = True, stream=None):
    """mux_linear_fwd.  Returns (Y, Hs)."""
    max_rows, K = X.shape
    N = W.shape[0]
    dev = X.device
    if Y is None:
        Y = torch.empty(max_rows, N, dtype=torch.bfloat16, device=dev)
    if Hs is None and want_hs:
        Hs = torch.empty(max_rows, r_cap, dtype=torch.bfloat16, device=dev)
    _check_linear(seg_off, seg_task, adapters, X, W, r_cap, Y=Y, Hs=Hs)
    S = len(seg_task)
    if workspace is None:
        workspace = torch.zeros(linear_workspace_size(S, max_rows, K, N, r_cap), dtype=torch.uint8, device=dev)
    tab = _adapter_table(adapters, False)
    st = _i32_host(seg_task)
    _check(lib().mux_linear_fwd(S, _ptr(seg_off), st, len(adapters), tab, max_rows, K, N, r_cap,
                                _ptr(X), _ptr(W), _ptr(Y), _ptr(Hs), _ptr(workspace), workspace.numel(),
                                _stream(stream)))
    return Y, Hs


def linear_fwd_hs(seg_off: torch.Tensor, seg_task: Sequence[int], adapters: Sequence[Adapter],
                  X: torch.Tensor, W: torch.Tensor, Hs: torch.Tensor, r_cap: int, Y: torch.Tensor = None,
                  workspace: torch.Tensor = None, stream=None):
    """mux_linear_fwd_hs: forward with the shrink Hs given (input).  Returns Y."""
    max_rows, K = X.shape
    N = W.shape[0]
    if Y is None:
        Y = torch.empty(max_rows, N, dtype=torch.bfloat16, device=X.device)
    _need(Hs is not None, "linear_fwd_hs needs Hs")
    _check_linear(seg_off, seg_task, adapters, X, W, r_cap, Y=Y, Hs=Hs)
    S = len(seg_task)
    if workspace is None:
        workspace = torch.zeros(linear_workspace_size(S, max_rows, K, N, r_cap), dtype=torch.uint8, device=X.device)
    _check(lib().mux_linear_fwd_hs(S, _ptr(seg_off), _i32_host(seg_task), len(adapters),
                                   _adapter_table(adapters, False), max_rows, K, N, r_cap, _ptr(X), _ptr(W),
                                   _ptr(Y), _ptr(Hs), _ptr(workspace), workspace.numel(), _stream(stream)))
    return Y


def linear_shrink(seg_off: torch.Tensor, seg_task: Sequence[int], adapters: Sequence[Adapter],
                  X: torch.Tensor, N: int, r_cap: int, row_begin: int = 0, row_end: int = None,
                  Hs: torch.Tensor = None, workspace: torch.Tensor = None, stream=None):
    """mux_linear_shrink: Hs rows of the pair row blocks in [row_begin, row_end).  Returns Hs."""
    max_rows, K = X.shape
    if row_end is None:
        row_end = max_rows
    if Hs is None:
        Hs = torch.empty(max_rows, r_cap, dtype=torch.bfloat16, device=X.device)
    _check_linear(seg_off, seg_task, adapters, X, None, r_cap, N=N, Hs=Hs)
    S = len(seg_task)
    if workspace is None:
        workspace = torch.zeros(linear_workspace_size(S, max_rows, K, N, r_cap), dtype=torch.uint8, device=X.device)
    _check(lib().mux_linear_shrink(S, _ptr(seg_off), _i32_host(seg_task), len(adapters),
                                   _adapter_table(adapters, False), max_rows, K, N, r_cap, _ptr(X), row_begin,
                                   row_end, _ptr(Hs), _ptr(workspace), workspace.numel(), _stream(stream)))
    return Hs


def linear_bwd(seg_off: torch.Tensor, seg_task: Sequence[int], adapters: Sequence[Adapter],
               dY: torch.Tensor, X: torch.Tensor, W: torch.Tensor, Hs: torch.Tensor, r_cap: int,
               dX: torch.Tensor = None, want_dx: bool = True, workspace: torch.Tensor = None, stream=None,
               part: int = 0):
    """mux_linear_bwd (part 0), or one half of it: part 1 = the dX GEMM (and Gs), part 2 = the
    adapter gradients (after part 1, same workspace).  Writes adapters[i].dA / .dB (allocated
    if None); returns dX."""
    max_rows, K = X.shape
    N = W.shape[0]
    dev = X.device
    if dX is None and want_dx:
        dX = torch.empty(max_rows, K, dtype=torch.bfloat16, device=dev)
    for a in adapters:
        if a.rank > 0:
            if a.dA is None:
                a.dA = torch.empty(a.rank, K, dtype=torch.float32, device=dev)
            if a.dB is None:
                a.dB = torch.empty(N, a.rank, dtype=torch.float32, device=dev)
    _check_linear(seg_off, seg_task, adapters, X, W, r_cap, Hs=Hs, dY=dY, dX=dX, grads=True)
    S = len(seg_task)
    if workspace is None:
        workspace = torch.zeros(linear_workspace_size(S, max_rows, K, N, r_cap), dtype=torch.uint8, device=dev)
    tab = _adapter_table(adapters, True)
    st = _i32_host(seg_task)
    if part == 0:
        _check(lib().mux_linear_bwd(S, _ptr(seg_off), st, len(adapters), tab, max_rows, K, N, r_cap,
                                    _ptr(dY), _ptr(X), _ptr(W), _ptr(Hs), _ptr(dX), _ptr(workspace),
                                    workspace.numel(), _stream(stream)))
    else:
        _check(lib().mux_linear_bwd_part(part, S, _ptr(seg_off), st, len(adapters), tab, max_rows, K, N, r_cap,
                                         _ptr(dY), _ptr(X), _ptr(W), _ptr(Hs), _ptr(dX), _ptr(workspace),
                                         workspace.numel(), _stream(stream)))
    return dX


# ---------------------------------------------------------------- fused projections (column slices)
OP_FWD, OP_FWD_HS, OP_SHRINK, OP_BWD, OP_BWD_DX, OP_BWD_GRADS, OP_SHRINK_BWD = 1, 2, 3, 4, 5, 6, 7


class _Slices(ctypes.Structure):
    _fields_ = [("num_slices", ctypes.c_int32), ("col_off", ctypes.c_int32 * (MAX_SLICES + 1))]


class _LinearArgs(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("num_segs", ctypes.c_int32), ("seg_off", ctypes.c_void_p),
                ("seg_task", ctypes.c_void_p), ("num_adapters", ctypes.c_int32), ("adapters", ctypes.c_void_p),
                ("slices", ctypes.c_void_p), ("max_rows", ctypes.c_int32), ("K", ctypes.c_int32),
                ("N", ctypes.c_int32), ("r_cap", ctypes.c_int32), ("X", ctypes.c_void_p), ("W", ctypes.c_void_p),
                ("dY", ctypes.c_void_p), ("Y", ctypes.c_void_p), ("Hs", ctypes.c_void_p), ("dX", ctypes.c_void_p),
                ("row_begin", ctypes.c_int32), ("row_end", ctypes.c_int32), ("rs", ctypes.c_void_p),
                ("ag", ctypes.c_void_p), ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("stream", ctypes.c_void_p), ("Gs", ctypes.c_void_p)]


def _flat_slots(adapters) -> List[Adapter]:
    """adapters[t][s] (one list per task) -> the task-major slot list of mux_linear_args."""
    S = len(adapters[0])
    _need(all(len(a) == S for a in adapters), "every task needs one adapter per slice (rank 0 = none)")
    return [a for per_task in adapters for a in per_task]


# Prepared adapter tables of sliced calls: (id(adapters), K, N, col_off, grads) -> (fingerprint, table).
# The fingerprint (every slot's object, rank, scale and tensor addresses) is ~30 us for 48 slots; the
# per-slot shape checks and the ctypes table (~2 ms together) run only when it changes.
_SLICED_TABLES = {}


def _slots_fingerprint(slots, grads):
    p = lambda t: 0 if t is None else t.data_ptr()  # noqa: E731
    return tuple((id(a), a.rank, a.scale, p(a.A), p(a.B), p(a.dA) if grads else 0, p(a.dB) if grads else 0)
                 for a in slots)


def _sliced_table(adapters, col_off, K, N, grads, dev):
    """The ctypes adapter table of a sliced call, validated once per distinct adapter set."""
    slots = _flat_slots(adapters)
    key = (id(adapters), K, N, tuple(col_off), grads)
    fp = _slots_fingerprint(slots, grads)
    hit = _SLICED_TABLES.get(key)
    if hit is not None and hit[0] == fp:
        return hit[1]
    for t, per_task in enumerate(adapters):
        for s, a in enumerate(per_task):
            if a.rank == 0:
                continue
            ns = col_off[s + 1] - col_off[s]
            _check_mat(f"adapters[{t}][{s}].A", a.A, (a.rank, K), device=dev)
            _check_mat(f"adapters[{t}][{s}].B", a.B, (ns, a.rank), device=dev, dense=False)
            if grads:
                _check_mat(f"adapters[{t}][{s}].dA", a.dA, (a.rank, K), torch.float32, dev)
                _check_mat(f"adapters[{t}][{s}].dB", a.dB, (ns, a.rank), torch.float32, dev)
    tab = _adapter_table(slots, grads)
    if len(_SLICED_TABLES) > 256:
        _SLICED_TABLES.clear()
    _SLICED_TABLES[key] = (fp, tab)
    return tab


def _check_sliced(seg_off, seg_task, adapters, col_off, K, N, rows, r_cap, grads=False, **mats):
    """Host-side checks of a sliced call (the tensors; the adapters are checked by _sliced_table:
    B_{t,s} is [slice width, rank], A_{t,s} [rank, K])."""
    S = len(col_off) - 1
    _need(1 <= S <= MAX_SLICES, f"1..{MAX_SLICES} slices")
    _need(col_off[0] == 0 and col_off[-1] == N, f"col_off must run from 0 to N={N}")
    dev = None
    for name, (t, shape, dt) in mats.items():
        if t is not None:
            dev = t.device if dev is None else dev
            _check_mat(name, t, shape, dt, dev)
    _need(isinstance(seg_off, torch.Tensor) and seg_off.dtype == torch.int32 and seg_off.is_cuda
          and seg_off.numel() == len(seg_task) + 1, "seg_off must be int32 CUDA [len(seg_task)+1]")


def linear(op: int, seg_off, seg_task, adapters, col_off, K: int, N: int, r_cap: int, max_rows: int, *, X=None,
           W=None, dY=None, Y=None, Hs=None, dX=None, Gs=None, row_begin: int = 0, row_end: int = None, rs=None,
           ag=None, workspace=None, stream=None, want_grads=False):
    """mux_linear: one call of any op over column slices col_off (adapters[t][s]).  Marshalling only."""
    S = len(col_off) - 1
    _need(1 <= S <= MAX_SLICES, f"1..{MAX_SLICES} slices")
    sl = _Slices()
    sl.num_slices = S
    for i, c in enumerate(col_off):
        sl.col_off[i] = int(c)
    tab = _sliced_table(adapters, col_off, K, N, want_grads, seg_off.device)
    st = _i32_host(seg_task)
    if workspace is None:
        dev = seg_off.device
        workspace = torch.zeros(linear_workspace_size(len(seg_task), max_rows, K, N, r_cap * S), dtype=torch.uint8,
                                device=dev)
    a = _LinearArgs()
    a.op, a.num_segs, a.seg_off, a.seg_task = op, len(seg_task), seg_off.data_ptr(), ctypes.addressof(st)
    a.num_adapters, a.adapters, a.slices = len(adapters), ctypes.addressof(tab), ctypes.addressof(sl)
    a.max_rows, a.K, a.N, a.r_cap = max_rows, K, N, r_cap
    for f, t in (("X", X), ("W", W), ("dY", dY), ("Y", Y), ("Hs", Hs), ("dX", dX), ("Gs", Gs)):
        setattr(a, f, None if t is None else t.data_ptr())
    a.row_begin = row_begin
    a.row_end = max_rows if row_end is None else row_end
    a.rs = None if rs is None else ctypes.addressof(rs)
    a.ag = None if ag is None else ctypes.addressof(ag)
    a.workspace, a.workspace_bytes = workspace.data_ptr(), workspace.numel()
    a.stream = _stream(stream).value
    _check(lib().mux_linear(ctypes.byref(a)))
    return workspace


def linear_fwd_sliced(seg_off, seg_task, adapters, X, W, col_off, r_cap: int, Y=None, Hs=None, workspace=None,
                      want_hs: bool = True, stream=None):
    """Fused projection forward: Y[:, slice s] = X W_s^T + s_{t,s} (X A_{t,s}^T) B_{t,s}^T in one GEMM
    (adapters[t][s]; Hs [rows, S * r_cap]).  Returns (Y, Hs)."""
    max_rows, K = X.shape
    N = W.shape[0]
    S = len(col_off) - 1
    if Y is None:
        Y = torch.empty(max_rows, N, dtype=torch.bfloat16, device=X.device)
    if Hs is None and want_hs:
        Hs = torch.empty(max_rows, S * r_cap, dtype=torch.bfloat16, device=X.device)
    _check_sliced(seg_off, seg_task, adapters, col_off, K, N, max_rows, r_cap,
                  X=(X, (max_rows, K), torch.bfloat16), W=(W, (N, K), torch.bfloat16),
                  Y=(Y, (max_rows, N), torch.bfloat16), Hs=(Hs, (max_rows, S * r_cap), torch.bfloat16))
    linear(OP_FWD, seg_off, seg_task, adapters, col_off, K, N, r_cap, max_rows, X=X, W=W, Y=Y, Hs=Hs,
           workspace=workspace, stream=stream)
    return Y, Hs


def linear_bwd_sliced(seg_off, seg_task, adapters, dY, X, W, Hs, col_off, r_cap: int, dX=None, want_dx=True,
                      workspace=None, stream=None, part: int = 0):
    """Fused projection backward (part 0 = all, 1 = dX GEMM, 2 = adapter gradients on the same
    workspace): dX = dY W + sum_s Gs_s A_{t,s}; writes adapters[t][s].dA / .dB (allocated if None)."""
    max_rows, K = X.shape
    N = W.shape[0]
    S = len(col_off) - 1
    dev = X.device
    if dX is None and want_dx and part != BWD_GRADS:
        dX = torch.empty(max_rows, K, dtype=torch.bfloat16, device=dev)
    for per_task in adapters:
        for s, a in enumerate(per_task):
            if a.rank > 0:
                if a.dA is None:
                    a.dA = torch.empty(a.rank, K, dtype=torch.float32, device=dev)
                if a.dB is None:
                    a.dB = torch.empty(col_off[s + 1] - col_off[s], a.rank, dtype=torch.float32, device=dev)
    _check_sliced(seg_off, seg_task, adapters, col_off, K, N, max_rows, r_cap, grads=True,
                  X=(X, (max_rows, K), torch.bfloat16), W=(W, (N, K), torch.bfloat16),
                  dY=(dY, (max_rows, N), torch.bfloat16), dX=(dX, (max_rows, K), torch.bfloat16),
                  Hs=(Hs, (max_rows, S * r_cap), torch.bfloat16))
    op = {0: OP_BWD, BWD_DX: OP_BWD_DX, BWD_GRADS: OP_BWD_GRADS}[part]
    linear(op, seg_off, seg_task, adapters, col_off, K, N, r_cap, max_rows, X=X, W=W, dY=dY, Hs=Hs, dX=dX,
           workspace=workspace, stream=stream, want_grads=True)
    return dX


def linear_shrink_bwd(seg_off, seg_task, adapters, dY, K: int, r_cap: int, row_begin: int = 0, row_end: int = None,
                      Gs=None, col_off=None, workspace=None, stream=None):
    """mux_linear(MUX_OP_SHRINK_BWD): Gs = bf16(s_t dY B_t) for the pair row blocks overlapping
    [row_begin, row_end) (rows outside are not written).  adapters: per task (or [t][s] with col_off).
    Returns Gs [rows, S * r_cap]."""
    max_rows, N = dY.shape
    nested = adapters if col_off is not None else [[a] for a in adapters]
    co = col_off if col_off is not None else [0, N]
    S = len(co) - 1
    if Gs is None:
        Gs = torch.empty(max_rows, S * r_cap, dtype=torch.bfloat16, device=dY.device)
    _check_sliced(seg_off, seg_task, nested, co, K, N, max_rows, r_cap,
                  dY=(dY, (max_rows, N), torch.bfloat16), Gs=(Gs, (max_rows, S * r_cap), torch.bfloat16))
    linear(OP_SHRINK_BWD, seg_off, seg_task, nested, co, K, N, r_cap, max_rows, dY=dY, Gs=Gs, row_begin=row_begin,
           row_end=max_rows if row_end is None else row_end, workspace=workspace, stream=stream)
    return Gs


def linear_bwd_gs(seg_off, seg_task, adapters, dY, X, W, Hs, Gs, r_cap: int, dX=None, col_off=None,
                  workspace=None, stream=None, part: int = 0):
    """mux_linear backward with Gs given (no shrink tiles; e.g. all-gathered rows of a row-parallel
    layer's Gs): dX = dY W + Gs A_t, dA_t = Gs^T X, dB_t = dY^T Hs.  Returns dX."""
    max_rows, K = X.shape
    N = W.shape[0]
    nested = adapters if col_off is not None else [[a] for a in adapters]
    co = col_off if col_off is not None else [0, N]
    if dX is None and part != BWD_GRADS:
        dX = torch.empty(max_rows, K, dtype=torch.bfloat16, device=X.device)
    for s_, per_task in enumerate(zip(*nested)):
        for a in per_task:
            if a.rank > 0:
                if a.dA is None:
                    a.dA = torch.empty(a.rank, K, dtype=torch.float32, device=X.device)
                if a.dB is None:
                    a.dB = torch.empty(co[s_ + 1] - co[s_], a.rank, dtype=torch.float32, device=X.device)
    S = len(co) - 1
    _check_sliced(seg_off, seg_task, nested, co, K, N, max_rows, r_cap, grads=True,
                  X=(X, (max_rows, K), torch.bfloat16), W=(W, (N, K), torch.bfloat16),
                  dY=(dY, (max_rows, N), torch.bfloat16), dX=(dX, (max_rows, K), torch.bfloat16),
                  Hs=(Hs, (max_rows, S * r_cap), torch.bfloat16), Gs=(Gs, (max_rows, S * r_cap), torch.bfloat16))
    op = {0: OP_BWD, BWD_DX: OP_BWD_DX, BWD_GRADS: OP_BWD_GRADS}[part]
    linear(op, seg_off, seg_task, nested, co, K, N, r_cap, max_rows, X=X, W=W, dY=dY, Hs=Hs, dX=dX, Gs=Gs,
           workspace=workspace, stream=stream, want_grads=True)
    return dX


# ---------------------------------------------------------------- decoder-block ops (NEXT-3)
def _ld(t: torch.Tensor) -> int:
    """row stride (elements) of a 2D bf16 view whose rows are contiguous."""
    assert t.dim() == 2 and t.stride(1) == 1, "rows must be contiguous"
    return int(t.stride(0))


def row_start(seq_len: torch.Tensor, seq_row: torch.Tensor, max_rows: int, out: torch.Tensor = None,
              stream=None) -> torch.Tensor:
    """mux_pack_row_start: first packed row of each row's sequence (-1 = pad)."""
    if out is None:
        out = torch.empty(max_rows, dtype=torch.int32, device=seq_len.device)
    _check(lib().mux_pack_row_start(seq_len.numel(), _ptr(seq_len), _ptr(seq_row), max_rows, _ptr(out),
                                    _stream(stream)))
    return out


def attn_fwd(q, k, v, row_start_, heads: int, kv_heads: int, scale: float, o=None, lse=None, stream=None):
    """mux_attn_fwd on 2D views q [R, H*128], k/v [R, Hkv*128] -> (o, lse)."""
    R = q.shape[0]
    if o is None:
        o = torch.empty(R, heads * 128, dtype=torch.bfloat16, device=q.device)
    if lse is None:
        lse = torch.empty(R, heads, dtype=torch.float32, device=q.device)
    _check(lib().mux_attn_fwd(R, heads, kv_heads, 128, _ptr(q), _ld(q), _ptr(k), _ld(k), _ptr(v), _ld(v),
                              _ptr(row_start_), scale, _ptr(o), _ld(o), _ptr(lse), _stream(stream)))
    return o, lse


def attn_workspace_size(rows: int, heads: int) -> int:
    return int(lib().mux_attn_workspace_size(rows, heads))


def attn_bwd(dO, q, k, v, o, lse, row_start_, heads: int, kv_heads: int, scale: float, dq=None, dk=None, dv=None,
             workspace=None, stream=None):
    """mux_attn_bwd -> (dq, dk, dv)."""
    R = q.shape[0]
    dev = q.device
    if dq is None:
        dq = torch.empty(R, heads * 128, dtype=torch.bfloat16, device=dev)
    if dk is None:
        dk = torch.empty(R, kv_heads * 128, dtype=torch.bfloat16, device=dev)
    if dv is None:
        dv = torch.empty(R, kv_heads * 128, dtype=torch.bfloat16, device=dev)
    if workspace is None:
        workspace = torch.empty(attn_workspace_size(R, heads), dtype=torch.uint8, device=dev)
    _check(lib().mux_attn_bwd(R, heads, kv_heads, 128, _ptr(dO), _ld(dO), _ptr(q), _ld(q), _ptr(k), _ld(k),
                              _ptr(v), _ld(v), _ptr(o), _ld(o), _ptr(lse), _ptr(row_start_), scale,
                              _ptr(dq), _ld(dq), _ptr(dk), _ld(dk), _ptr(dv), _ld(dv), _ptr(workspace),
                              workspace.numel(), _stream(stream)))
    return dq, dk, dv


def rope_(x, row_start_, heads: int, head_dim: int = 128, base: float = 10000.0, inverse: bool = False,
          stream=None):
    """mux_rope, in place on x [R, heads*head_dim] (a 2D view, rows contiguous)."""
    _check(lib().mux_rope(x.shape[0], heads, head_dim, _ptr(x), _ld(x), _ptr(row_start_), base, int(inverse),
                          _stream(stream)))
    return x


def rmsnorm_fwd(x, w, eps: float, y=None, res=None, xsum=None, stream=None):
    """mux_rmsnorm_fwd: y = RMSNorm(x [+ res]) * w; with res, x + res is also written to xsum."""
    if y is None:
        y = torch.empty(x.shape[0], x.shape[1], dtype=torch.bfloat16, device=x.device)
    if res is not None and xsum is None:
        xsum = torch.empty(x.shape[0], x.shape[1], dtype=torch.bfloat16, device=x.device)
    _check(lib().mux_rmsnorm_fwd(x.shape[0], x.shape[1], _ptr(x), _ld(x), _ptr(res), _ld(res) if res is not None else 0,
                                 _ptr(xsum), _ld(xsum) if xsum is not None else 0, _ptr(w), eps, _ptr(y), _ld(y),
                                 _stream(stream)))
    return y if res is None else (y, xsum)


def rmsnorm_bwd(dy, x, w, eps: float, dx=None, dy2=None, dy3=None, resid=None, stream=None):
    """mux_rmsnorm_bwd: dx = RMSNorm'(x)^T ((dy [+ dy2 [+ dy3]]) * w) [+ resid]."""
    if dx is None:
        dx = torch.empty(x.shape[0], x.shape[1], dtype=torch.bfloat16, device=x.device)
    ld = lambda t: _ld(t) if t is not None else 0  # noqa: E731
    _check(lib().mux_rmsnorm_bwd(x.shape[0], x.shape[1], _ptr(dy), _ld(dy), _ptr(dy2), ld(dy2), _ptr(dy3), ld(dy3),
                                 _ptr(x), _ld(x), _ptr(w), eps, _ptr(resid), ld(resid), _ptr(dx), _ld(dx),
                                 _stream(stream)))
    return dx


def swiglu_fwd(g, u, h=None, stream=None):
    if h is None:
        h = torch.empty(g.shape[0], g.shape[1], dtype=torch.bfloat16, device=g.device)
    _check(lib().mux_swiglu_fwd(g.shape[0], g.shape[1], _ptr(g), _ld(g), _ptr(u), _ld(u), _ptr(h), _ld(h),
                                _stream(stream)))
    return h


def swiglu_bwd(dh, g, u, dg=None, du=None, stream=None):
    if dg is None:
        dg = torch.empty(g.shape[0], g.shape[1], dtype=torch.bfloat16, device=g.device)
    if du is None:
        du = torch.empty(g.shape[0], g.shape[1], dtype=torch.bfloat16, device=g.device)
    _check(lib().mux_swiglu_bwd(g.shape[0], g.shape[1], _ptr(dh), _ld(dh), _ptr(g), _ld(g), _ptr(u), _ld(u),
                                _ptr(dg), _ld(dg), _ptr(du), _ld(du), _stream(stream)))
    return dg, du


def add(a, b, y=None, stream=None):
    """mux_add: y = a + b (y may alias a or b)."""
    if y is None:
        y = torch.empty(a.shape[0], a.shape[1], dtype=torch.bfloat16, device=a.device)
    _check(lib().mux_add(a.shape[0], a.shape[1], _ptr(a), _ld(a), _ptr(b), _ld(b), _ptr(y), _ld(y),
                         _stream(stream)))
    return y


# ---------------------------------------------------------------- fused GEMM -> reduce-scatter
RS_MAX_WORLD = 8


class _Rs(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("rows_per_rank", ctypes.c_int32),
                ("seq", ctypes.c_uint64), ("recv", ctypes.c_void_p * RS_MAX_WORLD),
                ("flags", ctypes.c_void_p * RS_MAX_WORLD)]


def rs_flags_elems(world: int) -> int:
    return int(lib().mux_rs_flags_elems(world))


def make_rs(world: int, rank: int, rows_per_rank: int, seq: int, recv: Sequence, flags: Sequence) -> _Rs:
    """mux_rs descriptor: recv[d] / flags[d] are rank d's receive buffer and flag block — tensors on
    this device, or raw (peer-mapped) device addresses: [world * rows_per_rank * cols] bf16 and
    [rs_flags_elems(world)] int64, zeroed once."""
    r = _Rs()
    r.world, r.rank, r.rows_per_rank, r.seq = world, rank, rows_per_rank, seq
    for d in range(world):
        r.recv[d] = recv[d] if isinstance(recv[d], int) else recv[d].data_ptr()
        r.flags[d] = flags[d] if isinstance(flags[d], int) else flags[d].data_ptr()
    return r


def linear_fwd_rs(rs: _Rs, seg_off, seg_task, adapters, X, W, r_cap: int, Hs=None, workspace=None, stream=None):
    """mux_linear_fwd_rs: forward whose output rows go straight to their owner ranks."""
    max_rows, K = X.shape
    N = W.shape[0]
    if Hs is None:
        Hs = torch.empty(max_rows, r_cap, dtype=torch.bfloat16, device=X.device)
    _check_linear(seg_off, seg_task, adapters, X, W, r_cap, Hs=Hs)
    _need(max_rows == rs.world * rs.rows_per_rank, "X rows must equal world * rows_per_rank")
    S = len(seg_task)
    if workspace is None:
        workspace = torch.zeros(linear_workspace_size(S, max_rows, K, N, r_cap), dtype=torch.uint8, device=X.device)
    _check(lib().mux_linear_fwd_rs(S, _ptr(seg_off), _i32_host(seg_task), len(adapters),
                                   _adapter_table(adapters, False), max_rows, K, N, r_cap, _ptr(X), _ptr(W),
                                   _ptr(Hs), ctypes.byref(rs), _ptr(workspace), workspace.numel(), _stream(stream)))
    return Hs


def linear_bwd_dx_rs(rs: _Rs, seg_off, seg_task, adapters, dY, X, W, Hs, r_cap: int, workspace, stream=None):
    """mux_linear_bwd_dx_rs: the dX GEMM whose output rows go straight to their owner ranks
    (follow with linear_bwd(..., part=BWD_GRADS) on the same workspace for dA/dB)."""
    max_rows, K = X.shape
    N = W.shape[0]
    _check_linear(seg_off, seg_task, adapters, X, W, r_cap, Hs=Hs, dY=dY)
    _need(max_rows == rs.world * rs.rows_per_rank, "X rows must equal world * rows_per_rank")
    _check(lib().mux_linear_bwd_dx_rs(len(seg_task), _ptr(seg_off), _i32_host(seg_task), len(adapters),
                                      _adapter_table(adapters, True), max_rows, K, N, r_cap, _ptr(dY), _ptr(X),
                                      _ptr(W), _ptr(Hs), ctypes.byref(rs), _ptr(workspace), workspace.numel(),
                                      _stream(stream)))


def rs_reduce(rs: _Rs, out: torch.Tensor, stream=None) -> torch.Tensor:
    """mux_rs_reduce: out [rows_per_rank, cols] = sum of the world partial slots (owner side)."""
    _check(lib().mux_rs_reduce(ctypes.byref(rs), out.shape[1], _ptr(out), _ld(out), _stream(stream)))
    return out


# ---------------------------------------------------------------- fused all-gather -> GEMM
make_ag = make_rs   # same descriptor layout: recv[d] = rank d's gather buffer


def ag_push(ag: _Rs, rows: torch.Tensor, stream=None):
    """mux_ag_push: copy this rank's rows [rows_per_rank, cols] into every rank's gather buffer
    (copy engines) and signal each destination."""
    _check(lib().mux_ag_push(ctypes.byref(ag), _ptr(rows), _ld(rows), rows.shape[1], _stream(stream)))


def ag_release(ag: _Rs, stream=None):
    """mux_ag_release: this rank is done with its gather buffer for call ag.seq."""
    _check(lib().mux_ag_release(ctypes.byref(ag), _stream(stream)))


def linear_fwd_ag(ag: _Rs, seg_off, seg_task, adapters, K: int, W, r_cap: int, Y=None, Hs=None, workspace=None,
                  stream=None):
    """mux_linear_fwd_ag: forward on the gather buffer (rows read as they land)."""
    max_rows = ag.world * ag.rows_per_rank
    N = W.shape[0]
    dev = W.device
    if Y is None:
        Y = torch.empty(max_rows, N, dtype=torch.bfloat16, device=dev)
    if Hs is None:
        Hs = torch.empty(max_rows, r_cap, dtype=torch.bfloat16, device=dev)
    _check_linear(seg_off, seg_task, adapters, None, W, r_cap, K=K, rows=max_rows, Y=Y, Hs=Hs)
    S = len(seg_task)
    if workspace is None:
        workspace = torch.zeros(linear_workspace_size(S, max_rows, K, N, r_cap), dtype=torch.uint8, device=dev)
    _check(lib().mux_linear_fwd_ag(S, _ptr(seg_off), _i32_host(seg_task), len(adapters),
                                   _adapter_table(adapters, False), max_rows, K, N, r_cap, ctypes.byref(ag),
                                   _ptr(W), _ptr(Y), _ptr(Hs), _ptr(workspace), workspace.numel(), _stream(stream)))
    return Y, Hs


def linear_bwd_ag(ag: _Rs, seg_off, seg_task, adapters, X, W, Hs, r_cap: int, dX=None, workspace=None,
                  stream=None):
    """mux_linear_bwd_ag: backward with dY = the gather buffer (rows read as they land)."""
    max_rows, K = X.shape
    N = W.shape[0]
    dev = X.device
    if dX is None:
        dX = torch.empty(max_rows, K, dtype=torch.bfloat16, device=dev)
    for a in adapters:
        if a.rank > 0:
            if a.dA is None:
                a.dA = torch.empty(a.rank, K, dtype=torch.float32, device=dev)
            if a.dB is None:
                a.dB = torch.empty(N, a.rank, dtype=torch.float32, device=dev)
    _check_linear(seg_off, seg_task, adapters, X, W, r_cap, Hs=Hs, dX=dX, grads=True)
    _need(max_rows == ag.world * ag.rows_per_rank, "X rows must equal world * rows_per_rank")
    S = len(seg_task)
    if workspace is None:
        workspace = torch.zeros(linear_workspace_size(S, max_rows, K, N, r_cap), dtype=torch.uint8, device=dev)
    _check(lib().mux_linear_bwd_ag(S, _ptr(seg_off), _i32_host(seg_task), len(adapters),
                                   _adapter_table(adapters, True), max_rows, K, N, r_cap, ctypes.byref(ag),
                                   _ptr(X), _ptr(W), _ptr(Hs), _ptr(dX), _ptr(workspace), workspace.numel(),
                                   _stream(stream)))
    return dX


# ---------------------------------------------------------------- NVLS (in-switch) collectives
class _Nvls(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("rows_per_rank", ctypes.c_int32),
                ("seq", ctypes.c_uint64), ("uc_buf", ctypes.c_void_p), ("mc_buf", ctypes.c_void_p),
                ("uc_flags", ctypes.c_void_p), ("mc_flags", ctypes.c_void_p)]


def make_nvls(world: int, rank: int, rows_per_rank: int, seq: int, uc_buf: int, mc_buf: int, uc_flags: int,
              mc_flags: int) -> _Nvls:
    """mux_nvls descriptor (raw device addresses: this rank's copy and the multicast address)."""
    d = _Nvls()
    d.world, d.rank, d.rows_per_rank, d.seq = world, rank, rows_per_rank, seq
    d.uc_buf, d.mc_buf, d.uc_flags, d.mc_flags = uc_buf, mc_buf, uc_flags, mc_flags
    return d


def nvls_flags_elems() -> int:
    return int(lib().mux_nvls_flags_elems())


def nvls_reduce_scatter(nv: _Nvls, out: torch.Tensor, ctas: int = 0, stream=None) -> torch.Tensor:
    """mux_nvls_reduce_scatter: out [rows_per_rank, cols] = in-switch sum of every rank's rows."""
    _need(out.dtype == torch.bfloat16 and out.dim() == 2 and out.shape[0] == nv.rows_per_rank,
          "out must be bf16 [rows_per_rank, cols]")
    _check(lib().mux_nvls_reduce_scatter(ctypes.byref(nv), out.shape[1], _ptr(out), _ld(out), ctas, _stream(stream)))
    return out


def nvls_all_gather(nv: _Nvls, rows: torch.Tensor, ctas: int = 0, stream=None):
    """mux_nvls_all_gather: this rank's rows [rows_per_rank, cols] into every rank's copy."""
    _need(rows.dtype == torch.bfloat16 and rows.dim() == 2 and rows.shape[0] == nv.rows_per_rank,
          "rows must be bf16 [rows_per_rank, cols]")
    _check(lib().mux_nvls_all_gather(ctypes.byref(nv), _ptr(rows), _ld(rows), rows.shape[1], ctas, _stream(stream)))


def nvls_release(nv: _Nvls, stream=None):
    """mux_nvls_release: this rank is done reading the last all-gather's buffer."""
    _check(lib().mux_nvls_release(ctypes.byref(nv), _stream(stream)))
