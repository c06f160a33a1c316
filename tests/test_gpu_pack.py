"""GPU parity: mux_pack_chunks / mux_pack_apply vs the pack oracle — bit-exact."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import synth  # noqa: E402
from oracle import pack as opk  # noqa: E402
from paper_2603_02885_b200 import mux  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gpu_pack(off, lens, cap, chunk_size, chunk_min, max_rows, max_chunks):
    o = mux.pack_chunks(off, lens, cap, chunk_size, chunk_min, max_rows=max_rows, max_chunks=max_chunks)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in o.items() if k != "workspace"}, mux.read_info(o["info"])


def _check(off, lens, cap=None, chunk_size=0, chunk_min=64, slack_rows=64, slack_chunks=3):
    ref = opk.pack_chunks(off, lens, cap, chunk_size, chunk_min)
    assert ref["status"] == 0
    R = ref["info"]["total_rows"]
    C = ref["info"]["num_chunks"]
    max_rows, max_chunks = R + slack_rows, C + slack_chunks
    ref = opk.pack_chunks(off, lens, cap, chunk_size, chunk_min, max_rows=max_rows, max_chunks=max_chunks)
    g, info = _gpu_pack(off, lens, cap, chunk_size, chunk_min, max_rows, max_chunks)
    for k in ("chunk_size", "num_chunks", "num_packs", "total_rows", "valid_rows", "zero_pad_rows",
              "overflow"):
        assert info[k] == ref["info"][k], (k, info[k], ref["info"][k])
    M = len(off) - 1
    S = len(lens)
    assert np.array_equal(g["seg_off"][: M + 1], ref["seg_off"])
    assert np.array_equal(g["seq_row"][:S], ref["seq_row"])
    for k in ("chunk_task", "chunk_pack", "chunk_valid", "chunk_dep"):
        assert np.array_equal(g[k][:C], ref[k]), k
    assert np.array_equal(g["row_src"][:max_rows], ref["row_src"])
    return ref


def test_fixture_P1():
    gld = json.load(open(os.path.join(GOLD, "pack_P1.json")))
    _check(gld["task_seq_off"], gld["seq_len"], gld["pack_capacity"], 0, 64)


@pytest.mark.parametrize("cid", ["1", "2", "3a", "3b", "3c", "4", "5"])
def test_configs(cid):
    wl = synth.workload(cid)
    off, lens = wl.csr()
    _check(list(off), list(lens), wl.pack_capacity, wl.chunk_size, wl.chunk_min)


def test_random_and_edges():
    rng = np.random.default_rng(7)
    for it in range(30):
        M = int(rng.integers(1, 9))
        lens_t = [rng.integers(1, 700, size=int(rng.integers(0, 40))).astype(np.int32) for _ in range(M)]
        off = [0]
        for x in lens_t:
            off.append(off[-1] + len(x))
        lens = [int(v) for x in lens_t for v in x]
        cmin = int(rng.choice([64, 128]))
        csz = int(rng.choice([0, 0, 64, 256]))
        cap = None if it % 2 else [int(max(list(x) + [1])) + int(rng.integers(0, 300)) for x in lens_t]
        _check(off, lens, cap, csz, cmin)


def test_many_sequences_one_task():
    rng = np.random.default_rng(8)
    lens = [int(x) for x in rng.integers(1, 512, size=2000)]
    _check([0, 2000], lens, [512], 0, 64)


def test_overflow_flags():
    off, lens = [0, 2], [64, 64]
    g, info = _gpu_pack(off, lens, [64], 0, 64, max_rows=64, max_chunks=8)
    assert info["overflow"] & 1
    g, info = _gpu_pack(off, lens, [64], 0, 64, max_rows=512, max_chunks=1)
    assert info["overflow"] & 2


def test_invalid_device_data_flag():
    g, info = _gpu_pack([0, 1], [100], [64], 0, 64, max_rows=256, max_chunks=8)   # cap < len
    assert info["overflow"] & 4
    g, info = _gpu_pack([0, 2], [5, 0], None, 0, 64, max_rows=256, max_chunks=8)  # len 0
    assert info["overflow"] & 4


def test_pack_apply_gather():
    wl = synth.workload("2")
    off, lens = wl.csr()
    ref = opk.pack_chunks(off, lens, wl.pack_capacity, 0, 64)
    R = ref["info"]["total_rows"]
    T = wl.valid_tokens
    tok = synth.token_input(wl, 0, "X", 256)
    expect = np.zeros((R + 64, 256), np.uint16)
    rs = np.concatenate([ref["row_src"], np.full(64, -1, np.int32)])
    expect[rs >= 0] = tok[rs[rs >= 0]]
    src = torch.from_numpy(tok.view(np.int16)).cuda().view(torch.bfloat16)
    o = mux.pack_chunks(list(off), list(lens), wl.pack_capacity, 0, 64, max_rows=R + 64,
                        max_chunks=ref["info"]["num_chunks"] + 1)
    packed = mux.pack_apply(o["row_src"], src, R + 64)
    torch.cuda.synchronize()
    got = packed.view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got, expect)
    assert T == int((rs >= 0).sum())


def test_no_sequences_at_all():
    """Degenerate micro-batch: every task empty (num_seqs = 0): c = chunk_min, total_rows = 0,
    seg_off all zero, every row_src entry -1 — bit-exact with the oracle."""
    _check([0, 0, 0, 0], [], None, 0, 64)
    _check([0, 0], [], [128], 0, 128)
