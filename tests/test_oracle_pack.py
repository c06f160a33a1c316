"""Pins for the pack oracle (oracle/pack.py) — against the paper, SPEC's hand
examples, brute force and invariants; never against the oracle itself.

P:n = PAPER.md line, S:n = SPEC.md line (see tests/golden/*.json citations).
"""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import pack as opk
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _csr(task_lens):
    off = [0]
    for x in task_lens:
        off.append(off[-1] + len(x))
    return off, [int(v) for x in task_lens for v in x]


# ---------------------------------------------------------------- chunk rule
@pytest.mark.parametrize("lens,expect", [
    ([64, 128, 256], 64),     # S:461, P:944 padded lengths -> 64
    ([128, 256], 128),
    ([96, 160], 64),          # common 2-power divisor 32 < 64 -> threshold
    ([512], 512),
    ([1024, 512, 2048], 512),
    ([65], 64),
    ([7, 9], 64),
])
def test_chunk_rule_examples(lens, expect):
    assert opk.choose_chunk_size(lens, 0, 64) == expect


def test_chunk_rule_closed_form_random():
    """c = max(64, largest power of two dividing every length),
    checked by enumerating divisors (independent of the v2 loop)."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        lens = list(rng.integers(1, 4096, size=rng.integers(1, 6)))
        best = 1
        for p in range(13):
            if all(L % (2 ** p) == 0 for L in lens):
                best = 2 ** p
        assert opk.choose_chunk_size(lens, 0, 64) == max(64, best)
        assert opk.choose_chunk_size(lens, 0, 128) == max(128, best)


def test_chunk_rule_explicit_overrides():
    # P:1128 used chunk 128 on an SST2(64)+RTE(256) mix: only an explicit value reproduces it.
    assert opk.choose_chunk_size([64, 256], 128, 64) == 128
    assert opk.choose_chunk_size([64, 256], 0, 128) == 128


# ---------------------------------------------------------------- FFD
def test_ffd_spec_example():
    """lengths [40,20,30,30], capacity 64 -> packs [40,20] and [30,30]."""
    pack_of, off, plen = opk.ffd([40, 20, 30, 30], 64)
    packs = {}
    for i, p in enumerate(pack_of):
        packs.setdefault(p, []).append([40, 20, 30, 30][i])
    assert sorted(sorted(v) for v in packs.values()) == [[20, 40], [30, 30]]
    assert plen == [60, 60]


def test_ffd_exact_fit():
    """[64] capacity 64 -> one full pack."""
    pack_of, off, plen = opk.ffd([64], 64)
    assert pack_of == [0] and plen == [64]


def _optimal_bins(lengths, cap):
    """Brute-force optimal bin packing (tiny n): try every assignment."""
    n = len(lengths)
    best = n
    for assign in itertools.product(range(n), repeat=n):
        if max(assign) + 1 >= best:
            continue
        loads = [0] * n
        ok = True
        for i, b in enumerate(assign):
            loads[b] += lengths[i]
            if loads[b] > cap:
                ok = False
                break
        if ok:
            best = max(assign) + 1
    return best


def test_ffd_vs_bruteforce_optimum():
    """ceil(sum/cap) <= FFD count <= 1.23 x optimum (+ a rounding slack of
    one bin for tiny instances, FFD <= 11/9 OPT + 6/9); each pack within capacity."""
    rng = np.random.default_rng(11)
    for _ in range(60):
        n = int(rng.integers(1, 7))
        cap = int(rng.choice([64, 100, 128]))
        lens = [int(x) for x in rng.integers(1, cap + 1, size=n)]
        pack_of, off, plen = opk.ffd(lens, cap)
        nb = len(plen)
        assert all(L <= cap for L in plen)
        assert nb >= -(-sum(lens) // cap)
        opt = _optimal_bins(lens, cap)
        assert nb <= (11 * opt + 6) // 9 + 0 or nb <= 1.23 * opt
        # each sequence placed exactly once, offsets tile each pack
        for p in range(nb):
            mem = sorted((off[i], lens[i]) for i in range(n) if pack_of[i] == p)
            pos = 0
            for o, L in mem:
                assert o == pos
                pos += L
            assert pos == plen[p]


# ---------------------------------------------------------------- golden P1
def test_pack_fixture_P1():
    g = json.load(open(os.path.join(GOLD, "pack_P1.json")))
    r = opk.pack_chunks(g["task_seq_off"], g["seq_len"], g["pack_capacity"], g["chunk_size"],
                        g["chunk_min"], max_rows=256)
    e = g["expect"]
    assert r["status"] == 0
    info = r["info"]
    for k in ("chunk_size", "total_rows", "valid_rows", "num_packs", "num_chunks", "zero_pad_rows"):
        assert info[k] == e[k], k
    for k in ("seg_off", "chunk_task", "chunk_pack", "chunk_valid", "chunk_dep", "seq_row"):
        assert list(r[k]) == e[k], k
    for a, b, v in e["row_src_ranges"]:
        want = np.full(b - a, -1) if v == -1 else np.arange(v, v + b - a)
        assert np.array_equal(r["row_src"][a:b], want)


# ---------------------------------------------------------------- invariants
def _check_invariants(task_lens, r, cap_list=None):
    info = r["info"]
    c = info["chunk_size"]
    off, lens = _csr(task_lens)
    T = sum(lens)
    seg = r["seg_off"]
    assert all(x % c == 0 for x in seg)                          # multiples of c
    assert all(seg[i] <= seg[i + 1] for i in range(len(seg) - 1))
    assert seg[-1] == info["total_rows"] == info["num_chunks"] * c
    rs = r["row_src"]
    valid = rs[rs >= 0]
    assert len(valid) == T == info["valid_rows"]                 # token conservation
    assert np.array_equal(np.sort(valid), np.arange(T))          # bijection onto tokens
    # seq_row consistent with row_src, sequences stay in their task's segment
    tok = 0
    for t in range(len(task_lens)):
        for s in range(off[t], off[t + 1]):
            L = lens[s]
            row = r["seq_row"][s]
            assert np.array_equal(rs[row:row + L], np.arange(tok, tok + L))
            assert seg[t] <= row and row + L <= seg[t + 1]
            tok += L
    # chunk table: valid + pad = c; dep chains disjoint, consecutive ids, one per multi-chunk pack
    cv, cd, ct, cp = r["chunk_valid"], r["chunk_dep"], r["chunk_task"], r["chunk_pack"]
    assert np.all((cv >= 1) & (cv <= c))
    assert int(cv.sum()) == T
    for i in range(len(cv)):
        if cd[i] >= 0:
            assert cd[i] == i - 1 and ct[i] == ct[i - 1] and cp[i] == cp[i - 1]
            assert cv[i - 1] == c                       # only the last chunk of a pack is partial
        if i > 0 and cd[i] < 0:
            assert (ct[i], cp[i]) != (ct[i - 1], cp[i - 1])
    # chunk padding never exceeds zero-padding every sequence to the global max
    # (S:485), both aligned to the chunk size (the unaligned count can be smaller
    # when every sequence has the same non-multiple-of-c length); default capacity.
    if cap_list is None and len(lens):
        aligned_zero_pad = len(lens) * (-(-max(lens) // c) * c)
        assert info["total_rows"] <= aligned_zero_pad


@pytest.mark.parametrize("cid", ["1", "2", "3a", "3b", "3c", "4", "5"])
def test_invariants_on_configs(cid):
    wl = synth.workload(cid)
    off, lens = wl.csr()
    r = opk.pack_chunks(off, lens, wl.pack_capacity, wl.chunk_size, wl.chunk_min)
    assert r["status"] == 0
    _check_invariants(wl.task_lens, r, wl.pack_capacity)
    assert r["info"]["total_rows"] <= r["info"]["zero_pad_rows"]


def test_wlb_prepadded_closed_form():
    """WL-B (tab:workloads P:1042-1046) with pre-padded lengths RTE 256 / SST2 64
    (P:944): every sequence is a whole number of 64-chunks, so packing adds no
    pad: R = sum b_t * l_t = 5504; zero-pad-to-max = 32 * 256 = 8192."""
    wl = synth.workload("3a")
    off, lens = wl.csr()
    r = opk.pack_chunks(off, lens, None, 0, 64)
    assert r["info"]["chunk_size"] == 64
    assert r["info"]["total_rows"] == 5504 == r["info"]["valid_rows"]
    assert r["info"]["zero_pad_rows"] == 8192


def test_random_invariants_and_edges():
    rng = np.random.default_rng(3)
    for it in range(40):
        M = int(rng.integers(1, 6))
        task_lens = []
        for t in range(M):
            n = int(rng.integers(0, 6))          # a task may be empty (Q16)
            task_lens.append(rng.integers(1, 300, size=n).astype(np.int32))
        off, lens = _csr(task_lens)
        cmin = int(rng.choice([64, 128]))
        r = opk.pack_chunks(off, lens, None, 0, cmin)
        assert r["status"] == 0
        if sum(lens) == 0:
            assert r["info"]["total_rows"] == 0
            continue
        _check_invariants(task_lens, r)


def test_empty_task_gets_empty_segment():
    r = opk.pack_chunks([0, 1, 1, 2], [10, 70], None, 0, 64)
    assert list(r["seg_off"]) == [0, 64, 64, 192]


def test_spec_partition_2p5_chunks():
    """a pack of 2.5 chunks -> 3 chunks, 0.5 chunk pad, 2 dependency links."""
    r = opk.pack_chunks([0, 1], [160], None, 64, 64)
    assert list(r["chunk_valid"]) == [64, 64, 32]
    assert list(r["chunk_dep"]) == [-1, 0, 1]
    assert r["info"]["total_rows"] - r["info"]["valid_rows"] == 32


def test_invalid_arguments():
    assert opk.pack_chunks([0, 1], [0], None, 0, 64)["status"] == 1          # len 0
    assert opk.pack_chunks([0, 1], [10], None, 0, 32)["status"] == 1         # chunk_min < 64
    assert opk.pack_chunks([0, 1], [10], None, 96, 64)["status"] == 1        # not a power of 2
    assert opk.pack_chunks([0, 1], [100], [64], 0, 64)["status"] == 1        # cap < len
    assert opk.pack_chunks([0, 2], [10], None, 0, 64)["status"] == 1         # CSR mismatch


def test_overflow_flag():
    r = opk.pack_chunks([0, 2], [64, 64], [64], 0, 64, max_rows=64)
    assert r["info"]["overflow"] == 1 and r["overflowed"]
