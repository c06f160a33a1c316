"""Pack oracle: chunk-based data alignment, written step by step from the paper.

ORACLE — test infrastructure only (see oracle/__init__.py).

Paper: P:833-843 (§3.5 "Reinventing Packing with Chunk-Based Alignment"):
  step 1 "adaptively packs sequences within a single global batch for each
          task, respectively"
  step 2 "uniformly partitions packed sequences into equal-sized chunks ...
          For sequences longer than the chunk size ... scatters them across
          multiple consecutive chunks with the dependency of KV cache reuse"
                                                                
  chunk  "greatest power-of-2 divisor of all sequence lengths, with a minimum
          threshold (typically 64)"
Readings where the paper is silent (SURVEY §8(c) Q4/Q5/
Q16/Q17): FFD with ties broken by caller index; default capacity
round_up(max(max len_t, c), c); task-major then pack-creation order; one
chunk size per call; a task may have zero sequences.
"""
from __future__ import annotations

import numpy as np

MUX_OK = 0
MUX_ERR_INVALID_ARGUMENT = 1


def _v2(x: int) -> int:
    """2-adic valuation of x >= 1 (exponent of the largest power of 2 dividing x)."""
    v = 0
    while x % 2 == 0:
        x //= 2
        v += 1
    return v


def _is_pow2(x: int) -> bool:
    return x >= 1 and (x & (x - 1)) == 0


def choose_chunk_size(seq_len, chunk_size: int = 0, chunk_min: int = 64) -> int:
    """c = max(chunk_min, 2^{min_s v2(len_s)}), or the caller's value."""
    if chunk_size != 0:
        return chunk_size
    if len(seq_len) == 0:
        return chunk_min
    g = min(_v2(int(L)) for L in seq_len)
    return max(chunk_min, 2 ** g)


def ffd(lengths, capacity: int):
    """First-fit decreasing of one task's sequences (reading Q5).

    Visit order: length descending, caller index ascending. Each sequence goes
    into the lowest-index open pack whose residual >= its length, else a new
    pack. Returns (pack_of[i], offset_of[i], pack_lengths)."""
    n = len(lengths)
    order = sorted(range(n), key=lambda i: (-int(lengths[i]), i))
    residual = []
    members = []
    pack_of = [-1] * n
    for i in order:
        L = int(lengths[i])
        for p in range(len(residual)):
            if residual[p] >= L:
                break
        else:
            residual.append(capacity)
            members.append([])
            p = len(residual) - 1
        residual[p] -= L
        members[p].append(i)
        pack_of[i] = p
    offset_of = [0] * n
    pack_len = []
    for p, mem in enumerate(members):           # members in insertion order
        off = 0
        for i in mem:
            offset_of[i] = off
            off += int(lengths[i])
        pack_len.append(off)
    return pack_of, offset_of, pack_len


def pack_chunks(task_seq_off, seq_len, pack_capacity=None, chunk_size: int = 0,
                chunk_min: int = 64, max_rows: int = None, max_chunks: int = None):
    """Full mux_pack_chunks semantics. Returns dict with
    status, seg_off, seq_row, chunk_task, chunk_pack, chunk_valid, chunk_dep,
    row_src (length max_rows, -1 = pad/unused) and info fields."""
    task_seq_off = [int(x) for x in task_seq_off]
    seq_len = [int(x) for x in seq_len]
    M = len(task_seq_off) - 1
    S = len(seq_len)
    # ---- step 1: validate
    if M < 1 or task_seq_off[0] != 0 or task_seq_off[M] != S:
        return {"status": MUX_ERR_INVALID_ARGUMENT}
    if any(task_seq_off[t + 1] < task_seq_off[t] for t in range(M)):
        return {"status": MUX_ERR_INVALID_ARGUMENT}
    if any(L < 1 for L in seq_len):
        return {"status": MUX_ERR_INVALID_ARGUMENT}
    if not (_is_pow2(chunk_min) and chunk_min >= 64):
        return {"status": MUX_ERR_INVALID_ARGUMENT}
    if chunk_size != 0 and not (_is_pow2(chunk_size) and chunk_size >= 64):
        return {"status": MUX_ERR_INVALID_ARGUMENT}
    # ---- step 2: chunk size
    c = choose_chunk_size(seq_len, chunk_size, chunk_min)
    # ---- step 3/4: per-task FFD
    chunks = []          # (task, pack, valid, dep)
    pack_row0 = {}       # (task, pack) -> first row
    per_task = []
    num_packs = 0
    for t in range(M):
        lens_t = seq_len[task_seq_off[t]:task_seq_off[t + 1]]
        max_len = max(lens_t) if lens_t else 0
        if pack_capacity is None:
            cap = -(-max(max_len, c) // c) * c
        else:
            cap = int(pack_capacity[t])
            if cap < max_len:
                return {"status": MUX_ERR_INVALID_ARGUMENT}
        pack_of, offset_of, pack_len = ffd(lens_t, cap) if lens_t else ([], [], [])
        per_task.append((pack_of, offset_of, pack_len))
        num_packs += len(pack_len)
    # ---- step 5: chunks, task-major, pack-creation order
    seg_off = [0] * (M + 1)
    for t in range(M):
        seg_off[t] = len(chunks) * c
        _, _, pack_len = per_task[t]
        for p, L in enumerate(pack_len):
            n_p = -(-L // c)
            pack_row0[(t, p)] = len(chunks) * c
            for j in range(n_p):
                cid = len(chunks)
                chunks.append((t, p, min(c, L - j * c), cid - 1 if j > 0 else -1))
    seg_off[M] = len(chunks) * c
    total_rows = seg_off[M]
    valid_rows = sum(seq_len)
    if max_rows is None:
        max_rows = total_rows
    if max_chunks is None:
        max_chunks = len(chunks)
    zero_pad_rows = (max(seq_len) * S) if S else 0
    info = {"chunk_size": c, "num_chunks": len(chunks), "num_packs": num_packs,
            "total_rows": total_rows, "valid_rows": valid_rows,
            "zero_pad_rows": zero_pad_rows, "overflow": 0}
    if total_rows > max_rows or len(chunks) > max_chunks:
        info["overflow"] = 1
        return {"status": MUX_OK, "info": info, "overflowed": True}
    # ---- step 6: maps
    tok_off = [0] * (S + 1)
    for s in range(S):
        tok_off[s + 1] = tok_off[s] + seq_len[s]
    seq_row = [0] * S
    row_src = np.full(max_rows, -1, dtype=np.int32)
    for t in range(M):
        pack_of, offset_of, _ = per_task[t]
        for i, s in enumerate(range(task_seq_off[t], task_seq_off[t + 1])):
            seq_row[s] = pack_row0[(t, pack_of[i])] + offset_of[i]
            for pos in range(seq_len[s]):
                row_src[seq_row[s] + pos] = tok_off[s] + pos
    ct = np.array([x[0] for x in chunks], np.int32)
    cp = np.array([x[1] for x in chunks], np.int32)
    cv = np.array([x[2] for x in chunks], np.int32)
    cd = np.array([x[3] for x in chunks], np.int32)
    return {"status": MUX_OK, "overflowed": False, "info": info,
            "seg_off": np.array(seg_off, np.int32), "seq_row": np.array(seq_row, np.int32),
            "chunk_task": ct, "chunk_pack": cp, "chunk_valid": cv, "chunk_dep": cd,
            "row_src": row_src}
