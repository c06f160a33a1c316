"""Workload recipes for BASELINE.json's five configs.

Only shapes, sequence-length mixes, ranks, scales and seeds live here; the
packing of those sequences into rows is the method's job (mux_pack_chunks on
the GPU side, oracle.pack on the oracle side).

Citations: P:n = /root/reference/PAPER.md line n.
  * LLaMA-7B/13B hidden sizes: `tab:models` P:896-913; FFN widths 11008/13824
    and the 70B shapes come from BASELINE.json's config strings (public LLaMA-2).
  * WL-B task order and batch sizes: `tab:workloads` P:1037-1048.
  * Padded lengths SST2 64 / QA 128 / RTE 256: P:944.
  * Ranks 4-64: P:294 ("rank <= 64").
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .gen import Stream, seq_lengths, normal, normal_bf16, int_bf16, sparse_int_bf16, bf16_bits_from_f64

CONFIG_IDS = ("1", "2", "3a", "3b", "3c", "4", "5")


def base_seed(config_id: str) -> int:
    """seed = 2603028850 + config number."""
    return 2603028850 + int(config_id[0])


@dataclass
class Linear:
    name: str
    K: int   # in features
    N: int   # out features


@dataclass
class Workload:
    config_id: str
    description: str
    task_lens: List[np.ndarray]        # per task: int32 sequence lengths (caller order)
    ranks: List[int]                   # per task
    scales: List[float]                # per task, s_t
    linears: List[Linear]
    pack_capacity: Optional[List[int]] = None   # None = default rule
    chunk_size: int = 0                # 0 = rule of P:843
    chunk_min: int = 64
    seed: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def num_tasks(self) -> int:
        return len(self.task_lens)

    @property
    def num_seqs(self) -> int:
        return int(sum(len(x) for x in self.task_lens))

    @property
    def valid_tokens(self) -> int:
        return int(sum(int(x.sum()) for x in self.task_lens))

    def csr(self):
        """(task_seq_off[M+1], seq_len[num_seqs]) int32, task-major caller order."""
        off = np.zeros(self.num_tasks + 1, dtype=np.int32)
        for t, x in enumerate(self.task_lens):
            off[t + 1] = off[t] + len(x)
        lens = (np.concatenate(self.task_lens).astype(np.int32)
                if self.num_seqs else np.zeros(0, np.int32))
        return off, lens

    def max_rows_bound(self) -> int:
        """Host-side worst case of packed rows: every sequence in its own pack,
        each rounded up to the chunk size (chunk >= chunk_min)."""
        c = max(self.chunk_size, self.chunk_min)
        cap_round = 0
        for t, x in enumerate(self.task_lens):
            for L in x:
                cap_round += -(-int(L) // c) * c
        return cap_round


# --------------------------------------------------------------------------
def workload(config_id: str, variant: str = "normal") -> Workload:
    seed = base_seed(config_id)
    st = Stream(seed, first=1000)      # stream ids for lengths (tensors use 1..999)
    if config_id == "1":
        lens = [np.array([64], np.int32), np.array([64], np.int32)]
        return Workload("1", "single linear d=256->256, 2 LoRA tasks r=8, 64 tokens each",
                        lens, [8, 8], [2.0, 2.0], [Linear("lin", 256, 256)], seed=seed)
    if config_id == "2":
        lens = [seq_lengths(seed, st.take(), 8, 128, 512) for _ in range(4)]
        return Workload("2", "LLaMA-7B linears 4096->4096/11008, 11008->4096; 4 tasks r=16; "
                        "8 seqs/task len U{128..512}, cap 512",
                        lens, [16] * 4, [2.0] * 4,
                        [Linear("qo_4096x4096", 4096, 4096), Linear("up_4096x11008", 4096, 11008),
                         Linear("down_11008x4096", 11008, 4096)],
                        pack_capacity=[512] * 4, seed=seed)
    if config_id.startswith("3"):
        # WL-B (tab:workloads): RTE, SST2, RTE, SST2, SST2, RTE, RTE, RTE
        datasets = ["RTE", "SST2", "RTE", "SST2", "SST2", "RTE", "RTE", "RTE"]
        bsz = [4, 2, 4, 4, 8, 2, 4, 4]
        ranks = [4, 8, 16, 32, 64, 16, 8, 64]
        padded = {"RTE": 256, "SST2": 64}
        raw = {"RTE": (16, 256), "SST2": (8, 64)}
        mult = 4 if config_id == "3c" else 1
        lens = []
        for t, (d, b) in enumerate(zip(datasets, bsz)):
            n = b * mult
            if config_id == "3b":
                lo, hi = raw[d]
                lens.append(seq_lengths(seed, st.take(), n, lo, hi))
            else:
                lens.append(np.full(n, padded[d], np.int32))
        desc = {"3a": "pre-padded 256/64", "3b": "raw lengths (alignment stress)",
                "3c": "pre-padded, x4 batch"}[config_id]
        return Workload(config_id, "LLaMA-13B linears 5120->5120/13824, 13824->5120; WL-B 8 tasks "
                        "ranks 4..64; " + desc, lens, ranks, [2.0] * 8,
                        [Linear("qo_5120x5120", 5120, 5120), Linear("up_5120x13824", 5120, 13824),
                         Linear("down_13824x5120", 13824, 5120)], seed=seed)
    if config_id == "4":
        lens = [seq_lengths(seed, st.take(), 4, 128, 512) for _ in range(16)]
        ranks = [(8, 16, 32, 64)[t % 4] for t in range(16)]
        lin = [Linear("q", 4096, 4096), Linear("k", 4096, 4096), Linear("v", 4096, 4096),
               Linear("o", 4096, 4096), Linear("gate", 4096, 11008), Linear("up", 4096, 11008),
               Linear("down", 11008, 4096)]
        return Workload("4", "LLaMA-7B decoder-block linears (q,k,v,o,gate,up,down), 16 tasks",
                        lens, ranks, [2.0] * 16, lin, pack_capacity=[512] * 16, seed=seed)
    if config_id == "5":
        lens = [seq_lengths(seed, st.take(), 2, 128, 512) for _ in range(32)]
        ranks = [(4, 8, 16, 32, 64)[t % 5] for t in range(32)]
        lin = [Linear("q", 8192, 8192), Linear("k", 8192, 1024), Linear("v", 8192, 1024),
               Linear("o", 8192, 8192), Linear("gate", 8192, 28672), Linear("up", 8192, 28672),
               Linear("down", 28672, 8192)]
        return Workload("5", "LLaMA-70B-shaped linears, 32 tasks mixed rank", lens, ranks,
                        [2.0] * 32, lin, pack_capacity=[512] * 32, seed=seed)
    raise KeyError(config_id)


# --------------------------------------------------------------------------
# Tensor recipes.  Stream ids: per linear index li, per task t.
def _sid(li: int, what: int, t: int = 0) -> int:
    return 1 + li * 4096 + what * 256 + t


def token_input(wl: Workload, li: int, which: str, cols: int, variant: str = "normal"):
    """Token-major tensor [T_valid, cols] (X: which='X', dY: which='dY')."""
    T = wl.valid_tokens
    w = {"X": 0, "dY": 1}[which]
    if variant == "int":
        return int_bf16(wl.seed, _sid(li, w), (T, cols), -4, 4)
    return normal_bf16(wl.seed, _sid(li, w), (T, cols), 1.0)


def weight(wl: Workload, li: int, variant: str = "normal"):
    """Backbone W [N, K] ~ N(0, 1/K)  (nn.Linear layout)."""
    L = wl.linears[li]
    if variant == "int":
        return int_bf16(wl.seed, _sid(li, 2), (L.N, L.K), -4, 4)
    return normal_bf16(wl.seed, _sid(li, 2), (L.N, L.K), 1.0 / np.sqrt(L.K))


def adapter(wl: Workload, li: int, t: int, variant: str = "normal"):
    """(A_t [r, K] ~ N(0,1/K), B_t [N, r] ~ N(0, 1/r)); variant 'zeroB' gives
    B_t = 0 (LoRA initialisation); 'int' gives sparse integers."""
    L = wl.linears[li]
    r = wl.ranks[t]
    if variant == "int":
        A = sparse_int_bf16(wl.seed, _sid(li, 3, t), (r, L.K), 8, 1, -2, 2)
        B = sparse_int_bf16(wl.seed, _sid(li, 4, t), (L.N, r), 8, 0, -2, 2)
        return A, B
    A = normal_bf16(wl.seed, _sid(li, 3, t), (r, L.K), 1.0 / np.sqrt(L.K))
    if variant == "zeroB":
        B = np.zeros((L.N, r), np.uint16)
    else:
        B = normal_bf16(wl.seed, _sid(li, 4, t), (L.N, r), 1.0 / np.sqrt(max(r, 1)))
    return A, B


def int_scales(wl: Workload):
    """s in {1,2} for the integer fixture."""
    return [float(1 + (t % 2)) for t in range(wl.num_tasks)]


def norm_weight(wl: Workload, i: int):
    """RMSNorm weight [hidden] of the decoder block (i = 0: before attention,
    1: before the MLP) ~ N(1, 0.1^2) (a trained norm's scale sits near 1)."""
    hidden = wl.linears[0].K
    z = normal(wl.seed, 900_000 + i, hidden)
    return bf16_bits_from_f64(1.0 + 0.1 * z)
