"""Seeded synthetic inputs shared by the oracle harness, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no packing, no GEMM, no LoRA):
only counter-based random numbers, bf16 rounding of those numbers, and the
workload recipes (sequence-length / rank / batch-size mixes) of BASELINE.json's
configs.  Both sides of every parity check consume the exact bf16 bit patterns
produced here.
"""
from .gen import (  # noqa: F401
    splitmix64, uniform01, normal, bf16_bits_from_f64, bf16_bits_to_f32,
    normal_bf16, int_bf16, sparse_int_bf16, seq_lengths, Stream,
)
from .configs import (  # noqa: F401
    Workload, Linear, workload, CONFIG_IDS, base_seed, token_input, weight, adapter, int_scales, norm_weight,
)
