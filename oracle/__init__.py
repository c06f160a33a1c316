"""fp64 CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import, call, link or execute anything under oracle/.
The product path (paper_2603_02885_b200/) never imports it and shares no code
with it: no kernels, headers, helpers, tables or pre/post-processing.

Contents
  pack.py    chunk-based alignment (§3.5) — pure Python, integer.
  linear.c   multiplexed LoRA linear fwd/bwd (Eq. 1-2 + north_star
             LoRA formula) — plain C, fp64, fixed ascending summation order.
  linear.py  ctypes wrapper around liboracle.so (bf16 bits -> fp64 widening).
  block.py   decoder-block ops around the linears (NEXT-3): causal attention
             inside packed sequences (chunk KV reuse), RoPE,
             RMSNorm, SwiGLU — numpy fp64, from the definitions.

Pins (tests/test_oracle_*.py, `-m "not gpu"`): see DESIGN.md §"Oracle pins".
Parity unpinned: none of the functions here (the paper's 0.07 MSD convergence
claim, is not implemented and is out of scope).
"""
