"""paper_2603_02885_b200 — B200-native multiplexed LoRA linear (MuxTune hot path).

The product is libmux.so (C ABI, include/mux.h) built from csrc/ for sm_100a;
`mux` is its thin Python binding.  No CPU fallback exists.
"""
from . import mux  # noqa: F401
from .mux import (  # noqa: F401
    Adapter, MuxError, pack_chunks, pack_apply, linear_fwd, linear_bwd, read_info,
    make_B_storage, linear_workspace_size, pack_bound_rows, version,
)
from .autograd import MuxLoRALinear  # noqa: F401,E402
