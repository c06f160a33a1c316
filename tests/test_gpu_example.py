"""The public-API example (examples/multitask_lora_train.py): three tasks trained
together through pack_chunks / pack_apply / MuxLoRALinear; every task's loss falls."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples"))


def test_multitask_example_losses_fall():
    import multitask_lora_train as ex
    hist = ex.main(steps=25, verbose=False)
    first, last = hist[0], hist[-1]
    for t in range(len(first)):
        assert last[t] < 0.8 * first[t], (t, first[t], last[t])
