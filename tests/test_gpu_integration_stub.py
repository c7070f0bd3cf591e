"""The reference-side ctypes stubs printed in INTEGRATION.md actually work:
the Python blocks are extracted from the document, pointed at the in-tree
libs5.so and run against the oracle (one GPU; workers > 1 over a repeated
device needs several GPUs in the stub, so it runs with G = device_count)."""
import os
import re
import types

import numpy as np
import pytest

import oracle as O
from paper_1305_1157_b200 import SampleSortConfig, datasets

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_module():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    src = "\n".join(b for b in blocks if "_S5Config" in b or "s5_sort_multi" in b)
    src = src.replace("/path/to/paper_1305_1157_b200/libs5.so",
                      os.path.join(ROOT, "paper_1305_1157_b200", "libs5.so"))
    mod = types.ModuleType("integration_stub")
    mod.SampleSortConfig = SampleSortConfig
    exec(compile(src, "INTEGRATION.md", "exec"), mod.__dict__)
    return mod


@pytest.mark.parametrize("config,n", [(1, None), (3, 1 << 15)])
def test_integration_stubs_match_oracle(config, n):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mod = _stub_module()
    arena, h0 = datasets.generate(config, n)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, 8)
    want_lcp = O.adjacent_lcps(arena, want)
    for fn, workers in ((mod.gpu_parallel_sample_sort, 1),
                        (mod.gpu_parallel_sample_sort_multi, 8)):
        h = h0.copy()
        lcp = np.full(h.size - 1, -3, np.int64)
        fn(arena, h, workers, None, lcp_out=lcp)
        assert O.contents_equal(arena, h, want)
        assert np.array_equal(lcp, want_lcp)
