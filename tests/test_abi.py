"""CPU checks of the drop-in boundary: libs5.so loads and exports exactly the
C-ABI declared in include/s5.h; argument validation runs without a GPU."""
import ctypes as C
import os
import re

import pytest

from paper_1305_1157_b200 import _lib
from conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "s5.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(s5_[a-z0-9_]+)\s*\(", text,
                                 re.M)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("s5_sort", "s5_sort_host", "s5_workspace_bytes", "s5_pack_keys",
                 "s5_adjacent_lcp", "s5_classify", "s5_build_tree", "s5_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_declared()) <= set(_lib.SIGNATURES)


def test_config_validation_without_gpu():
    L = _lib.lib()
    good = _lib.S5Config(8191, 2, 0, 32, 16384, 0, 1)
    assert L.s5_workspace_bytes(1 << 20, 1 << 24, C.byref(good)) > 24 * (1 << 20)
    bad = _lib.S5Config(100, 2, 0, 32, 16384, 0, 1)   # not 2^d - 1
    assert L.s5_workspace_bytes(1000, 1000, C.byref(bad)) == 0
    rc = L.s5_sort(None, 10, None, 5, 0, None, C.byref(bad), None, 0, None, None)
    assert rc == -1 and b"2**d - 1" in L.s5_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc, "s5_sort")


def test_trivial_sizes_are_noops_without_gpu():
    L = _lib.lib()
    cfg = _lib.S5Config(8191, 2, 0, 32, 16384, 0, 1)
    assert L.s5_sort(None, 0, None, 1, 0, None, C.byref(cfg), None, 0, None, None) == 0
    assert L.s5_sort(None, 0, None, 0, 0, None, C.byref(cfg), None, 0, None, None) == 0


def test_sort_multi_argument_validation_without_gpu():
    """s5_sort_multi rejects bad device counts and null tables before it
    touches a device (include/s5.h)."""
    L = _lib.lib()
    one = (C.c_uint64 * 1)(0)
    dev = (C.c_int * 1)(0)
    ptr = (C.c_void_p * 1)(None)
    assert L.s5_sort_multi(0, dev, ptr, 0, ptr, one, ptr, None, one, one, None, None) == -1
    assert b"n_gpus" in L.s5_last_error()
    assert L.s5_sort_multi(65, dev, ptr, 0, ptr, one, ptr, None, one, one, None, None) == -1
    assert L.s5_sort_multi(1, dev, ptr, 0, ptr, None, ptr, None, one, one, None, None) == -1
    assert b"null" in L.s5_last_error()


def test_markov_helper_matches_numpy_searchsorted():
    import numpy as np
    from paper_1305_1157_b200 import _native
    rng = np.random.default_rng(0)
    P = rng.dirichlet(np.full(8, 0.3), size=(8, 8))
    cdf = np.cumsum(P, axis=2)
    u = rng.random(5000)
    got = _native.markov_text(cdf, u, 8)
    a, b = 0, 1
    want = np.empty(u.size, np.uint8)
    for i in range(u.size):
        s = min(int(np.searchsorted(cdf[a, b], u[i], side="left")), 7)
        want[i] = 0x40 + s
        a, b = b, s
    assert np.array_equal(got, want)


def test_product_has_no_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_1305_1157_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "s5_oracle" not in src and "libs5oracle" not in src, f


def test_copy_pieces_helper_matches_numpy():
    import numpy as np
    from paper_1305_1157_b200 import _native, datasets
    rng = np.random.default_rng(1)
    blob = rng.integers(0, 256, 5000, dtype=np.uint8)
    m = 200_000  # above the helper's threading threshold
    ln = rng.integers(0, 9, m)
    src = rng.integers(0, blob.size - 8, m)
    dst = np.concatenate([[0], np.cumsum(ln)[:-1]])
    got = np.zeros(int(ln.sum()) + 1, np.uint8)
    _native.copy_pieces(got, dst, src, ln, blob)
    want = np.zeros_like(got)
    rep = np.repeat(np.arange(m), ln)
    within = np.arange(int(ln.sum())) - np.repeat(np.cumsum(ln) - ln, ln)
    want[dst[rep] + within] = blob[src[rep] + within]
    assert np.array_equal(got, want)
    with pytest.raises(ValueError):
        _native.copy_pieces(got, dst + got.size, src, ln, blob)
    # config 3's generator through the helper still reproduces SURVEY's N
    arena, h = datasets.generate(3, 1 << 12)
    assert h.size == 1 << 12 and arena.data[-1] == 0
