"""Splitter trees and branch-free classification on the B200.

Mirror of the reference module ``strsort.classifier``
(pkg/src/strsort/classifier.py).  The sorter itself builds and uses trees
inside its kernels (csrc/s5_kernels.cuh: build_tree_levels, classify); the
functions here expose the same device code as operation surfaces:

- ``select_splitters(sample, v)`` / ``build_tree_from_sample`` run the
  device tree builder (classifier.py:85-126);
- ``classify_tree_unrolled`` / ``classify_tree_equal`` run the device
  classifiers (classifier.py:259-278);
- ``build_tree`` is the host-side record of a tree (classifier.py:159-176).

The bucket layout (boundaries, depth gains, finished flags;
classifier.py:284-304) exists only on the device: ``k_wide_bscan`` and
``emit_block`` in csrc/s5_kernels.cuh (audited by the Eq. (1) tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .strings import WORD_CHARS


class BadSplitterCount(ValueError):
    """Splitter array length must be 2**d - 1 (classifier.py:30-31)."""


def oracle_dtype(v: int):
    """classifier.py:34-36."""
    return np.uint8 if 2 * v + 1 <= 256 else np.uint16


@dataclass
class SplitterTree:
    """classifier.py:39-53."""
    level_order: np.ndarray
    in_order: np.ndarray
    splitter_lcp: np.ndarray
    terminated: np.ndarray
    depth: int

    @property
    def v(self) -> int:
        return self.in_order.size

    @property
    def num_buckets(self) -> int:
        return 2 * self.in_order.size + 1


def _depth_of(v: int) -> int:
    d = int(v).bit_length()
    if v < 1 or (1 << d) - 1 != v:
        raise BadSplitterCount(f"need 2**d - 1 splitters, got {v}")
    return d


def _inorder_rank(i: int, level: int, d: int) -> int:
    return (2 * (i - (1 << level)) + 1) * (1 << (d - 1 - level)) - 1


def inorder_rank(i: int, level: int, d: int) -> int:
    """classifier.py:179-181."""
    return _inorder_rank(i, level, d)


def _has_zero_byte(w: np.ndarray) -> np.ndarray:
    w = np.asarray(w, np.uint64)
    out = np.zeros(w.shape, bool)
    for k in range(8):
        out |= ((w >> np.uint64(56 - 8 * k)) & np.uint64(0xFF)) == 0
    return out


def build_tree(in_order) -> SplitterTree:
    """Level order, splitter LCPs and terminator flags (classifier.py:159-176)."""
    in_order = np.ascontiguousarray(in_order, np.uint64)
    v = in_order.size
    d = _depth_of(v)
    idx = np.arange(1, v + 1)
    lvl = np.floor(np.log2(idx)).astype(np.int64)
    ranks = (2 * (idx - (1 << lvl)) + 1) * (1 << (d - 1 - lvl)) - 1
    level_order = np.zeros(v + 1, np.uint64)
    level_order[1:] = in_order[ranks]
    lcps = np.zeros(v, np.int64)
    if v > 1:
        x = in_order[:-1] ^ in_order[1:]
        nz = x != 0
        clz = np.full(x.shape, 64, np.int64)
        xv = x[nz]
        # leading zero bits via float-free bit scan
        lz = np.zeros(xv.shape, np.int64)
        for shift in (32, 16, 8, 4, 2, 1):
            top = (xv >> np.uint64(64 - shift)) == 0
            lz += np.where(top, shift, 0)
            xv = np.where(top, xv << np.uint64(shift), xv)
        clz[nz] = lz
        lcps[1:] = np.where(nz, clz // 8, WORD_CHARS)
    return SplitterTree(level_order, in_order, lcps, _has_zero_byte(in_order), d)


def select_splitters(sample, v: int) -> np.ndarray:
    """Recursive middle selection (classifier.py:85-115), run by the device
    tree builder the sorter uses; returns the in-order splitters."""
    _, in_order = build_tree_from_sample(sample, v)
    return in_order


def build_tree_from_sample(sample, v: int):
    """(level_order[v+1], in_order[v]) from a sorted sample, on the device."""
    import torch
    from .strings import _dev
    _depth_of(v)
    s = np.ascontiguousarray(sample, np.uint64)
    if s.size == 0:
        raise ValueError("empty sample")
    dev = _dev()
    ds = torch.from_numpy(s.view(np.int64)).to(dev)
    lo = torch.zeros(v + 1, dtype=torch.int64, device=dev)
    io = torch.zeros(v, dtype=torch.int64, device=dev)
    rc = _lib.lib().s5_build_tree(ds.data_ptr(), s.size, v, lo.data_ptr(), io.data_ptr(),
                                  _lib.current_stream_ptr())
    _lib.check(rc, "s5_build_tree")
    return lo.cpu().numpy().view(np.uint64), io.cpu().numpy().view(np.uint64)


def _classify(keys, tree: SplitterTree, variant: int, out=None) -> np.ndarray:
    import torch
    from .strings import _dev
    keys = np.ascontiguousarray(keys, np.uint64)
    if out is None:
        out = np.empty(keys.size, oracle_dtype(tree.v))
    if keys.size == 0:
        return out
    dev = _dev()
    dk = torch.from_numpy(keys.view(np.int64)).to(dev)
    di = torch.from_numpy(np.ascontiguousarray(tree.in_order, np.uint64).view(np.int64)).to(dev)
    db = torch.empty(keys.size, dtype=torch.int16, device=dev)
    rc = _lib.lib().s5_classify(dk.data_ptr(), keys.size, di.data_ptr(), tree.v, variant,
                                db.data_ptr(), _lib.current_stream_ptr())
    _lib.check(rc, "s5_classify")
    out[:] = db.cpu().numpy().view(np.uint16)
    return out


def classify_tree_unrolled(keys, tree: SplitterTree, interleave: int = 3, out=None):
    """Full branch-free descent + leaf equality test (classifier.py:259-268)."""
    return _classify(keys, tree, 0, out)


def classify_tree_equal(keys, tree: SplitterTree, out=None):
    """Equality test per node with early exit (classifier.py:271-278)."""
    return _classify(keys, tree, 1, out)


def classify_tree_lut(keys, tree: SplitterTree, out=None):
    """Table over the 12 key bits after the splitters' common prefix + binary
    search: the classifier of the multi-CTA count kernel (same buckets)."""
    return _classify(keys, tree, 2, out)
