"""Host-side helpers exported by libs5.so (dataset generation only)."""

from __future__ import annotations

import numpy as np

from . import _lib


def copy_pieces(data: np.ndarray, dst_start, src_start, lengths, blob: np.ndarray) -> None:
    """data[dst_start[i] + j] = blob[src_start[i] + j], j < lengths[i] (s5_host_copy_pieces)."""
    d = np.ascontiguousarray(dst_start, np.int64)
    s = np.ascontiguousarray(src_start, np.int64)
    ln = np.ascontiguousarray(lengths, np.int64)
    b = np.ascontiguousarray(blob, np.uint8)
    if ln.size and (int((d + ln).max()) > data.size or int((s + ln).max()) > b.size
                    or int(d.min()) < 0 or int(s.min()) < 0):
        raise ValueError("piece outside its buffer")
    assert data.flags.c_contiguous and data.dtype == np.uint8
    rc = _lib.lib().s5_host_copy_pieces(data.ctypes.data, d.ctypes.data, s.ctypes.data,
                                        ln.ctypes.data, b.ctypes.data, ln.size)
    _lib.check(rc, "s5_host_copy_pieces")


def markov_text(cdf: np.ndarray, u: np.ndarray, sigma: int) -> np.ndarray:
    """Order-2 Markov text (SURVEY.md 8(d) recipe 5) via s5_host_markov_text."""
    cdf = np.ascontiguousarray(cdf, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    out = np.empty(u.size, np.uint8)
    rc = _lib.lib().s5_host_markov_text(cdf.ctypes.data, u.ctypes.data, u.size, sigma,
                                        out.ctypes.data)
    _lib.check(rc, "s5_host_markov_text")
    return out
