"""Host-side helpers exported by libs5.so (dataset generation only)."""

from __future__ import annotations

import numpy as np

from . import _lib


def markov_text(cdf: np.ndarray, u: np.ndarray, sigma: int) -> np.ndarray:
    """Order-2 Markov text (SURVEY.md 8(d) recipe 5) via s5_host_markov_text."""
    cdf = np.ascontiguousarray(cdf, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    out = np.empty(u.size, np.uint8)
    rc = _lib.lib().s5_host_markov_text(cdf.ctypes.data, u.ctypes.data, u.size, sigma,
                                        out.ctypes.data)
    _lib.check(rc, "s5_host_markov_text")
    return out
