"""String sample sort entry points, executed by libs5.so on a B200.

Keeps the reference signatures (pkg/src/strsort/samplesort.py):

- ``sample_sort(arena, handles, depth=0, cfg=None, counters=None, audit=None)``
  (samplesort.py:241-267)
- ``parallel_sample_sort(arena, handles, workers=1, cfg=None, counters=None,
  audit=None)`` (samplesort.py:437-444)

Both sort ``handles`` in place and return it.  ``handles`` may be a numpy
int64 array (uploaded, sorted, downloaded) or a CUDA ``torch.int64`` tensor
(sorted in HBM).  The new keyword ``lcp_out`` receives the LCP array
(``_adjacent_lcps`` semantics, strings.py:99-102); ``sort_with_lcp`` returns
it.  ``workers`` is accepted for signature compatibility: one call runs on
one GPU (multi-GPU sorting is ``paper_1305_1157_b200.distributed``).

The reference is not stable; neither is this sorter.  Output is defined up to
the order of identical strings; the string sequence and the LCP array are
unique.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .counters import Counters
from .strings import StringArena

T_MEDIUM = 64 * 1024  # samplesort.py:34
T_INSERTION = 64      # basesort.py:26


@dataclass
class SampleSortConfig:
    """samplesort.py:37-45 plus the GPU tiering knobs.

    ``t_m``/``t_i``/``interleave`` are kept for signature compatibility; the
    GPU tiers are ``narrow_max`` (segments up to it take the one-CTA S^5
    step; 0 = the library default, 4096 = off), ``local_max`` (one-CTA base case,
    <= 4096) and ``small_max`` (warp base case, <= 32 strings).  ``alpha`` defaults to 4
    (the reference's 2 is accepted): the wide steps' samples are cheap on the
    device and better balanced buckets pay (measured 1-2 %); splitters only
    move the order of identical strings, never the output.
    """
    v: int = 8191
    alpha: int = 4
    t_m: int = T_MEDIUM
    t_i: int = T_INSERTION
    classifier: str = "unroll"
    interleave: int = 3
    seed: int = 1
    small_max: int = 32
    narrow_max: int = 0
    local_max: int = 4096
    wide_v: int = 511
    wide_target: int = 512
    local_target: int = 8
    flags: int = 0

    def to_c(self) -> _lib.S5Config:
        if self.classifier not in ("unroll", "equal"):
            raise ValueError(f"unknown classifier {self.classifier!r}")
        return _lib.S5Config(self.v, self.alpha, 1 if self.classifier == "equal" else 0,
                             self.small_max, self.narrow_max, self.flags, self.seed,
                             self.local_max,
                             self.wide_v, self.wide_target, self.local_target)


#: wall-clock phases of the last host-buffer call (H2D, sort, D2H), ms
LAST_HOST_MS: dict = {}

_ws_lock = threading.Lock()
_ws_cache: dict = {}


def _workspace(nbytes: int, device):
    """Cached device workspace per (device, calling thread): a sort's last
    kernels may still be in flight on its stream when the call returns, so
    concurrent callers (threads driving several GPUs, or several streams of
    one GPU) never share a buffer."""
    import torch
    key = (str(device), threading.get_ident())
    with _ws_lock:
        if len(_ws_cache) > 1:  # buffers of threads that have exited
            alive = {t.ident for t in threading.enumerate()}
            for k in [k for k in _ws_cache if k[1] not in alive]:
                del _ws_cache[k]
        buf = _ws_cache.get(key)
        if buf is None or buf.numel() < nbytes:
            _ws_cache.pop(key, None)
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
            _ws_cache[key] = buf
        return buf


def release_workspace():
    with _ws_lock:
        _ws_cache.clear()


def _device_of(handles):
    import torch
    if isinstance(handles, torch.Tensor) and handles.is_cuda:
        return handles.device
    return torch.device("cuda", torch.cuda.current_device())


def gpu_sort(arena: StringArena, d_handles, depth: int = 0, cfg: SampleSortConfig | None = None,
             d_lcp=None, stats: _lib.S5Stats | None = None):
    """Sort a CUDA int64 handle tensor in place (HBM resident); optional LCP."""
    import torch
    cfg = cfg or SampleSortConfig()
    n = int(d_handles.numel())
    if d_handles.dtype != torch.int64 or not d_handles.is_contiguous():
        raise ValueError("handles must be a contiguous int64 tensor")
    if n <= 1:
        return d_handles
    dev = d_handles.device
    arena_dev = arena.device(dev)
    c = cfg.to_c()
    need = int(_lib.lib().s5_workspace_bytes(n, arena.size, C.byref(c)))
    if need == 0:
        _lib.check(-1, "s5_workspace_bytes")
    ws = _workspace(need, dev)
    if d_lcp is not None and (d_lcp.numel() < n - 1 or d_lcp.dtype != torch.int64):
        raise ValueError("lcp buffer must be int64 with n-1 elements")
    st = stats if stats is not None else _lib.S5Stats()
    with torch.cuda.device(dev):
        rc = _lib.lib().s5_sort(
            arena_dev.data_ptr(), arena.size, d_handles.data_ptr(), n, int(depth),
            d_lcp.data_ptr() if d_lcp is not None else None, C.byref(c), ws.data_ptr(),
            ws.numel(), _lib.current_stream_ptr(), C.byref(st))
    _lib.check(rc, "s5_sort")
    return d_handles


def _record(counters: Counters | None, st: _lib.S5Stats):
    if counters is None:
        return
    counters.add("parallel_steps", int(st.levels))
    counters.add("sample_steps", int(st.wide_steps + st.narrow_steps))
    counters.add("fetches", int(st.key_fetches))
    counters.add("base_segments", int(st.small_segments))
    counters.add("boundary_lcps", int(st.boundary_lcps))


def _sort(arena, handles, depth, cfg, counters, audit, lcp_out):
    import torch
    if audit is not None:
        from ._audit import audited_sort
        return audited_sort(arena, handles, depth, cfg or SampleSortConfig(), counters, audit,
                            lcp_out)
    n = int(len(handles))
    if n <= 1:
        return handles
    on_device = isinstance(handles, torch.Tensor) and handles.is_cuda
    dev = _device_of(handles)
    if not on_device:
        if not isinstance(handles, np.ndarray) or handles.dtype != np.int64:
            raise TypeError("handles must be a numpy int64 array or a CUDA int64 tensor")
        return _sort_host(arena, handles, depth, cfg, counters, lcp_out, dev)
    d_h = handles
    d_lcp = None
    if lcp_out is not None:
        if isinstance(lcp_out, torch.Tensor) and lcp_out.is_cuda:
            d_lcp = lcp_out
        else:
            d_lcp = torch.empty(n - 1, dtype=torch.int64, device=dev)
    st = _lib.S5Stats()
    gpu_sort(arena, d_h, depth, cfg, d_lcp, st)
    _record(counters, st)
    if lcp_out is not None and d_lcp is not lcp_out:
        lcp_out[: n - 1] = d_lcp.cpu().numpy()
    return handles


def _sort_host(arena, handles, depth, cfg, counters, lcp_out, dev):
    """numpy handles: the C-ABI host path (s5_sort_host) -- H2D, sort, D2H."""
    import torch
    n = int(handles.size)
    cfg = cfg or SampleSortConfig()
    h = handles if handles.flags.c_contiguous and handles.flags.writeable else \
        np.ascontiguousarray(handles)
    lcp_buf = None
    if lcp_out is not None:
        if isinstance(lcp_out, np.ndarray) and lcp_out.dtype == np.int64 and \
                lcp_out.flags.c_contiguous and lcp_out.size >= n - 1:
            lcp_buf = lcp_out
        else:
            lcp_buf = np.empty(n - 1, np.int64)
    c = cfg.to_c()
    st = _lib.S5Stats()
    with torch.cuda.device(dev):
        arena_dev = arena.device(dev)
        rc = _lib.lib().s5_sort_host(arena_dev.data_ptr(), arena.size, h.ctypes.data, n,
                                     int(depth), lcp_buf.ctypes.data if lcp_buf is not None
                                     else None, C.byref(c), _lib.current_stream_ptr(),
                                     C.byref(st))
    _lib.check(rc, "s5_sort_host")
    _record(counters, st)
    global LAST_HOST_MS
    LAST_HOST_MS = {"h2d": float(st.host_h2d_ms), "sort": float(st.host_sort_ms),
                    "d2h": float(st.host_d2h_ms), "h2d_bytes": int(st.host_h2d_bytes),
                    "d2h_bytes": int(st.host_d2h_bytes)}
    if h is not handles:
        handles[:] = h
    if lcp_out is not None and lcp_buf is not lcp_out:
        if isinstance(lcp_out, torch.Tensor):
            lcp_out.copy_(torch.from_numpy(lcp_buf))
        else:
            lcp_out[: n - 1] = lcp_buf
    return handles


def sample_sort(arena: StringArena, handles, depth: int = 0, cfg: SampleSortConfig | None = None,
                counters: Counters | None = None, audit=None, lcp_out=None):
    """String sample sort from common depth ``depth`` (samplesort.py:241-267)."""
    return _sort(arena, handles, depth, cfg, counters, audit, lcp_out)


def parallel_sample_sort(arena: StringArena, handles, workers: int = 1,
                         cfg: SampleSortConfig | None = None, counters: Counters | None = None,
                         audit=None, lcp_out=None, devices=None):
    """Fully parallel string sample sort (samplesort.py:437-444).

    ``workers`` is the number of GPUs (the reference's worker threads): with
    ``workers > 1`` and several visible devices the sort runs on
    ``min(workers, device_count)`` of them from this process (sample-sort
    partitioning + peer copies, ``multi.multi_gpu_sort``); ``devices`` names
    them explicitly (a device may repeat: several shards on one GPU).  One
    GPU otherwise.  ``audit`` runs single-GPU."""
    import torch
    if devices is None and workers > 1 and torch.cuda.is_available():
        devices = list(range(min(int(workers), torch.cuda.device_count())))
    n = int(len(handles))
    # the multi-GPU exchange carries u32 offsets: an arena of >= 4 GiB sorts on
    # one GPU (index mode, include/s5.h)
    if audit is None and devices is not None and len(devices) > 1 and n > 1 \
            and arena.size <= 0xFFFFFFFF:
        from .multi import multi_gpu_sort
        on_device = isinstance(handles, torch.Tensor) and handles.is_cuda
        if not on_device and (not isinstance(handles, np.ndarray) or handles.dtype != np.int64):
            raise TypeError("handles must be a numpy int64 array or a CUDA int64 tensor")
        h = handles if on_device or (handles.flags.c_contiguous and handles.flags.writeable) \
            else np.ascontiguousarray(handles)
        lo = lcp_out
        if lcp_out is not None and not on_device and not (
                isinstance(lcp_out, np.ndarray) and lcp_out.dtype == np.int64
                and lcp_out.flags.c_contiguous):
            lo = np.empty(n - 1, np.int64)
        multi_gpu_sort(arena, h, devices, cfg, lo, counters=counters)
        if h is not handles:
            handles[:] = h
        if lo is not lcp_out:
            lcp_out[: n - 1] = lo
        return handles
    return _sort(arena, handles, 0, cfg, counters, audit, lcp_out)


def sort_with_lcp(arena: StringArena, handles, cfg: SampleSortConfig | None = None,
                  counters: Counters | None = None):
    """Sort in place and return ``(handles, lcp)`` (lcp int64[n-1])."""
    import torch
    n = int(len(handles))
    if isinstance(handles, torch.Tensor) and handles.is_cuda:
        lcp = torch.empty(max(n - 1, 0), dtype=torch.int64, device=handles.device)
    else:
        lcp = np.empty(max(n - 1, 0), np.int64)
    _sort(arena, handles, 0, cfg, counters, None, lcp if n > 1 else None)
    return handles, lcp
