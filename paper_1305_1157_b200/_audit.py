"""The reference's ``audit(side, lo, hi, depth)`` hook on the device sorter.

The reference calls ``audit`` for every pending child segment with the
handle array that holds it (samplesort.py:235-236, :431-432); its tests use
it to check Eq. (1): every pair in a child shares ``depth`` leading bytes.
``s5_sort_audit`` replays each level's child segment list and both ping-pong
offset arrays to the host (debug only; it copies 8n bytes per level).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def audited_sort(arena, handles, depth, cfg, counters, audit, lcp_out):
    import torch
    from .samplesort import _record, _workspace, _device_of
    n = int(len(handles))
    if n <= 1:
        return handles
    on_device = isinstance(handles, torch.Tensor) and handles.is_cuda
    dev = _device_of(handles)
    d_h = handles if on_device else torch.from_numpy(np.ascontiguousarray(handles)).to(dev)
    d_lcp = torch.empty(n - 1, dtype=torch.int64, device=dev) if lcp_out is not None else None
    c = cfg.to_c()
    need = int(_lib.lib().s5_workspace_bytes(n, arena.size, C.byref(c)))
    ws = _workspace(need, dev)
    errors = []

    def cb(user, level, segs, nsegs, side0, side1, nn):
        try:
            s0 = np.ctypeslib.as_array(side0, shape=(nn,)).astype(np.int64)
            s1 = np.ctypeslib.as_array(side1, shape=(nn,)).astype(np.int64)
            for i in range(nsegs):
                sg = segs[i]
                audit(s1 if sg.side & 1 else s0, int(sg.begin), int(sg.begin + sg.size), int(sg.depth))
        except Exception as e:  # surface after the C call returns
            errors.append(e)

    fn = _lib.AUDIT_FN(cb)
    st = _lib.S5Stats()
    rc = _lib.lib().s5_sort_audit(arena.device(dev).data_ptr(), arena.size, d_h.data_ptr(), n,
                                  int(depth), d_lcp.data_ptr() if d_lcp is not None else None,
                                  C.byref(c), ws.data_ptr(), ws.numel(), _lib.current_stream_ptr(),
                                  C.byref(st), fn, None)
    _lib.check(rc, "s5_sort_audit")
    if errors:
        raise errors[0]
    _record(counters, st)
    if not on_device:
        handles[:] = d_h.cpu().numpy()
    if lcp_out is not None:
        if isinstance(lcp_out, torch.Tensor):
            lcp_out.copy_(d_lcp)
        else:
            lcp_out[: n - 1] = d_lcp.cpu().numpy()
    return handles
