"""Several GPUs from one process: ``parallel_sample_sort(..., workers=G)``.

The reference's ``workers`` is the number of threads of one pS^5 call
(samplesort.py:437-444; the fully parallel step splits every stage over
them, :369-434).  Here it is the number of GPUs: the same sample-sort
partitioning as ``distributed.distributed_sample_sort``,
driven by one host thread per device instead of one process per GPU, and
with the exchange done as direct device-to-device copies (NVLink peer
copies) instead of NCCL.  Steps 2-5 are one C-ABI call, ``s5_sort_multi``
(csrc/s5_multi.cuh); this module moves the caller's buffers in and out:

1. the handles are split into G contiguous shards, one per device (host
   arrays cross PCIe as u32 offsets, ``s5_upload_handles``);
2. every device draws ``max(64 * G, 2048)`` sample handles; the samples are
   gathered on the first device, sorted there by (string, handle) and the
   G-1 splitter strings sent to every device;
3. every device groups its shard by destination (``s5_partition``);
4. group (g -> d) is copied from device g into device d's receive buffer
   as u32 offsets;
5. every device sorts what it received (``s5_sort`` reading the u32 payload
   in place, flags bit9) and emits its LCP array; the LCP across each slice
   boundary is one comparison on the left device;
6. the slices are the global order: written back into the caller's array
   (host: ``s5_download``'s narrow staging; device tensor: peer copies).

A device may appear more than once in ``devices`` (several shards on one
GPU, serialised by the library): the tests use that to run the G > 1 path
on a one-GPU machine.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .distributed import GpuBackend


def _on(dev, fn, *a):
    import torch
    with torch.cuda.device(dev):
        return fn(*a)


def multi_gpu_sort(arena, handles, devices, cfg=None, lcp_out=None, counters=None):
    """Sort ``handles`` (numpy int64 or a CUDA int64 tensor) in place over the
    GPUs ``devices``; the LCP array goes to ``lcp_out`` (same kind of
    buffer, n-1 entries) when given.  Returns ``handles``."""
    import torch
    devs = [torch.device("cuda", int(d)) for d in devices]
    G = len(devs)
    n = int(len(handles))
    on_device = isinstance(handles, torch.Tensor) and handles.is_cuda
    bes = [_on(d, GpuBackend, arena, cfg) for d in devs]
    pool = ThreadPoolExecutor(max_workers=G)
    try:
        def par(fn, *lists):
            futs = [pool.submit(_on, devs[g], fn, g, *[x[g] for x in lists]) for g in range(G)]
            return [f.result() for f in futs]

        bounds = [(n * g // G, n * (g + 1) // G) for g in range(G)]

        # 1. shards on their devices
        def load(g):
            lo, hi = bounds[g]
            if on_device:
                return handles[lo:hi].to(devs[g])
            return bes[g].upload(np.ascontiguousarray(handles[lo:hi]))
        shards = par(load)

        # 2.-5. samples, splitters, partition, exchange, local sorts and the
        # boundary LCPs: one library call (s5_sort_multi, include/s5.h)
        out_h, out_l = sort_multi_device(arena, shards, [d.index for d in devs], cfg,
                                         want_lcp=lcp_out is not None, counters=counters)
        sizes = [int(t.numel()) for t in out_h]
        if out_l is None:
            out_l = [t[:0] for t in out_h]

        # 6. the slices back into the caller's buffers, in global order
        offs = [sum(sizes[:d]) for d in range(G)]

        def store(d):
            a, m = offs[d], sizes[d]
            if not m:
                return
            nl = out_l[d].numel()
            if on_device:
                handles[a:a + m].copy_(out_h[d])
                if lcp_out is not None and nl:
                    lcp_out[a:a + nl].copy_(out_l[d])
                torch.cuda.synchronize(devs[d])
            else:
                bes[d].download(out_h[d], out_l[d] if lcp_out is not None else out_l[d][:0],
                                handles[a:a + m], lcp_out[a:a + nl] if lcp_out is not None else None)
        par(lambda d: store(d))
    finally:
        pool.shutdown(wait=True)
    return handles


def sort_multi_device(arena, shards, devices, cfg=None, want_lcp: bool = True, counters=None):
    """``s5_sort_multi`` (include/s5.h): the same split done by the library
    itself from C -- one call, device shards in, sorted device slices out.

    ``shards[g]`` is a CUDA int64 tensor of handles on ``devices[g]`` (left
    untouched).  Returns ``(slices, lcps)``: ``slices[d]`` the sorted handles
    of slice d on ``devices[d]``; the concatenation in device order is the
    global order and that of ``lcps`` its LCP array (``None`` without
    ``want_lcp``)."""
    import ctypes as C

    import torch
    from . import _lib
    from .samplesort import SampleSortConfig
    G = len(devices)
    if G != len(shards):
        raise ValueError("one shard per device")
    devs = [torch.device("cuda", int(d)) for d in devices]
    total = sum(int(s.numel()) for s in shards)
    arenas = [arena.device(d) for d in devs]
    shards = [s.contiguous() for s in shards]
    outs = [torch.empty(max(total, 1), dtype=torch.int64, device=d) for d in devs]
    lcps = [torch.empty(max(total, 1), dtype=torch.int64, device=d) for d in devs] if want_lcp else None
    for d in devs:
        torch.cuda.synchronize(d)
    ptrs = lambda ts: (C.c_void_p * G)(*[t.data_ptr() for t in ts])
    dev_ids = (C.c_int * G)(*[d.index for d in devs])
    ns = (C.c_uint64 * G)(*[int(s.numel()) for s in shards])
    cap = (C.c_uint64 * G)(*[max(total, 1)] * G)
    counts = (C.c_uint64 * G)()
    ccfg = (cfg or SampleSortConfig()).to_c()
    st = _lib.S5Stats()
    rc = _lib.lib().s5_sort_multi(G, dev_ids, ptrs(arenas), arena.size, ptrs(shards), ns, ptrs(outs),
                                  ptrs(lcps) if want_lcp else None, cap, counts, C.byref(ccfg),
                                  C.byref(st))
    _lib.check(rc, "s5_sort_multi")
    if counters is not None:
        counters.add("gpus", G)
        counters.add("parallel_steps", int(st.levels))
        counters.add("fetches", int(st.key_fetches))
    sizes = [int(c) for c in counts]
    last = max((d for d in range(G) if sizes[d]), default=-1)
    slices = [outs[d][:sizes[d]] for d in range(G)]
    if not want_lcp:
        return slices, None
    return slices, [lcps[d][:max(sizes[d] - (1 if d == last else 0), 0)] for d in range(G)]
