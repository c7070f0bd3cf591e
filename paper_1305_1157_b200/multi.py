"""Several GPUs from one process: ``parallel_sample_sort(..., workers=G)``.

The reference's ``workers`` is the number of threads of one pS^5 call
(samplesort.py:437-444; the fully parallel step splits every stage over
them, :369-434).  Here it is the number of GPUs: the same sample-sort
partitioning as ``distributed.distributed_sample_sort``,
driven by one host thread per device instead of one process per GPU, and
with the exchange done as direct device-to-device copies (NVLink peer
copies through ``Tensor.copy_``) instead of NCCL:

1. the handles are split into G contiguous shards, one per device (host
   arrays cross PCIe as u32 offsets, ``s5_upload_handles``);
2. every device draws ``oversample * G`` sample handles; the samples are
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

from .distributed import GpuBackend, _pick_splitters


def _on(dev, fn, *a):
    import torch
    with torch.cuda.device(dev):
        return fn(*a)


def multi_gpu_sort(arena, handles, devices, cfg=None, lcp_out=None, oversample: int = 64,
                   seed: int = 1, counters=None):
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

        # 2. samples -> first device -> splitters -> every device
        s = oversample * G

        def sample(g):
            h = shards[g]
            if not h.numel():
                return torch.full((s,), -1, dtype=torch.int64, device=devs[g])
            gen = torch.Generator(device=devs[g]).manual_seed(seed * 1_000_003 + g)
            return h[torch.randint(0, h.numel(), (s,), generator=gen, device=devs[g])]
        samp = par(sample)
        with torch.cuda.device(devs[0]):
            allsamp = torch.cat([x.to(devs[0]) for x in samp])
            top = allsamp.max().clamp(min=0)
            allsamp = torch.where(allsamp >= 0, allsamp, top)
            splitters = _pick_splitters(bes[0], allsamp, G)
        spl = [splitters.to(d) for d in devs]

        # 3. group by destination
        def part(g):
            return bes[g].partition(shards[g], spl[g])
        parts = par(part)
        send32 = [_on(devs[g], lambda t: t.to(torch.int32), parts[g][0]) for g in range(G)]
        counts = [p[1] for p in parts]  # counts[src][dst]
        sizes = [sum(counts[g][d] for g in range(G)) for d in range(G)]

        # 4. exchange (peer copies into each destination's buffer)
        def exchange(d):
            buf = torch.empty(sizes[d], dtype=torch.int64, device=devs[d])
            b32 = buf.view(torch.int32)
            at = 0
            for g in range(G):
                c = counts[g][d]
                if c:
                    lo = sum(counts[g][:d])
                    b32[at:at + c].copy_(send32[g][lo:lo + c])
                at += c
            torch.cuda.synchronize(devs[d])
            return buf
        recv = par(exchange)
        for g in range(G):
            torch.cuda.synchronize(devs[g])

        # 5. local sorts (the library releases the GIL: the devices overlap)
        def local(d):
            return bes[d].sort_u32(recv[d], sizes[d])
        res = par(local)
        out_h = [r[0] for r in res]
        out_l = [r[1] for r in res]
        for d in range(G):  # boundary LCP on the left device
            nxt = next((r for r in range(d + 1, G) if sizes[r]), None)
            if sizes[d] and nxt is not None:
                pair = torch.cat([out_h[d][-1:], out_h[nxt][:1].to(devs[d])])
                out_l[d] = torch.cat([out_l[d], _on(devs[d], bes[d].lcp_pair, pair)])
        if counters is not None:
            counters.add("gpus", G)
            for be in bes:
                st = getattr(be, "last_stats", None)
                if st is not None:
                    counters.add("parallel_steps", int(st.levels))
                    counters.add("fetches", int(st.key_fetches))

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
