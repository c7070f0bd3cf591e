"""Multi-GPU S^5: one process per GPU, sample-sort partitioning over NCCL.

SURVEY.md 8(e).  The arena is replicated on every rank; rank g holds a
contiguous shard of the handles.  One exchange step turns the shards into
contiguous slices of the global sorted order:

1. every rank draws ``oversample * G`` sample handles from its shard;
   ``all_gather`` of the sample handles (the arena is replicated, so
   handles are enough);
2. every rank sorts all samples by full string content with a
   (string, handle) tie-break, so identical strings may be split across
   ranks (their order is free: the reference is not stable), and picks the
   same G-1 splitters;
3. every local string is classified to a destination rank by binary search
   over the splitters with full-string comparison and the handles are
   grouped by destination -- one library call (``s5_partition``: a counting
   kernel with the splitters' keys in shared memory, a column scan, a
   scatter);
4. ``all_gather`` of the per-destination counts (every rank learns the
   G x G matrix: its receive sizes and all slice sizes), then one
   ``all_to_all_single`` of the handles as u32 offsets (NCCL over NVLink on
   GPUs; gloo in the CPU tests);
5. each rank sorts its received strings with the single-GPU sorter (which
   reads the u32 payload in place) and emits their LCP array;
6. the LCP across each rank boundary is one string comparison (the next
   rank's first handle is all-gathered).

The string primitives come from a backend: ``GpuBackend`` (libs5.so; the
product path) or, in the CPU tests only, an oracle-backed stand-in injected
by the test.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

PHASES = None  # profiles/dist_phases.py sets a dict: per-phase wall ms (device synchronised)


def _mark(name, t):
    """Phase timing for profiles/dist_phases.py (no-op unless PHASES is a dict)."""
    if PHASES is None:
        return t
    import torch
    torch.cuda.synchronize()
    now = time.perf_counter()
    PHASES[name] = PHASES.get(name, 0.0) + 1e3 * (now - t)
    return now


class GpuBackend:
    """String primitives on the local GPU (libs5.so)."""

    def __init__(self, arena, cfg=None):
        import torch
        self.arena = arena
        self.cfg = cfg
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.launches = 0  # library kernels launched (sorts, partition, LCP)
        arena.device(self.device)

    def pack_keys(self, handles, depth: int):
        from .strings import pack_keys
        k = pack_keys(self.arena, handles, depth)
        return k.view(handles.dtype) if k.dtype != handles.dtype else k

    def lengths(self, handles):
        from .strings import string_lengths
        return string_lengths(self.arena, handles)

    def ends_at(self, handles, pos):
        """True where the string at ``handles`` has its terminator at ``pos``."""
        buf = self.arena.device(self.device)
        return buf[(handles + pos).clamp(0, self.arena.size - 1)] == 0

    def partition(self, handles, splitters):
        """Handles grouped by destination rank (s5_partition) and the group
        sizes."""
        import ctypes as C

        import torch
        from . import _lib
        n, ns = handles.numel(), splitters.numel()
        out = torch.empty_like(handles)
        counts = (C.c_uint64 * (ns + 1))()
        rc = _lib.lib().s5_partition(self.arena.device(self.device).data_ptr(),
                                     self.arena.size, handles.data_ptr(), n,
                                     splitters.contiguous().data_ptr(), ns, out.data_ptr(), counts,
                                     _lib.current_stream_ptr())
        _lib.check(rc, "s5_partition")
        self.launches += 3
        return out, [int(x) for x in counts]

    def lcp_pair(self, pair):
        """LCP of two strings (one-element tensor)."""
        import torch
        from . import _lib
        out = torch.empty(1, dtype=torch.int64, device=pair.device)
        rc = _lib.lib().s5_adjacent_lcp(self.arena.device(self.device).data_ptr(),
                                        self.arena.size, pair.contiguous().data_ptr(), 2,
                                        out.data_ptr(), _lib.current_stream_ptr())
        _lib.check(rc, "s5_adjacent_lcp")
        self.launches += 1
        return out

    def upload(self, host_handles):
        """Host int64 shard -> device tensor through the library's pinned u32
        staging (s5_upload_handles)."""
        import torch
        from . import _lib
        h = np.ascontiguousarray(host_handles, np.int64)
        out = torch.empty(h.size, dtype=torch.int64, device=self.device)
        rc = _lib.lib().s5_upload_handles(h.ctypes.data, h.size, self.arena.size, out.data_ptr(),
                                          _lib.current_stream_ptr())
        _lib.check(rc, "s5_upload_handles")
        return out

    def download(self, handles, lcp, out_h=None, out_l=None):
        """Device slice + LCPs -> host int64 arrays (s5_download); reuses the
        given host buffers (their leading elements) when large enough."""
        from . import _lib
        n, nl = handles.numel(), lcp.numel()
        hh = out_h[:n] if out_h is not None and out_h.size >= n else np.empty(n, np.int64)
        hl = out_l[:nl] if out_l is not None and out_l.size >= nl else np.empty(nl, np.int64)
        rc = _lib.lib().s5_download(handles.data_ptr(), hh.size, lcp.data_ptr(), hl.size,
                                    hh.ctypes.data, hl.ctypes.data if hl.size else None,
                                    _lib.current_stream_ptr())
        _lib.check(rc, "s5_download")
        return hh, hl

    def sort_u32(self, buf, n: int):
        """Sort n u32 offsets packed into the first 4n bytes of the int64
        tensor ``buf`` (the exchange payload); the sorted int64 handles land
        in ``buf`` itself (s5_sort flags bit9).  Returns (handles, lcp)."""
        import dataclasses

        import torch
        from . import _lib
        from .samplesort import SampleSortConfig, gpu_sort
        lcp = torch.empty(max(n - 1, 0), dtype=torch.int64, device=buf.device)
        if getattr(self, "keep_input", False):  # bench.py's profiled re-run of the local sort
            self.last_input = buf.view(torch.int32)[:n].to(torch.int64) & 0xFFFFFFFF
        if n == 1:
            buf.copy_(buf.view(torch.int32)[:1].to(torch.int64) & 0xFFFFFFFF)
        if n > 1:
            cfg = dataclasses.replace(self.cfg or SampleSortConfig())
            cfg.flags |= 512
            st = _lib.S5Stats()
            gpu_sort(self.arena, buf, 0, cfg, lcp, stats=st)
            self.launches += int(st.launches)
            self.last_stats = st
        return buf, lcp

    def sort(self, handles):
        """Sort a device int64 tensor in place; returns (handles, lcp)."""
        import torch
        from . import _lib
        from .samplesort import gpu_sort
        n = handles.numel()
        lcp = torch.empty(max(n - 1, 0), dtype=torch.int64, device=handles.device)
        if n > 1:
            st = _lib.S5Stats()
            gpu_sort(self.arena, handles, 0, self.cfg, lcp, stats=st)
            self.launches += int(st.launches)
        return handles, lcp


def _u64_less(a, b):
    """Unsigned a < b for int64 tensors holding uint64 bit patterns."""
    import torch
    sign = torch.tensor(-(1 << 63), dtype=torch.int64, device=a.device)
    return (a ^ sign) < (b ^ sign)


def compare_strings(backend, a, b):
    """Three-way compare of strings a[i] vs b[i] with (string, handle)
    tie-break: -1, 0, +1 per element (strings.py:64-74 order, extended)."""
    import torch
    out = torch.zeros(a.numel(), dtype=torch.int64, device=a.device)
    live = torch.arange(a.numel(), device=a.device)
    depth = 0
    while live.numel():
        ka = backend.pack_keys(a[live], depth)
        kb = backend.pack_keys(b[live], depth)
        lt = _u64_less(ka, kb)
        gt = _u64_less(kb, ka)
        out[live[lt]] = -1
        out[live[gt]] = 1
        eq = ~(lt | gt)
        # equal keys containing the terminator: identical strings -> tie-break
        w = ka[eq]
        zero = torch.zeros_like(w, dtype=torch.bool)
        for s in range(8):
            zero |= ((w >> (56 - 8 * s)) & 0xFF) == 0
        idx = live[eq]
        term = idx[zero]
        out[term] = torch.sign(a[term] - b[term])
        live = idx[~zero]
        depth += 8
    return out


@dataclass
class ShardResult:
    handles: object       # this rank's slice of the global sorted order
    lcp: object           # LCPs of the slice plus the one across the next boundary
    offset: int           # global index of handles[0]
    counts: list          # slice sizes of all ranks


def distributed_sample_sort(arena, local_handles, group=None, oversample: int = 64,
                            seed: int = 1, backend=None) -> ShardResult:
    """Globally sort the union of every rank's ``local_handles``.

    Returns this rank's contiguous slice of the global order and its LCP
    array: ``lcp[i]`` is the LCP of slice[i] and slice[i+1], and the last
    entry (absent on the last nonempty rank) is the LCP of slice[-1] and
    the next rank's first string, so concatenating all ranks' ``lcp``
    gives the global LCP array of length n-1.

    Host round trips: the partition's group sizes (one small D2H inside
    ``s5_partition``) and the G x G count matrix (one all-gather read on the
    host, which sizes the receive buffer and gives every rank all slice
    sizes); everything else stays on the device.  Handles cross the
    interconnect as u32 offsets (arena < 4 GiB) and the local sort reads
    them in place (``s5_sort`` flags bit9).
    """
    import torch
    import torch.distributed as dist

    G = dist.get_world_size(group)
    rank = dist.get_rank(group)
    be = backend or GpuBackend(arena)
    dev = local_handles.device
    h = local_handles.contiguous()
    n_local = h.numel()

    t = time.perf_counter()
    if G == 1:
        # one rank: no splitters, no count matrix, no boundary -- the shard is
        # the slice; the same u32 payload and in-place local sort as below
        recv = torch.empty(n_local, dtype=torch.int64, device=dev)
        recv.view(torch.int32)[:n_local].copy_(h)  # u32 offsets (bit pattern kept)
        t = _mark("exchange", t)
        recv, lcp = be.sort_u32(recv, n_local)
        _mark("local_sort", t)
        return ShardResult(recv, lcp, 0, [n_local])
    # 1. samples (with replacement, seeded per rank) -> all_gather
    s = oversample * G
    if n_local:  # drawn on the device (a multiplicative hash of the slot: no
        # generator object, no host round trip)
        slot = torch.arange(s, dtype=torch.int64, device=dev)
        salt = ((seed * 1_000_003 + rank) * 0x2545F4914F6CDD1D) & 0x3FFFFFFFFFFFFFFF
        pick = (slot + 1) * 0x9E3779B97F4A7C1 + salt  # wraps in int64
        pick = (pick ^ (pick >> 29)) * 0x3F58476D1CE4E5B9  # one splitmix round
        samp = h[((pick ^ (pick >> 32)) & 0x7FFFFFFFFFFFFFFF).remainder(n_local)]
    else:
        samp = torch.full((s,), -1, dtype=torch.int64, device=dev)
    allsamp = torch.empty(G * s, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allsamp, samp, group=group)
    # empty ranks' slots repeat a drawn handle, so the splitters stay strings
    # (no strings anywhere: handle 0, and every partition below is empty)
    top = allsamp.max().clamp(min=0)
    allsamp = torch.where(allsamp >= 0, allsamp, top)

    t = _mark("sample", t)
    # 2. identical splitters on every rank: sort by (string, handle)
    splitters = _pick_splitters(be, allsamp, G)
    t = _mark("splitters", t)

    # 3. destination of every local string, handles grouped by destination
    send, counts = be.partition(h, splitters)
    t = _mark("partition", t)

    # 4. the G x G count matrix on every rank (row = source, column =
    #    destination), then one exchange of u32 offsets
    mine = torch.tensor(counts, dtype=torch.int64, device=dev)
    allc = torch.empty(G * G, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allc, mine, group=group)
    M = allc.view(G, G).tolist()
    recv_sizes = [int(M[src][rank]) for src in range(G)]
    slice_sizes = [sum(int(M[src][d]) for src in range(G)) for d in range(G)]
    n_recv = slice_sizes[rank]
    recv = torch.empty(n_recv, dtype=torch.int64, device=dev)
    recv32 = recv.view(torch.int32)[:n_recv]  # the first 4 n_recv bytes
    send32 = send.to(torch.int32)  # u32 offsets (bit pattern kept)
    dist.all_to_all_single(recv32, send32, output_split_sizes=recv_sizes,
                           input_split_sizes=[int(c) for c in counts], group=group)
    t = _mark("exchange", t)

    # 5. local sort of the received u32 offsets (in place) + LCP
    recv, lcp = be.sort_u32(recv, n_recv)
    t = _mark("local_sort", t)

    # 6. boundary LCP: the next nonempty rank's first handle (one all-gather;
    #    which rank that is, every rank already knows from the count matrix)
    first = recv[:1] if n_recv else torch.full((1,), -1, dtype=torch.int64, device=dev)
    firsts = torch.empty(G, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(firsts, first.contiguous(), group=group)
    nxt = next((r for r in range(rank + 1, G) if slice_sizes[r]), None)
    if n_recv and nxt is not None:
        pair = torch.cat([recv[-1:], firsts[nxt:nxt + 1]])
        lcp = torch.cat([lcp, be.lcp_pair(pair)])
    offset = sum(slice_sizes[:rank])
    _mark("boundary", t)
    return ShardResult(recv, lcp, offset, slice_sizes)


def _pick_splitters(be, samples, G: int):
    """G-1 evenly spaced samples of the (string, handle)-sorted sample set."""
    import torch
    if G <= 1 or samples.numel() == 0:
        return samples[:0]
    s = samples.clone()
    s, lcp = be.sort(s)
    # identical strings: order by handle so every rank picks the same splitters
    # (neighbours are identical iff both end right after their common prefix)
    if s.numel() > 1:
        same = be.ends_at(s[:-1], lcp) & be.ends_at(s[1:], lcp)
        run = torch.cat([torch.zeros(1, dtype=torch.int64, device=s.device),
                         torch.cumsum((~same).to(torch.int64), 0)])
        key = run * 0  # stable two-key sort: by handle, then by run
        order = torch.argsort(s, stable=True)
        s, run = s[order], run[order]
        order = torch.argsort(run, stable=True)
        s = s[order]
        del key
    m = s.numel()
    idx = torch.tensor([(j + 1) * m // G for j in range(G - 1)], dtype=torch.int64,
                       device=s.device).clamp(max=m - 1)
    return s[idx]
