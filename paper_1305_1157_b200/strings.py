"""String arena, handles, packed keys, LCP and verification -- B200 backed.

Mirrors the reference module ``strsort.strings`` (pkg/src/strsort/strings.py):
the text lives in one contiguous byte arena in which every string is a run of
bytes 1..255 closed by one 0 terminator, and the object being sorted is an
int64 handle array of string offsets.  Key extraction, LCP and verification
run as sm_100a kernels in ``libs5.so`` (csrc/); the arena is mirrored once
into HBM (padded with zero bytes so unaligned 16-byte key loads never fault)
and cached on the ``StringArena`` object.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

#: characters per packed key word (strings.py:26)
WORD_CHARS = 8
#: zero bytes appended to the device mirror of every arena
ARENA_PAD = 128


class EmptyInput(ValueError):
    """Raised when an operation needs at least one string (strings.py:29-30)."""


class StringArena:
    """Contiguous zero-terminated character storage (strings.py:108-144).

    ``data`` is a read-only-by-convention uint8 numpy array.  In line mode each
    handle points at the byte after a terminator (or offset 0); in suffix mode
    handles may start anywhere and the arena carries exactly one terminator,
    at the very end.  ``device()`` returns the padded HBM mirror (a
    ``torch.uint8`` CUDA tensor), uploaded on first use.
    """

    __slots__ = ("_data", "_size", "_dev", "_dev_key")

    def __init__(self, data):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        if data.size and data[-1] != 0:
            raise ValueError("arena must end with a terminator byte")
        self._data = data
        self._size = int(data.size)
        self._dev = None
        self._dev_key = None

    @classmethod
    def from_device(cls, buf, size: int):
        """An arena born in HBM (``ingest_lines``, ``materialize``): ``buf`` is
        the padded CUDA mirror; ``data`` is downloaded on first access."""
        obj = cls.__new__(cls)
        obj._data = None
        obj._size = int(size)
        obj._dev = buf
        obj._dev_key = ("born", str(buf.device))
        return obj

    @property
    def data(self):
        if self._data is None:
            self._data = self._dev[: self._size].cpu().numpy()
        return self._data

    @property
    def size(self) -> int:
        """Arena bytes (without the device pad)."""
        return self._size

    @property
    def sigma(self) -> int:
        """Number of distinct non-zero byte values present."""
        present = np.bincount(self.data, minlength=256)
        return int(np.count_nonzero(present[1:]))

    def string_at(self, handle: int) -> bytes:
        """One string's bytes, terminator excluded (debugging)."""
        end = int(np.argmax(self.data[handle:] == 0)) + handle
        return self.data[handle:end].tobytes()

    def length_at(self, handle: int) -> int:
        return int(np.argmax(self.data[handle:] == 0))

    def __len__(self):
        return self._size

    def device(self, device=None):
        """Padded device mirror of the arena (uploaded once, then cached)."""
        import torch
        dev = torch.device(device if device is not None else "cuda")
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        if self._dev_key is not None and self._dev_key[0] == "born":
            if self._dev_key[1] == str(dev):
                return self._dev
            self.data  # noqa: B018 -- host copy, then a mirror on the other device
            self._dev_key = None
        key = (str(dev), self.data.ctypes.data, self.data.size)
        if self._dev is None or self._dev_key != key:
            buf = torch.zeros(self.data.size + ARENA_PAD, dtype=torch.uint8, device=dev)
            if self.data.size:
                src = self.data if self.data.flags.writeable else self.data.copy()
                buf[: self.data.size].copy_(torch.from_numpy(src), non_blocking=False)
            self._dev = buf
            self._dev_key = key
        return self._dev

    def drop_device(self):
        if self._data is None:
            self.data  # noqa: B018 -- keep the host copy of a device-born arena
        self._dev = None
        self._dev_key = None


def arena_from_strings(strings) -> tuple[StringArena, np.ndarray]:
    """Arena plus handle array from an iterable of bytes/str (strings.py:147-170).

    Embedded zero bytes are rejected; each string gets its own terminator.
    """
    chunks = []
    handles = []
    pos = 0
    for s in strings:
        if isinstance(s, str):
            s = s.encode()
        if 0 in s:
            raise ValueError("strings must not contain byte 0")
        handles.append(pos)
        chunks.append(bytes(s))
        pos += len(s) + 1
    if not handles:
        return StringArena(np.zeros(0, np.uint8)), np.zeros(0, np.int64)
    data = np.frombuffer(b"\x00".join(chunks) + b"\x00", np.uint8).copy()
    return StringArena(data), np.asarray(handles, np.int64)


@dataclass(frozen=True)
class VerifyResult:
    """strings.py:207-218."""
    ok: bool
    reason: str | None = None   # "not_permutation" | "not_sorted"
    index: int = -1

    def message(self) -> str:
        if self.ok:
            return "ok"
        if self.reason == "not_permutation":
            return f"not a permutation of the input (first offending handle {self.index})"
        return f"not sorted (first offending index {self.index})"


@dataclass(frozen=True)
class DatasetStats:
    """strings.py:240-246."""
    n: int
    N: int
    D: int
    sigma: int
    avg_len: float


# ---------------------------------------------------------------------------
# device operations (libs5.so); handles may be numpy or CUDA int64 tensors

def _to_dev_handles(handles, dev):
    import torch
    if isinstance(handles, torch.Tensor):
        return handles.to(dev, torch.int64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(handles, np.int64)).to(dev)


def _dev():
    import torch
    return torch.device("cuda", torch.cuda.current_device())


def pack_keys(arena: StringArena, handles, depth: int = 0, out=None):
    """Packed word key of every handle at ``depth`` (strings.py:176-182)."""
    import torch
    from . import _lib
    dev = handles.device if isinstance(handles, torch.Tensor) and handles.is_cuda else _dev()
    h = _to_dev_handles(handles, dev)
    keys = torch.empty(h.numel(), dtype=torch.int64, device=dev)
    if h.numel():
        rc = _lib.lib().s5_pack_keys(arena.device(dev).data_ptr(), arena.size, h.data_ptr(),
                                     h.numel(), int(depth), keys.data_ptr(),
                                     _lib.current_stream_ptr())
        _lib.check(rc, "s5_pack_keys")
    if isinstance(handles, torch.Tensor) and handles.is_cuda:
        return keys.view(torch.uint64) if hasattr(torch, "uint64") else keys
    res = keys.cpu().numpy().view(np.uint64)
    if out is not None:
        out[:] = res
        return out
    return res


def extract_key(arena: StringArena, handle: int, depth: int = 0) -> int:
    """Packed key of one string at ``depth`` (strings.py:185-191)."""
    return int(pack_keys(arena, np.asarray([handle], np.int64), depth)[0])


def adjacent_lcps(arena: StringArena, sorted_handles):
    """LCP array of a sorted handle array (_adjacent_lcps, strings.py:99-102)."""
    import torch
    from . import _lib
    dev = (sorted_handles.device if isinstance(sorted_handles, torch.Tensor)
           and sorted_handles.is_cuda else _dev())
    h = _to_dev_handles(sorted_handles, dev)
    n = h.numel()
    out = torch.empty(max(n - 1, 0), dtype=torch.int64, device=dev)
    if n > 1:
        rc = _lib.lib().s5_adjacent_lcp(arena.device(dev).data_ptr(), arena.size,
                                        h.data_ptr(), n, out.data_ptr(), _lib.current_stream_ptr())
        _lib.check(rc, "s5_adjacent_lcp")
    if isinstance(sorted_handles, torch.Tensor) and sorted_handles.is_cuda:
        return out
    return out.cpu().numpy()


def lcp(arena: StringArena, a: int, b: int) -> int:
    """Longest common prefix of two strings, terminators excluded (strings.py:194-196)."""
    return int(adjacent_lcps(arena, np.asarray([a, b], np.int64))[0])


def first_unsorted(arena: StringArena, handles) -> int:
    """First i with s[i] > s[i+1], or -1 (strings.py:77-82), on the device."""
    import torch
    from . import _lib
    dev = handles.device if isinstance(handles, torch.Tensor) and handles.is_cuda else _dev()
    h = _to_dev_handles(handles, dev)
    res = torch.empty(1, dtype=torch.int64, device=dev)
    rc = _lib.lib().s5_first_unsorted(arena.device(dev).data_ptr(), arena.size, h.data_ptr(),
                                      h.numel(), res.data_ptr(), _lib.current_stream_ptr())
    _lib.check(rc, "s5_first_unsorted")
    return int(res.item())


def verify_sorted_permutation(arena: StringArena, original, result) -> VerifyResult:
    """Permutation + sortedness check (strings.py:221-234), on the device."""
    import torch
    dev = _dev()
    if len(original) != len(result):
        return VerifyResult(False, "not_permutation", int(result[0]) if len(result) else -1)
    a = torch.sort(_to_dev_handles(original, dev)).values
    b = torch.sort(_to_dev_handles(result, dev)).values
    diff = torch.nonzero(a != b)
    if diff.numel():
        return VerifyResult(False, "not_permutation", int(b[diff[0, 0]].item()))
    bad = first_unsorted(arena, result)
    if bad >= 0:
        return VerifyResult(False, "not_sorted", bad)
    return VerifyResult(True)


def string_lengths(arena: StringArena, handles):
    """Distance from every handle to its terminator (strings.py:85-96, 249-253):
    ordered compaction of the arena's terminators + binary search (s5_string_lengths)."""
    import torch
    from . import _lib
    dev = handles.device if isinstance(handles, torch.Tensor) and handles.is_cuda else _dev()
    h = _to_dev_handles(handles, dev)
    out = torch.empty(h.numel(), dtype=torch.int64, device=dev)
    if h.numel():
        rc = _lib.lib().s5_string_lengths(arena.device(dev).data_ptr(), arena.size, h.data_ptr(),
                                          h.numel(), out.data_ptr(), _lib.current_stream_ptr())
        _lib.check(rc, "s5_string_lengths")
    if isinstance(handles, torch.Tensor) and handles.is_cuda:
        return out
    return out.cpu().numpy()


class EmbeddedNul(ValueError):
    """The input holds a 0 byte (harness.py:36-39)."""

    def __init__(self, offset: int):
        super().__init__(f"input contains byte 0 at offset {offset}")
        self.offset = offset


def ingest_lines(raw, device=None):
    """load_lines (harness.py:72-95) on the device: one string per line of
    ``raw`` (bytes / uint8 array / CUDA uint8 tensor), newlines become
    terminators, a terminator is appended after an unterminated last line.
    Returns (StringArena born in HBM, CUDA int64 handles)."""
    import ctypes as C
    import torch
    from . import _lib
    dev = torch.device(device) if device is not None else _dev()
    if isinstance(raw, torch.Tensor):
        d_raw = raw.to(dev, torch.uint8).contiguous()
    else:
        arr = np.frombuffer(raw, np.uint8) if isinstance(raw, (bytes, bytearray, memoryview)) \
            else np.ascontiguousarray(raw, np.uint8)
        d_raw = torch.from_numpy(arr.copy() if not arr.flags.writeable else arr).to(dev)
    n = d_raw.numel()
    buf = torch.zeros(n + 1 + ARENA_PAD, dtype=torch.uint8, device=dev)
    handles = torch.empty(n + 2, dtype=torch.int64, device=dev)
    hn, hlen, hnul = C.c_uint64(0), C.c_uint64(0), C.c_int64(-1)
    rc = _lib.lib().s5_ingest_lines(d_raw.data_ptr(), n, buf.data_ptr(), handles.data_ptr(),
                                    C.byref(hn), C.byref(hlen), C.byref(hnul),
                                    _lib.current_stream_ptr())
    if rc != 0 and hnul.value >= 0:
        raise EmbeddedNul(int(hnul.value))
    _lib.check(rc, "s5_ingest_lines")
    return StringArena.from_device(buf, hlen.value), handles[: hn.value]


def load_lines(path, device=None):
    """load_lines (harness.py:83-95): read the file, ingest on the device."""
    with open(path, "rb") as f:
        raw = f.read()
    return ingest_lines(raw, device)


def materialize(arena: StringArena, sorted_handles):
    """The strings of ``sorted_handles`` gathered in order into a new arena
    (strings_of, tests/helpers.py:62-68), on the device.
    Returns (StringArena born in HBM, CUDA int64 handles into it)."""
    import ctypes as C
    import torch
    from . import _lib
    dev = (sorted_handles.device if isinstance(sorted_handles, torch.Tensor)
           and sorted_handles.is_cuda else _dev())
    h = _to_dev_handles(sorted_handles, dev)
    n = h.numel()
    out_h = torch.empty(n, dtype=torch.int64, device=dev)
    need = C.c_uint64(0)
    ad = arena.device(dev).data_ptr()
    L = _lib.lib()
    # size, then gather
    rc = L.s5_materialize(ad, arena.size, h.data_ptr(), n, None, 0, out_h.data_ptr(),
                          C.byref(need), _lib.current_stream_ptr())
    if rc not in (0, -3):
        _lib.check(rc, "s5_materialize")
    buf = torch.zeros(need.value + ARENA_PAD, dtype=torch.uint8, device=dev)
    rc = L.s5_materialize(ad, arena.size, h.data_ptr(), n, buf.data_ptr(), need.value,
                          out_h.data_ptr(), C.byref(need), _lib.current_stream_ptr())
    _lib.check(rc, "s5_materialize")
    return StringArena.from_device(buf, need.value), out_h


def distinguishing_prefix(arena: StringArena, sorted_handles, lcp_arr=None) -> int:
    """D = sum min(|s|+1, max(lcp_prev, lcp_next)+1) over a sorted order
    (compute_stats, strings.py:256-284); uses a given LCP array if supplied."""
    import torch
    dev = _dev()
    h = _to_dev_handles(sorted_handles, dev)
    n = h.numel()
    if n == 0:
        raise EmptyInput("compute_stats needs at least one string")
    lens = string_lengths(arena, h)
    if n == 1:
        return int(min(int(lens[0].item()) + 1, 1))
    if lcp_arr is None:
        lcp_arr = adjacent_lcps(arena, h)
    l = _to_dev_handles(lcp_arr, dev)
    best = torch.zeros(n, dtype=torch.int64, device=dev)
    best[:-1] = l
    best[1:] = torch.maximum(best[1:], l)
    return int(torch.minimum(lens + 1, best + 1).sum().item())


def compute_stats(arena: StringArena, handles, sorted_handles=None) -> DatasetStats:
    """n, N, D, sigma, mean length (strings.py:256-284); sorts on the GPU if needed."""
    n = int(len(handles))
    if n == 0:
        raise EmptyInput("compute_stats needs at least one string")
    lens = string_lengths(arena, handles)
    lens = lens.cpu().numpy() if hasattr(lens, "cpu") else lens
    total = int(lens.sum()) + n
    if sorted_handles is None:
        from .samplesort import parallel_sample_sort
        sorted_handles = np.array(handles, np.int64, copy=True)
        parallel_sample_sort(arena, sorted_handles)
    D = distinguishing_prefix(arena, sorted_handles)
    return DatasetStats(n, total, D, arena.sigma, float(lens.mean()))
