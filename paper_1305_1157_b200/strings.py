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
ARENA_PAD = 64


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

    __slots__ = ("data", "_dev", "_dev_key")

    def __init__(self, data):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        if data.size and data[-1] != 0:
            raise ValueError("arena must end with a terminator byte")
        self.data = data
        self._dev = None
        self._dev_key = None

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
        return self.data.size

    def device(self, device=None):
        """Padded device mirror of the arena (uploaded once, then cached)."""
        import torch
        dev = torch.device(device if device is not None else "cuda")
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        key = (str(dev), self.data.ctypes.data, self.data.size)
        if self._dev is None or self._dev_key != key:
            buf = torch.zeros(self.data.size + ARENA_PAD, dtype=torch.uint8, device=dev)
            if self.data.size:
                buf[: self.data.size].copy_(torch.from_numpy(self.data), non_blocking=False)
            self._dev = buf
            self._dev_key = key
        return self._dev

    def drop_device(self):
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
