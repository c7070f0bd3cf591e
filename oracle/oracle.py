"""ctypes front-end of the C oracle (test infrastructure only; see __init__)."""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
from dataclasses import dataclass

import numpy as np

__all__ = [
    "OracleConfig", "lib", "build", "pack_keys", "lcp", "compare", "first_unsorted",
    "string_lengths", "adjacent_lcps", "distinguishing_prefix", "effective_v",
    "select_splitters", "build_tree", "classify_oracle", "classify_unrolled",
    "classify_equal", "bucket_layout", "insertion_sort", "mkqs_cache_sort",
    "sample_sort", "parallel_sample_sort", "same_contents", "contents_equal",
    "digest_strings", "digest_lcp", "max_threads",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "libs5oracle.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_i64 = C.c_int64


class _Cfg(C.Structure):
    _fields_ = [(f, C.c_int64) for f in
                ("v", "alpha", "t_m", "t_i", "classifier", "interleave", "seed")]


@dataclass
class OracleConfig:
    """Mirror of SampleSortConfig (samplesort.py:37-45)."""
    v: int = 8191
    alpha: int = 2
    t_m: int = 64 * 1024
    t_i: int = 64
    classifier: str = "unroll"
    interleave: int = 3
    seed: int = 1

    def c(self) -> _Cfg:
        return _Cfg(self.v, self.alpha, self.t_m, self.t_i,
                    1 if self.classifier == "equal" else 0, self.interleave, self.seed)


def build() -> str:
    """Compile the oracle with its Makefile (gcc; no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
                os.path.join(_HERE, "s5_oracle.c")):
            build()
        L = C.CDLL(_SO)
        sig = {
            "or_pack_one": (C.c_uint64, [_u8p, _i64]),
            "or_pack_keys": (None, [_u8p, _i64p, _i64, _i64, _u64p]),
            "or_lcp_pair": (_i64, [_u8p, _i64, _i64]),
            "or_compare_from": (C.c_int, [_u8p, _i64, _i64, _i64]),
            "or_first_unsorted": (_i64, [_u8p, _i64p, _i64]),
            "or_string_lengths": (C.c_int, [_u8p, _i64, _i64p, _i64, _i64p]),
            "or_adjacent_lcps": (None, [_u8p, _i64p, _i64, _i64p]),
            "or_distinguishing_prefix": (_i64, [_u8p, _i64, _i64p, _i64]),
            "or_effective_v": (_i64, [_i64, _i64]),
            "or_select_splitters": (None, [_u64p, _i64, _i64, _u64p]),
            "or_build_tree": (C.c_int, [_u64p, _i64, _u64p, _i64p,
                                        np.ctypeslib.ndpointer(np.uint8)]),
            "or_classify_oracle": (None, [_u64p, _i64, _u64p, _i64, _i64p]),
            "or_classify_unrolled": (None, [_u64p, _i64, _u64p, _u64p, C.c_int, C.c_int, _u16p]),
            "or_classify_equal": (None, [_u64p, _i64, _u64p, _u64p, C.c_int, _u16p]),
            "or_bucket_layout": (None, [_i64p, _i64, _i64p, _u8p, _i64p, _i64p, _u8p]),
            "or_insertion_sort": (None, [_u8p, _i64p, _i64, _i64]),
            "or_mkqs_cache_sort": (C.c_int, [_u8p, _i64p, _i64, _i64, _i64, C.c_void_p]),
            "or_sample_sort": (C.c_int, [_u8p, _i64p, _i64, _i64, C.POINTER(_Cfg), _i64p]),
            "or_parallel_sample_sort": (C.c_int, [_u8p, _i64p, _i64, C.c_int,
                                                  C.POINTER(_Cfg), _i64p]),
            "or_same_contents": (_i64, [_u8p, _i64p, _i64p, _i64]),
            "or_gather_strings": (_i64, [_u8p, _i64p, _i64, _i64, _i64, _u8p, _i64,
                                         C.POINTER(_i64)]),
            "or_max_threads": (C.c_int, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _data(arena) -> np.ndarray:
    d = getattr(arena, "data", arena)
    return np.ascontiguousarray(d, np.uint8)


def _h(handles) -> np.ndarray:
    return np.ascontiguousarray(handles, np.int64)


def max_threads() -> int:
    return int(lib().or_max_threads())


def pack_keys(arena, handles, depth: int = 0) -> np.ndarray:
    h = _h(handles)
    out = np.empty(h.size, np.uint64)
    if h.size:
        lib().or_pack_keys(_data(arena), h, h.size, depth, out)
    return out


def lcp(arena, a: int, b: int) -> int:
    return int(lib().or_lcp_pair(_data(arena), a, b))


def compare(arena, a: int, b: int, depth: int = 0) -> int:
    return int(lib().or_compare_from(_data(arena), a, b, depth))


def first_unsorted(arena, handles) -> int:
    h = _h(handles)
    return int(lib().or_first_unsorted(_data(arena), h, h.size))


def string_lengths(arena, handles) -> np.ndarray:
    d = _data(arena)
    h = _h(handles)
    out = np.empty(h.size, np.int64)
    if h.size:
        lib().or_string_lengths(d, d.size, h, h.size, out)
    return out


def adjacent_lcps(arena, sorted_handles) -> np.ndarray:
    h = _h(sorted_handles)
    out = np.empty(max(h.size - 1, 0), np.int64)
    if h.size > 1:
        lib().or_adjacent_lcps(_data(arena), h, h.size, out)
    return out


def distinguishing_prefix(arena, sorted_handles) -> int:
    d = _data(arena)
    h = _h(sorted_handles)
    r = int(lib().or_distinguishing_prefix(d, d.size, h, h.size))
    if r == -2:
        raise ValueError("distinguishing prefix needs at least one string")
    if r < 0:
        raise MemoryError("oracle allocation failed")
    return r


def effective_v(v_max: int, size: int) -> int:
    return int(lib().or_effective_v(v_max, size))


def select_splitters(sample, v: int) -> np.ndarray:
    s = np.ascontiguousarray(sample, np.uint64)
    out = np.empty(v, np.uint64)
    lib().or_select_splitters(s, s.size, v, out)
    return out


def build_tree(in_order):
    """Returns (level_order[v+1], splitter_lcp[v], terminated[v], d)."""
    io = np.ascontiguousarray(in_order, np.uint64)
    v = io.size
    lo = np.zeros(v + 1, np.uint64)
    lcps = np.zeros(max(v, 1), np.int64)
    term = np.zeros(max(v, 1), np.uint8)
    d = lib().or_build_tree(io, v, lo, lcps, term)
    if d < 0:
        raise ValueError(f"need 2**d - 1 splitters, got {v}")
    return lo, lcps[:v], term[:v].astype(bool), d


def classify_oracle(keys, in_order) -> np.ndarray:
    k = np.ascontiguousarray(np.atleast_1d(keys), np.uint64)
    io = np.ascontiguousarray(in_order, np.uint64)
    out = np.empty(k.size, np.int64)
    if k.size:
        lib().or_classify_oracle(k, k.size, io, io.size, out)
    return out


def classify_unrolled(keys, in_order, interleave: int = 3) -> np.ndarray:
    k = np.ascontiguousarray(keys, np.uint64)
    io = np.ascontiguousarray(in_order, np.uint64)
    lo, _, _, d = build_tree(io)
    out = np.empty(k.size, np.uint16)
    if k.size:
        lib().or_classify_unrolled(k, k.size, lo, io, d, interleave, out)
    return out


def classify_equal(keys, in_order) -> np.ndarray:
    k = np.ascontiguousarray(keys, np.uint64)
    io = np.ascontiguousarray(in_order, np.uint64)
    lo, _, _, d = build_tree(io)
    out = np.empty(k.size, np.uint16)
    if k.size:
        lib().or_classify_equal(k, k.size, lo, io, d, out)
    return out


def bucket_layout(counts, in_order):
    """Returns (boundaries, depth_delta, finished) per classifier.py:284-304."""
    io = np.ascontiguousarray(in_order, np.uint64)
    _, lcps, term, _ = build_tree(io)
    c = np.ascontiguousarray(counts, np.int64)
    k = 2 * io.size + 1
    bnd = np.zeros(k + 1, np.int64)
    delta = np.zeros(k, np.int64)
    fin = np.zeros(k, np.uint8)
    lib().or_bucket_layout(c, io.size, np.ascontiguousarray(lcps, np.int64),
                           np.ascontiguousarray(term, np.uint8), bnd, delta, fin)
    return bnd, delta, fin.astype(bool)


def insertion_sort(arena, handles, depth: int = 0):
    h = _h(handles)
    lib().or_insertion_sort(_data(arena), h, h.size, depth)
    return h


def mkqs_cache_sort(arena, handles, depth: int = 0, t_i: int = 64):
    h = _h(handles)
    if lib().or_mkqs_cache_sort(_data(arena), h, h.size, depth, t_i, None):
        raise MemoryError("oracle allocation failed")
    return h


def sample_sort(arena, handles, depth: int = 0, cfg: OracleConfig | None = None):
    """Sequential S^5 (samplesort.py:241-267); sorts ``handles`` in place."""
    h = _h(handles)
    assert h is handles or not isinstance(handles, np.ndarray) or handles.dtype == np.int64
    c = (cfg or OracleConfig()).c()
    ctr = np.zeros(3, np.int64)
    if lib().or_sample_sort(_data(arena), h, h.size, depth, C.byref(c), ctr):
        raise MemoryError("oracle allocation failed")
    return h


def parallel_sample_sort(arena, handles, workers: int = 1, cfg: OracleConfig | None = None):
    """Fully parallel S^5 port (samplesort.py:273-444); sorts in place."""
    h = _h(handles)
    c = (cfg or OracleConfig()).c()
    ctr = np.zeros(3, np.int64)
    if lib().or_parallel_sample_sort(_data(arena), h, h.size, int(workers), C.byref(c), ctr):
        raise MemoryError("oracle allocation failed")
    return h


def same_contents(arena, a, b) -> int:
    a = _h(a)
    b = _h(b)
    if a.size != b.size:
        return 0
    return int(lib().or_same_contents(_data(arena), a, b, a.size))


def contents_equal(arena, got, expected) -> bool:
    """helpers.py:95-103: positionwise string-content equality."""
    got = _h(got)
    expected = _h(expected)
    if got.size != expected.size:
        return False
    return got.size == 0 or same_contents(arena, got, expected) == -1


def digest_strings(arena, sorted_handles, maxlen: int = -1, chunk: int = 1 << 26) -> str:
    """sha256 over the sorted strings, each followed by its 0 terminator
    (truncated to ``maxlen`` bytes first when maxlen >= 0): SURVEY.md 8(d)."""
    d = _data(arena)
    h = _h(sorted_handles)
    buf = np.empty(chunk, np.uint8)
    used = _i64(0)
    sha = hashlib.sha256()
    i = 0
    while i < h.size:
        took = lib().or_gather_strings(d, h, h.size, i, maxlen, buf, chunk, C.byref(used))
        if took == 0:
            raise ValueError("string longer than digest chunk")
        sha.update(buf[:used.value].tobytes())
        i += took
    return sha.hexdigest()


def digest_lcp(lcp_arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(lcp_arr, "<i8").tobytes()).hexdigest()
