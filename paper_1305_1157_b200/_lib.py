"""ctypes binding of libs5.so (C-ABI declared in include/s5.h).

There is no fallback: if the shared library is missing or fails to load, every
entry point raises.  ``build()`` compiles it in-tree with nvcc for sm_100a.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# S5_LIB: an alternative build of the same library (A/B timing of kernel variants)
SO_PATH = os.environ.get("S5_LIB") or os.path.join(_HERE, "libs5.so")
CSRC = os.path.join(_HERE, "csrc")

S5_ARENA_PAD = 128
S5_MAX_LEVELS = 128

ERRORS = {
    -1: ValueError,       # S5_E_INVALID
    -2: RuntimeError,     # S5_E_CUDA
    -3: RuntimeError,     # S5_E_WORKSPACE
    -4: ValueError,       # S5_E_RANGE
    -5: RuntimeError,     # S5_E_INTERNAL
    -6: RuntimeError,     # S5_E_NCCL
}


class S5Config(C.Structure):
    _fields_ = [("v", C.c_uint32), ("alpha", C.c_uint32), ("classifier", C.c_uint32),
                ("small_max", C.c_uint32), ("narrow_max", C.c_uint32), ("flags", C.c_uint32),
                ("seed", C.c_uint64), ("local_max", C.c_uint32), ("wide_v", C.c_uint32),
                ("wide_target", C.c_uint32), ("local_target", C.c_uint32)]


S5_MAX_LAUNCH_RECS = 512


class S5LaunchRec(C.Structure):
    _fields_ = [("kernel", C.c_uint32), ("level", C.c_uint32), ("strings", C.c_uint64),
                ("ms", C.c_float), ("start_ms", C.c_float)]


class S5Stats(C.Structure):
    _fields_ = [("levels", C.c_uint32), ("pad_", C.c_uint32),
                ("n_per_pass", C.c_uint64 * S5_MAX_LEVELS),
                ("wide_elems", C.c_uint64 * S5_MAX_LEVELS),
                ("narrow_elems", C.c_uint64 * S5_MAX_LEVELS),
                ("small_elems", C.c_uint64 * S5_MAX_LEVELS),
                ("wide_steps", C.c_uint64), ("narrow_steps", C.c_uint64),
                ("small_segments", C.c_uint64), ("key_fetches", C.c_uint64),
                ("boundary_lcps", C.c_uint64), ("launches", C.c_uint64),
                ("ms_total", C.c_float), ("pad2_", C.c_float),
                ("kern_ms", C.c_float * 16), ("kern_launches", C.c_uint32 * 16),
                ("local_elems", C.c_uint64 * S5_MAX_LEVELS), ("local_steps", C.c_uint64),
                ("kern_strings", C.c_uint64 * 16), ("n_launch_recs", C.c_uint32),
                ("pad3_", C.c_uint32), ("host_h2d_ms", C.c_float), ("host_sort_ms", C.c_float),
                ("host_d2h_ms", C.c_float), ("pad4_", C.c_float),
                ("launch_recs", S5LaunchRec * S5_MAX_LAUNCH_RECS),
                ("host_h2d_bytes", C.c_uint64), ("host_d2h_bytes", C.c_uint64)]

    def as_dict(self) -> dict:
        L = min(self.levels, S5_MAX_LEVELS)
        return {
            "levels": int(self.levels),
            "n_per_pass": [int(x) for x in self.n_per_pass[:L]],
            "wide_elems": [int(x) for x in self.wide_elems[:L]],
            "narrow_elems": [int(x) for x in self.narrow_elems[:L]],
            "small_elems": [int(x) for x in self.small_elems[:L]],
            "local_elems": [int(x) for x in self.local_elems[:L]],
            "local_steps": int(self.local_steps),
            "wide_steps": int(self.wide_steps), "narrow_steps": int(self.narrow_steps),
            "small_segments": int(self.small_segments), "key_fetches": int(self.key_fetches),
            "boundary_lcps": int(self.boundary_lcps), "ms_total": float(self.ms_total),
            "launches": int(self.launches),
            "host_ms": {"h2d": float(self.host_h2d_ms), "sort": float(self.host_sort_ms),
                        "d2h": float(self.host_d2h_ms)},
            "launch_recs": [(KERNELS[r.kernel] if r.kernel < len(KERNELS) else str(r.kernel),
                             int(r.level), int(r.strings), round(float(r.ms), 4),
                             round(float(r.start_ms), 4))
                            for r in self.launch_recs[:min(self.n_launch_recs, S5_MAX_LAUNCH_RECS)]],
            "kernels": {KERNELS[i]: {"ms": float(self.kern_ms[i]),
                                     "launches": int(self.kern_launches[i]),
                                     "strings": int(self.kern_strings[i])}
                        for i in range(len(KERNELS)) if self.kern_launches[i]},
        }


KERNELS = ["k_gather", "k_wide_plan", "k_wide_tree", "k_wide_count", "k_wide_colscan",
           "k_wide_bscan", "k_wide_scatter", "k_narrow", "k_small", "k_lcp_fix", "k_init_root",
           "k_local", "k_local_s", "k_local_m", "k_local_xs", "k_local_w"]

_vp = C.c_void_p
_u64 = C.c_uint64
_u32 = C.c_uint32


class S5Segment(C.Structure):
    _fields_ = [("begin", C.c_uint32), ("size", C.c_uint32), ("depth", C.c_uint32),
                ("side", C.c_uint32)]


AUDIT_FN = C.CFUNCTYPE(None, _vp, _u32, C.POINTER(S5Segment), _u64, C.POINTER(_u32),
                       C.POINTER(_u32), _u64)

SIGNATURES = {
    "s5_workspace_bytes": (_u64, [_u64, _u64, C.POINTER(S5Config)]),
    "s5_sort": (C.c_int, [_vp, _u64, _vp, _u64, _u64, _vp, C.POINTER(S5Config), _vp, _u64, _vp,
                          C.POINTER(S5Stats)]),
    "s5_sort_audit": (C.c_int, [_vp, _u64, _vp, _u64, _u64, _vp, C.POINTER(S5Config), _vp, _u64,
                                _vp, C.POINTER(S5Stats), AUDIT_FN, _vp]),
    "s5_sort_host": (C.c_int, [_vp, _u64, _vp, _u64, _u64, _vp, C.POINTER(S5Config), _vp,
                               C.POINTER(S5Stats)]),
    "s5_pack_keys": (C.c_int, [_vp, _u64, _vp, _u64, _u64, _vp, _vp]),
    "s5_adjacent_lcp": (C.c_int, [_vp, _u64, _vp, _u64, _vp, _vp]),
    "s5_first_unsorted": (C.c_int, [_vp, _u64, _vp, _u64, _vp, _vp]),
    "s5_partition": (C.c_int, [_vp, _u64, _vp, _u64, _vp, C.c_uint32, _vp, _vp, _vp]),
    "s5_sort_multi": (C.c_int, [C.c_int, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp,
                                C.POINTER(S5Config), C.POINTER(S5Stats)]),
    "s5_ingest_lines": (C.c_int, [_vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "s5_release_caches": (C.c_int, []),
    "s5_upload_handles": (C.c_int, [_vp, _u64, _u64, _vp, _vp]),
    "s5_download": (C.c_int, [_vp, _u64, _vp, _u64, _vp, _vp, _vp]),
    "s5_string_lengths": (C.c_int, [_vp, _u64, _vp, _u64, _vp, _vp]),
    "s5_materialize": (C.c_int, [_vp, _u64, _vp, _u64, _vp, _u64, _vp, _vp, _vp]),
    "s5_classify": (C.c_int, [_vp, _u64, _vp, _u32, _u32, _vp, _vp]),
    "s5_build_tree": (C.c_int, [_vp, _u32, _u32, _vp, _vp, _vp]),
    "s5_host_markov_text": (C.c_int, [_vp, _vp, _u64, _u32, _vp]),
    "s5_host_copy_pieces": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _u64]),
    "s5_last_error": (C.c_char_p, []),
    "s5_version": (C.c_int, []),
}

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile libs5.so in-tree (nvcc -gencode arch=compute_100a,code=sm_100a)."""
    cmd = ["make", "-s", "-C", CSRC]
    if force:
        cmd.insert(1, "-B")
    subprocess.run(cmd, check=True)
    return SO_PATH


def lib():
    """The loaded library; raises if it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(SO_PATH):
                    raise ImportError(
                        f"{SO_PATH} is missing: build it with paper_1305_1157_b200._lib.build() "
                        "(nvcc, sm_100a); there is no CPU fallback")
                L = C.CDLL(SO_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().s5_last_error().decode(errors="replace")
        raise ERRORS.get(rc, RuntimeError)(f"{what}: {msg} (code {rc})")


def current_stream_ptr():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)
