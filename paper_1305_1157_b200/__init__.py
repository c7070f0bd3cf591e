"""B200-native super scalar string sample sort (S^5, arXiv 1305.1157).

Drop-in for the S^5 path of the reference package ``strsort``
(pkg/src/strsort/__init__.py:22-30): the same entry points and records,
executed by hand-written sm_100a kernels in ``libs5.so`` through a C-ABI
(include/s5.h) bound with ctypes.  New: the LCP array of the sorted order
(``sort_with_lcp``, ``lcp_out=``).
"""

from .counters import Counters
from .samplesort import (SampleSortConfig, gpu_sort, parallel_sample_sort, sample_sort,
                         sort_with_lcp)
from .strings import (DatasetStats, EmbeddedNul, EmptyInput, StringArena, VerifyResult,
                      WORD_CHARS, adjacent_lcps, arena_from_strings, compute_stats,
                      distinguishing_prefix, extract_key, first_unsorted, ingest_lines, lcp,
                      load_lines, materialize, pack_keys, string_lengths,
                      verify_sorted_permutation)

__all__ = [
    "Counters", "DatasetStats", "EmbeddedNul", "EmptyInput", "SampleSortConfig", "StringArena",
    "VerifyResult", "WORD_CHARS", "adjacent_lcps", "arena_from_strings", "compute_stats",
    "distinguishing_prefix", "extract_key", "first_unsorted", "gpu_sort", "ingest_lines", "lcp",
    "load_lines", "materialize", "pack_keys",
    "parallel_sample_sort", "sample_sort", "sort_with_lcp", "string_lengths",
    "verify_sorted_permutation",
]
