"""Pin the CPU oracle (oracle/s5_oracle.c) against the reference's own outputs.

Fixtures come from tests/golden/make_golden.py, which ran the reference
package itself; the config-1 digests are the reference outputs quoted in
SURVEY.md 8(d).  CPU only.
"""
import numpy as np
import pytest

import oracle as O
from paper_1305_1157_b200 import datasets
from paper_1305_1157_b200.strings import StringArena


@pytest.mark.parametrize("workers", [1, 3])
def test_oracle_parallel_sort_matches_reference(sort_cases, workers):
    for name, c in sort_cases.items():
        arena = StringArena(c["arena"])
        h = c["handles"].copy()
        O.parallel_sample_sort(arena, h, workers)
        assert O.contents_equal(arena, h, c["sorted"]), name
        assert np.array_equal(np.sort(h), np.sort(c["handles"])), name
        assert np.array_equal(O.adjacent_lcps(arena, h), c["lcp"]), name
        if h.size:
            assert O.distinguishing_prefix(arena, h) == int(c["D"]), name


def test_oracle_sequential_sort_matches_reference(sort_cases):
    cfg = O.OracleConfig(v=15, t_m=256, t_i=16, seed=3)
    for name, c in sort_cases.items():
        arena = StringArena(c["arena"])
        h = c["handles"].copy()
        O.sample_sort(arena, h, cfg=cfg)
        assert O.contents_equal(arena, h, c["sorted"]), name
        assert O.first_unsorted(arena, h) == -1


def test_oracle_lcp_of_reference_order(sort_cases):
    for name, c in sort_cases.items():
        arena = StringArena(c["arena"])
        assert np.array_equal(O.adjacent_lcps(arena, c["sorted"]), c["lcp"]), name


def test_oracle_classifier_matches_reference(classifier_cases):
    for name, c in classifier_cases.items():
        spl = c["splitters"]
        if name != "cterm":
            assert np.array_equal(O.select_splitters(c["sample"], spl.size), spl), name
        lo, lcps, term, d = O.build_tree(spl)
        assert np.array_equal(lo, c["level_order"]), name
        assert np.array_equal(lcps, c["splitter_lcp"]), name
        assert np.array_equal(term, c["terminated"]), name
        want = c["buckets"]
        assert np.array_equal(O.classify_oracle(c["keys"], spl), want), name
        assert np.array_equal(O.classify_unrolled(c["keys"], spl).astype(np.int64), want), name
        assert np.array_equal(O.classify_equal(c["keys"], spl).astype(np.int64), want), name
        if name != "cterm":
            counts = np.bincount(want, minlength=2 * spl.size + 1)
            bnd, delta, fin = O.bucket_layout(counts, spl)
            assert np.array_equal(bnd, c["boundaries"]), name
            assert np.array_equal(delta, c["depth_delta"]), name
            assert np.array_equal(fin, c["finished"]), name


def test_oracle_pack_keys_matches_reference():
    import os
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "pack_keys.npz"))
    arena = z["arena"]
    for depth in range(17):
        h = z[f"d{depth}__handles"]
        assert np.array_equal(O.pack_keys(arena, h, depth), z[f"d{depth}__keys"]), depth


def test_reference_kats():
    # inline known answers of the reference suite
    arena = StringArena(np.frombuffer(b"ab\x00", np.uint8).copy())
    assert O.pack_keys(arena, np.zeros(1, np.int64))[0] == 0x6162_0000_0000_0000  # test_strings.py:15-17
    lo, _, _, _ = O.build_tree(np.asarray([10, 20, 30], np.uint64))
    assert lo[1:].tolist() == [20, 10, 30]                                    # test_classifier.py:92-94
    spl = np.asarray([100, 200, 300], np.uint64)
    cases = {50: 0, 100: 1, 150: 2, 200: 3, 250: 4, 300: 5, 400: 6}           # test_classifier.py:153-158
    assert O.classify_oracle(np.asarray(list(cases), np.uint64), spl).tolist() == list(cases.values())
    bnd, delta, _ = O.bucket_layout(np.asarray([2, 3, 4]), np.asarray([50], np.uint64))
    assert bnd.tolist() == [0, 2, 5, 9] and delta.tolist() == [0, 8, 0]       # test_classifier.py:247-251
    assert [O.effective_v(8191, s) for s in (200_000, 16, 2)] == [8191, 7, 1]  # :281-285
    assert O.effective_v(3, 1000) == 3


def test_oracle_config1_reproduces_reference_digests():
    arena, h = datasets.generate(1)
    n, N, D = datasets.EXPECTED[1]
    assert h.size == n and arena.data.size == N
    s = h.copy()
    O.parallel_sample_sort(arena, s, 4)
    assert O.distinguishing_prefix(arena, s) == D
    ds, dl = datasets.DIGESTS[1]
    assert O.digest_strings(arena, s)[:16] == ds
    assert O.digest_lcp(O.adjacent_lcps(arena, s))[:16] == dl
