"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (the reference tree does not exist on the GPU
box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports ``strsort`` from /root/reference/pkg/src (read-only; numba caches
are redirected to /tmp) and the reference test helpers for the dataset
builders, runs the reference's own ``parallel_sample_sort`` / ``sample_sort``
and ``_adjacent_lcps`` / ``compute_stats`` on the SPEC.md acceptance-sweep
shapes (scaled down), and writes compressed ``.npz`` fixtures next to this
script.  The fixtures pin both the CPU oracle (tests/test_oracle_golden.py)
and the B200 library (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.path.join(REF, "src"))
    sys.path.insert(0, os.path.join(REF, "tests"))
    import strsort  # noqa: F401
    import helpers  # noqa: F401
    return strsort, helpers


def sort_cases(strsort, helpers):
    from strsort import arena_from_strings, StringArena
    from strsort.harness import generate_dna, generate_random
    cases = {}
    H = helpers
    cases["random_10"] = arena_from_strings(H.random_strings(10, seed=10))
    cases["random_1000"] = arena_from_strings(H.random_strings(1000, seed=11))
    cases["random_20000"] = arena_from_strings(H.random_strings(20000, seed=12))
    cases["identical_3000"] = H.identical_dataset(3000, length=17)
    cases["identical_long_500"] = H.identical_dataset(500, length=100)
    cases["empty_1000"] = H.empty_dataset(1000)
    cases["shared_prefix_2000"] = H.shared_prefix_dataset(2000, prefix_len=1000, seed=3)
    cases["low_alphabet_30000"] = arena_from_strings(
        H.random_strings(30000, seed=9, lo=97, hi=99, max_len=25))
    cases["dna9_20000"] = generate_dna(20000, 9, seed=4)
    cases["harness_random_50000"] = generate_random(50000, seed=5)
    text = H.word_text(40000, seed=6)
    cases["suffix_words_40000"] = (StringArena(np.frombuffer(text + b"\x00", np.uint8).copy()),
                                   np.arange(len(text), dtype=np.int64))
    rng = np.random.default_rng(7)
    hi_bytes = [bytes(rng.integers(1, 256, rng.integers(0, 12)).tolist()) for _ in range(4000)]
    cases["binary_bytes_4000"] = arena_from_strings(hi_bytes)
    cases["appendix_a"] = arena_from_strings(
        [b"\xff", b"a", b"", b"ab", b"\x80z", b"\x01", b"a", b""])
    chain = [b"a" * i for i in range(40)] + [b"a" * i + b"b" for i in range(40)]
    rng.shuffle(chain)
    cases["prefix_chain_80"] = arena_from_strings(chain)
    dup = H.random_strings(3000, seed=13, max_len=30)
    dup = dup + dup[:1500] + dup[:700]
    cases["dups_5200"] = arena_from_strings(dup)
    return cases


def main():
    strsort, H = _import_reference()
    from strsort import SampleSortConfig, compute_stats, parallel_sample_sort, sample_sort
    from strsort.strings import _adjacent_lcps
    out = {}
    for name, (arena, handles) in sort_cases(strsort, H).items():
        n = handles.size
        par = handles.copy()
        parallel_sample_sort(arena, par, 4)
        small = handles.copy()
        parallel_sample_sort(arena, small, 2, cfg=SampleSortConfig(v=15, t_m=256, t_i=16, seed=3))
        seq = handles.copy()
        sample_sort(arena, seq)
        lcp = np.empty(max(n - 1, 0), np.int64)
        if n > 1:
            _adjacent_lcps(arena.data, par, lcp)
        D = compute_stats(arena, handles, sorted_handles=par).D if n else 0
        assert H.contents_equal(arena, par, seq) and H.contents_equal(arena, par, small)
        out[name] = dict(arena=arena.data, handles=handles, sorted=par, lcp=lcp,
                         D=np.int64(D))
        print(f"{name:24s} n={n:6d} N={arena.data.size:8d} D={D}")
    np.savez_compressed(os.path.join(HERE, "sort_cases.npz"),
                        **{f"{k}__{f}": v for k, d in out.items() for f, v in d.items()})

    # classifier known answers from the reference (classifier.py)
    from strsort.classifier import (bucket_layout, build_tree, classify_oracle,
                                    classify_tree_equal, classify_tree_unrolled,
                                    select_splitters)
    rng = np.random.default_rng(2024)
    cls = {}
    for t, (v, dup, lo, hi) in enumerate([(1, False, 0, 50), (3, True, 0, 40), (7, True, 0, 40),
                                          (63, False, 0, 2**63), (255, True, 0, 300),
                                          (8191, False, 0, 2**63), (8191, True, 0, 5000)]):
        sample = np.sort(rng.integers(lo, hi, 2 * v, dtype=np.uint64))
        if dup:
            sample[: v // 2] = sample[0]
            sample = np.sort(sample)
        spl = select_splitters(sample, v)
        tree = build_tree(spl)
        keys = np.concatenate([rng.integers(lo, hi, 20000, dtype=np.uint64), spl,
                               spl + np.uint64(1), np.asarray([0, 2**64 - 1], np.uint64)])
        want = classify_oracle(keys, spl)
        assert np.array_equal(classify_tree_unrolled(keys, tree).astype(np.int64), want)
        assert np.array_equal(classify_tree_equal(keys, tree).astype(np.int64), want)
        counts = np.bincount(want, minlength=2 * v + 1)
        lay = bucket_layout(counts, tree, 0)
        cls[f"c{t}"] = dict(sample=sample, splitters=spl, level_order=tree.level_order,
                            splitter_lcp=tree.splitter_lcp, terminated=tree.terminated,
                            keys=keys, buckets=want, boundaries=lay.boundaries,
                            depth_delta=lay.depth_delta, finished=lay.finished)
    # terminated-splitter case built from real strings
    from strsort import arena_from_strings, pack_keys
    a, h = arena_from_strings([b"ab", b"cd", b"longenough", b"x", b"abcdefgh", b"abcdefg"])
    k = np.sort(pack_keys(a, h))[:3]
    tree = build_tree(k)
    cls["cterm"] = dict(sample=k, splitters=k, level_order=tree.level_order,
                        splitter_lcp=tree.splitter_lcp, terminated=tree.terminated,
                        keys=pack_keys(a, h), buckets=classify_oracle(pack_keys(a, h), k),
                        boundaries=np.zeros(1, np.int64), depth_delta=np.zeros(1, np.int64),
                        finished=np.zeros(1, bool))
    np.savez_compressed(os.path.join(HERE, "classifier_cases.npz"),
                        **{f"{k}__{f}": v for k, d in cls.items() for f, v in d.items()})

    # packed keys at several depths (strings.py:176-191)
    a, h = arena_from_strings(H.random_strings(3000, seed=21, max_len=24))
    lens = np.asarray([a.length_at(int(x)) for x in h])
    keys = {}
    for depth in range(0, 17):
        sel = h[lens >= depth]
        keys[f"d{depth}__handles"] = sel
        keys[f"d{depth}__keys"] = pack_keys(a, sel, depth)
    np.savez_compressed(os.path.join(HERE, "pack_keys.npz"), arena=a.data, **keys)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
