"""Parity of the B200 library (libs5.so through its C-ABI) with the reference.

Golden fixtures were produced by the reference package itself
(tests/golden/make_golden.py); larger inputs are checked against the CPU
oracle (oracle/, pinned to the reference in test_oracle_golden.py); full-size
configurations against the reference's published digests
and size-independent properties.  Integer path: every comparison is exact.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_1305_1157_b200 import (SampleSortConfig, StringArena, adjacent_lcps, compute_stats,
                                  datasets, distinguishing_prefix, first_unsorted, pack_keys,
                                  parallel_sample_sort, sample_sort, sort_with_lcp,
                                  verify_sorted_permutation)
from paper_1305_1157_b200 import classifier as CL
from paper_1305_1157_b200 import Counters

pytestmark = pytest.mark.gpu

CONFIGS = {
    "default": SampleSortConfig(),
    "equal": SampleSortConfig(classifier="equal"),
    "tiny_tiers": SampleSortConfig(v=15, small_max=8, narrow_max=64, seed=3),
    "wide_everywhere": SampleSortConfig(v=255, small_max=32, narrow_max=32, seed=5),
    "alpha8": SampleSortConfig(v=1023, alpha=8, small_max=16, narrow_max=2048, flags=128),
    "local_only": SampleSortConfig(v=255, local_max=4096, narrow_max=4096, seed=7),
    "no_local": SampleSortConfig(local_max=32, seed=11),
    "local_small8": SampleSortConfig(v=63, small_max=8, local_max=256, narrow_max=1024),
    # bulk-copy staged scatter at every level; bitonic local sort + separate gather pass
    "wide_tma": SampleSortConfig(v=255, small_max=32, narrow_max=32, seed=5, flags=32),
    "bitonic_gather": SampleSortConfig(seed=9, flags=16 | 64),
    # one-CTA S^5 step (narrow tier) for segments of 4097..16384 strings
    "narrow_tier": SampleSortConfig(narrow_max=16384, seed=13),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _check_sorted(arena, h0, got, want_sorted=None, got_lcp=None, want_lcp=None, name=""):
    assert np.array_equal(np.sort(got), np.sort(h0)), f"{name}: not a permutation"
    if want_sorted is not None:
        assert O.contents_equal(arena, got, want_sorted), f"{name}: string sequence differs"
    else:
        assert O.first_unsorted(arena, got) == -1, f"{name}: not sorted"
    if want_lcp is not None:
        assert np.array_equal(got_lcp, want_lcp), f"{name}: LCP differs"


@pytest.mark.parametrize("cfg_name", list(CONFIGS))
def test_sort_matches_reference_golden(sort_cases, cfg_name):
    cfg = CONFIGS[cfg_name]
    for name, c in sort_cases.items():
        arena = StringArena(c["arena"])
        h = c["handles"].copy()
        h2, lcp = sort_with_lcp(arena, h, cfg=cfg)
        assert h2 is h
        _check_sorted(arena, c["handles"], h, c["sorted"], lcp, c["lcp"], f"{cfg_name}/{name}")
        if h.size:
            assert distinguishing_prefix(arena, h, lcp) == int(c["D"]), name


def test_sample_sort_entry_and_counters(sort_cases):
    c = sort_cases["random_20000"]
    arena = StringArena(c["arena"])
    h = c["handles"].copy()
    ctr = Counters()
    sample_sort(arena, h, cfg=SampleSortConfig(v=63), counters=ctr)
    assert O.contents_equal(arena, h, c["sorted"])
    assert ctr.get("parallel_steps") >= 1 and ctr.get("fetches") >= h.size
    h = c["handles"].copy()
    parallel_sample_sort(arena, h, 8)
    assert O.contents_equal(arena, h, c["sorted"])


def test_device_resident_handles(sort_cases):
    import torch
    c = sort_cases["harness_random_50000"]
    arena = StringArena(c["arena"])
    d = torch.from_numpy(c["handles"].copy()).cuda()
    lcp = torch.empty(d.numel() - 1, dtype=torch.int64, device="cuda")
    parallel_sample_sort(arena, d, lcp_out=lcp)
    got = d.cpu().numpy()
    _check_sorted(arena, c["handles"], got, c["sorted"], lcp.cpu().numpy(), c["lcp"])


def test_sort_from_depth():
    # sample_sort's depth argument: all strings share the first `depth` bytes
    rng = np.random.default_rng(3)
    strs = [b"prefix" + bytes(rng.integers(97, 100, rng.integers(0, 9)).tolist()) for _ in range(5000)]
    from paper_1305_1157_b200 import arena_from_strings
    arena, h = arena_from_strings(strs)
    want = np.asarray(h)[np.argsort(np.array(strs, dtype=object), kind="stable")]
    lcp = np.empty(h.size - 1, np.int64)
    sample_sort(arena, h, depth=6, lcp_out=lcp)
    assert O.contents_equal(arena, h, want)
    assert np.array_equal(lcp, O.adjacent_lcps(arena, h))


def test_tiny_inputs():
    from paper_1305_1157_b200 import arena_from_strings
    for n in (0, 1, 2, 3, 10, 31, 32, 33, 64, 65):
        strs = [bytes([97 + (i * 7) % 5]) * ((i * 3) % 4) for i in range(n)]
        arena, h = arena_from_strings(strs)
        parallel_sample_sort(arena, h)
        raw = arena.data.tobytes()
        got = [raw[x:raw.index(0, x)] for x in h]
        assert got == sorted(strs), n


def test_host_path_lcp_widths_and_range():
    # the host path returns LCPs in the narrowest width that holds them:
    # LCPs above 255 and 65535 take the 2- and 4-byte transfers
    from paper_1305_1157_b200 import arena_from_strings
    for L in (300, 70000):
        strs = [b"x" * L + bytes([97 + i % 3, 98 + (i * 7) % 5]) for i in range(40)] + [b"a", b"b"]
        arena, h = arena_from_strings(strs)
        h2, lcp = sort_with_lcp(arena, h.copy())
        raw = arena.data.tobytes()
        assert [raw[x:raw.index(0, x)] for x in h2] == sorted(strs)
        assert np.array_equal(lcp, O.adjacent_lcps(arena, h2))
        assert lcp.max() >= L
    # handles outside the arena are rejected before any sorting
    arena, h = arena_from_strings([b"ab", b"cd", b"ef", b"gh"])
    for badv in (arena.data.size + 10, -1, 1 << 33):
        bad = h.copy()
        bad[2] = badv
        with pytest.raises((IndexError, ValueError)):
            sort_with_lcp(arena, bad)


def test_partition_kernel_groups_by_full_string_rank():
    # multi-GPU step 3 (s5_partition): destination = number of splitters below
    # the string in (string, handle) order; identical strings straddle a splitter
    import bisect
    import torch
    from paper_1305_1157_b200 import arena_from_strings
    from paper_1305_1157_b200.distributed import GpuBackend
    rng = np.random.default_rng(5)
    strs = [bytes(rng.integers(97, 100, rng.integers(0, 20)).tolist()) for _ in range(20000)]
    strs += [b"abcabcabcabcabcabc" * 3] * 50 + [b""] * 7
    arena, h = arena_from_strings(strs)
    raw = arena.data.tobytes()
    text = {int(x): raw[x:raw.index(0, x)] for x in h}
    ident = [int(x) for x in h if text[int(x)] == b"abcabcabcabcabcabc" * 3]
    sample = sorted({int(x) for x in rng.choice(h, 40, replace=False)} | set(ident[20:23]),
                    key=lambda x: (text[x], x))
    be = GpuBackend(arena)
    out, counts = be.partition(torch.from_numpy(h.copy()).cuda(),
                               torch.tensor(sample, dtype=torch.int64, device="cuda"))
    out = out.cpu().numpy()
    keys = [(text[x], x) for x in sample]
    dest = np.array([bisect.bisect_left(keys, (text[int(x)], int(x))) for x in h])
    assert counts == np.bincount(dest, minlength=len(sample) + 1).tolist()
    at = 0
    for g, c in enumerate(counts):
        assert sorted(out[at:at + c].tolist()) == sorted(h[dest == g].tolist()), g
        at += c


@pytest.mark.parametrize("shape", ["identical", "empty", "prefix1000", "binary", "len1", "nested"])
def test_adversarial_shapes_through_every_tier(shape):
    # shapes that drive the wide tier's equality buckets, the local tiers'
    # common-prefix skip, truncated sort words and long tie walks at sizes
    # above the one-CTA limit
    from paper_1305_1157_b200 import arena_from_strings
    rng = np.random.default_rng(17)
    n = 300_000
    if shape == "identical":
        strs = [b"the-same-string-repeated"] * n
    elif shape == "empty":
        strs = [b""] * (n // 2) + [b"x"] * (n // 2)
    elif shape == "prefix1000":
        base = bytes(rng.integers(97, 123, 1000).tolist())
        strs = [base + bytes(rng.integers(97, 99, rng.integers(0, 12)).tolist()) for _ in range(n // 10)]
    elif shape == "binary":
        strs = [bytes(rng.integers(1, 256, rng.integers(0, 24)).tolist()) for _ in range(n)]
    elif shape == "len1":
        strs = [bytes([int(x)]) for x in rng.integers(1, 4, n)]
    else:  # prefix chains: every string a prefix of the next ones
        strs = [b"a" * int(k) for k in rng.integers(0, 300, n // 3)]
    arena, h = arena_from_strings(strs)
    want = h.copy()
    O.parallel_sample_sort(arena, want, 8)
    got, lcp = sort_with_lcp(arena, h.copy())
    _check_sorted(arena, h, got, want, lcp, O.adjacent_lcps(arena, want), shape)


def _load_lines_reference(raw: bytes):
    # harness.py:83-95 restated on numpy (newline -> terminator, one appended
    # after an unterminated last line)
    data = np.frombuffer(raw, np.uint8).copy()
    if data.size == 0:
        return data, np.zeros(0, np.int64)
    data[data == ord("\n")] = 0
    if data[-1] != 0:
        data = np.append(data, np.uint8(0))
    ends = np.nonzero(data == 0)[0]
    handles = np.zeros(ends.size, np.int64)
    handles[1:] = ends[:-1] + 1
    return data, handles


@pytest.mark.parametrize("tail", [b"", b"\n", b"last-line-no-newline", b"\n\n"])
def test_ingest_lines_matches_harness(tail):
    from paper_1305_1157_b200 import ingest_lines
    rng = np.random.default_rng(4)
    lines = [bytes(rng.integers(32, 127, rng.integers(0, 40)).tolist()) for _ in range(70_000)]
    raw = b"\n".join(lines) + tail
    want_data, want_h = _load_lines_reference(raw)
    arena, h = ingest_lines(raw)
    assert arena.size == want_data.size
    assert np.array_equal(arena.data, want_data)
    assert np.array_equal(h.cpu().numpy(), want_h)
    # the device-born arena sorts like any other
    got, lcp = sort_with_lcp(arena, h.cpu().numpy())
    ref_arena = StringArena(want_data)
    want = want_h.copy()
    O.parallel_sample_sort(ref_arena, want, 4)
    assert O.contents_equal(ref_arena, got, want)
    assert np.array_equal(lcp, O.adjacent_lcps(ref_arena, want))


def test_ingest_rejects_embedded_nul_and_handles_empty():
    from paper_1305_1157_b200 import EmbeddedNul, ingest_lines
    with pytest.raises(EmbeddedNul) as e:
        ingest_lines(b"abc\ndef\x00gh\nij\x00")
    assert e.value.offset == 7
    arena, h = ingest_lines(b"")
    assert arena.size == 0 and h.numel() == 0


def test_string_lengths_and_materialize():
    from paper_1305_1157_b200 import arena_from_strings, materialize, string_lengths
    rng = np.random.default_rng(9)
    strs = [bytes(rng.integers(1, 256, rng.integers(0, 50)).tolist()) for _ in range(50_000)]
    arena, h = arena_from_strings(strs)
    assert np.array_equal(string_lengths(arena, h), np.array([len(x) for x in strs]))
    sh, _ = sort_with_lcp(arena, h.copy())
    out, oh = materialize(arena, sh)
    want = sorted(strs)
    assert out.size == sum(len(x) + 1 for x in strs)
    raw = out.data.tobytes()
    oh = oh.cpu().numpy()
    assert [raw[a:raw.index(0, a)] for a in oh] == want
    assert np.array_equal(np.diff(oh), np.array([len(x) + 1 for x in want[:-1]]))
    # suffix-mode arena: one terminator at the end
    text = bytes(rng.integers(97, 100, 3000).tolist()) + b"\x00"
    sa = StringArena(np.frombuffer(text, np.uint8))
    hh = np.arange(3000, dtype=np.int64)
    assert np.array_equal(string_lengths(sa, hh), 3000 - hh)


def test_standalone_upload_download_roundtrip():
    # the multi-GPU path's host staging (s5_upload_handles / s5_download)
    import torch
    from paper_1305_1157_b200 import arena_from_strings
    from paper_1305_1157_b200.distributed import GpuBackend
    strs = [b"x" * (i % 700) + b"y" for i in range(40_000)]
    arena, h = arena_from_strings(strs)
    be = GpuBackend(arena)
    d = be.upload(h)
    assert torch.equal(d.cpu(), torch.from_numpy(h))
    d2, lcp = be.sort(d.clone())
    hh, hl = be.download(d2, lcp)
    assert np.array_equal(hh, d2.cpu().numpy()) and np.array_equal(hl, lcp.cpu().numpy())
    assert hl.max() > 255  # two-byte LCP transfer
    bad = h.copy()
    bad[5] = arena.size + 3
    with pytest.raises(ValueError):
        be.upload(bad)


def test_release_caches_then_sort_again(sort_cases):
    from paper_1305_1157_b200 import _lib
    c = sort_cases["random_20000"]
    arena = StringArena(c["arena"])
    for _ in range(2):
        h, lcp = sort_with_lcp(arena, c["handles"].copy())
        _check_sorted(arena, c["handles"], h, c["sorted"], lcp, c["lcp"], "after release")
        assert _lib.lib().s5_release_caches() == 0


def test_pack_keys_matches_reference():
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "pack_keys.npz"))
    arena = StringArena(z["arena"])
    for depth in range(17):
        got = pack_keys(arena, z[f"d{depth}__handles"], depth)
        assert np.array_equal(got, z[f"d{depth}__keys"]), depth


def test_adjacent_lcp_and_verify_match_reference(sort_cases):
    for name, c in sort_cases.items():
        arena = StringArena(c["arena"])
        assert np.array_equal(adjacent_lcps(arena, c["sorted"]), c["lcp"]), name
        assert first_unsorted(arena, c["sorted"]) == -1
        assert verify_sorted_permutation(arena, c["handles"], c["sorted"]).ok
    c = sort_cases["random_1000"]
    arena = StringArena(c["arena"])
    bad = c["sorted"].copy()
    bad[[3, 700]] = bad[[700, 3]]
    r = verify_sorted_permutation(arena, c["handles"], bad)
    assert not r.ok and r.reason == "not_sorted" and r.index == O.first_unsorted(arena, bad)
    bad = c["sorted"].copy()
    bad[0] = bad[1]
    assert verify_sorted_permutation(arena, c["handles"], bad).reason == "not_permutation"


def test_classifier_and_tree_match_reference(classifier_cases):
    for name, c in classifier_cases.items():
        spl = c["splitters"]
        if name != "cterm":
            lo, io = CL.build_tree_from_sample(c["sample"], spl.size)
            assert np.array_equal(io, spl), name
            assert np.array_equal(lo[1:], c["level_order"][1:]), name
        tree = CL.build_tree(spl)
        assert np.array_equal(tree.level_order, c["level_order"])
        assert np.array_equal(tree.splitter_lcp, c["splitter_lcp"])
        want = c["buckets"]
        assert np.array_equal(CL.classify_tree_unrolled(c["keys"], tree).astype(np.int64), want), name
        assert np.array_equal(CL.classify_tree_equal(c["keys"], tree).astype(np.int64), want), name
        assert np.array_equal(CL.classify_tree_lut(c["keys"], tree).astype(np.int64), want), name


def test_classifier_exhaustive_small_trees():
    # test_classifier.py:181-196 shape: v in {1,3,7}, adversarial keys, duplicate splitters
    rng = np.random.default_rng(11)
    for v in (1, 3, 7, 15):
        for dup in (False, True):
            for _ in range(20):
                pool = rng.integers(1, 40, v).astype(np.uint64)
                if dup and v > 1:
                    pool[rng.integers(0, v)] = pool[0]
                spl = np.sort(pool)
                keys = set()
                for x in spl.tolist():
                    keys.update((x, max(0, x - 1), x + 1))
                keys.update((0, 2**64 - 1))
                keys = np.asarray(sorted(keys), np.uint64)
                want = O.classify_oracle(keys, spl)
                tree = CL.build_tree(spl)
                assert np.array_equal(CL.classify_tree_unrolled(keys, tree).astype(np.int64), want)
                assert np.array_equal(CL.classify_tree_equal(keys, tree).astype(np.int64), want)
                assert np.array_equal(CL.classify_tree_lut(keys, tree).astype(np.int64), want)


@pytest.mark.parametrize("config,n", [(1, None), (2, 1 << 20), (3, 1 << 19), (4, 1 << 19),
                                      (5, 1 << 20)])
def test_configs_reduced_vs_oracle(config, n):
    arena, h0 = datasets.generate(config, n)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, O.max_threads())
    want_lcp = O.adjacent_lcps(arena, want)
    for cfg in (SampleSortConfig(), SampleSortConfig(classifier="equal", seed=9)):
        h = h0.copy()
        _, lcp = sort_with_lcp(arena, h, cfg=cfg)
        _check_sorted(arena, h0, h, want, lcp, want_lcp, f"cfg{config}")
        if config == 5:
            assert np.array_equal(h, want)  # no duplicates: permutation is unique


def test_config1_reference_digests():
    arena, h = datasets.generate(1)
    _, lcp = sort_with_lcp(arena, h)
    ds, dl = datasets.DIGESTS[1]
    assert O.digest_strings(arena, h)[:16] == ds
    assert O.digest_lcp(lcp)[:16] == dl
    assert distinguishing_prefix(arena, h, lcp) == datasets.EXPECTED[1][2]


@pytest.mark.slow
@pytest.mark.parametrize("config", [2, 3, 4, 5])
def test_full_config_reference_digests(config):
    """Full BASELINE sizes: digests of the reference's output + properties."""
    import torch
    arena, h0 = datasets.generate(config)
    n, N, D = datasets.EXPECTED[config]
    assert h0.size == n and arena.data.size == N
    d = torch.from_numpy(h0).cuda()
    lcp = torch.empty(n - 1, dtype=torch.int64, device="cuda")
    parallel_sample_sort(arena, d, lcp_out=lcp)
    assert first_unsorted(arena, d) == -1
    assert torch.equal(torch.sort(d).values, torch.from_numpy(h0).cuda())
    assert torch.equal(adjacent_lcps(arena, d), lcp)   # independent LCP kernel
    assert distinguishing_prefix(arena, d, lcp) == D
    got = d.cpu().numpy()
    ds, dl = datasets.DIGESTS[config]
    assert O.digest_lcp(lcp.cpu().numpy())[:16] == dl
    if config in datasets.HANDLE_DIGESTS:
        import hashlib
        hd, first5 = datasets.HANDLE_DIGESTS[config]
        assert got[:5].tolist() == first5
        assert hashlib.sha256(got.astype("<i8").tobytes()).hexdigest()[:16] == hd
    else:
        assert O.digest_strings(arena, got)[:16] == ds
    del arena


def _random_strings(n, seed, max_len=20, lo=33, hi=127):
    # helpers.random_strings (pkg/tests/helpers.py:134-138) shape, vectorised
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len, n)
    body = rng.integers(lo, hi, int(lens.sum())).astype(np.uint8).tobytes()
    out, at = [], 0
    for ln in lens.tolist():
        out.append(body[at:at + ln])
        at += ln
    return out


@pytest.mark.parametrize("cfg", [SampleSortConfig(v=255, small_max=16, narrow_max=512),
                                 SampleSortConfig(v=15, small_max=8, narrow_max=32)])
def test_eq1_audit(cfg):
    """test_samplesort.py:144-160, :206-225: every child's claimed depth is a
    lower bound on the pairwise lcp of its strings."""
    from paper_1305_1157_b200 import arena_from_strings
    strs = _random_strings(100_000, seed=14)
    arena, h = arena_from_strings(strs)
    rng = np.random.default_rng(1)
    seen, violations = [], []

    def audit(side, lo, hi, depth):
        seen.append((lo, hi, depth))
        idx = rng.integers(lo, hi, (min(100, hi - lo), 2))
        for i, j in idx:
            if O.lcp(arena, int(side[i]), int(side[j])) < depth:
                violations.append((lo, hi, depth))
                return

    orig = h.copy()
    parallel_sample_sort(arena, h, 2, cfg=cfg, audit=audit)
    assert violations == []
    assert seen and all(0 <= lo < hi <= h.size for lo, hi, _ in seen)
    # children of one level are disjoint (segments of later levels nest inside)
    first = {}
    for lo, hi, d in seen:
        first.setdefault(lo, (hi, d))
    spans = sorted((lo, hi) for lo, (hi, _) in first.items())
    assert all(a_hi <= b_lo or b_hi <= a_hi for (_, a_hi), (b_lo, b_hi) in zip(spans, spans[1:]))
    assert O.first_unsorted(arena, h) == -1
    assert np.array_equal(np.sort(h), np.sort(orig))


def test_identical_strings_equality_chain():
    """test_samplesort.py:126-132 / :228-232: identical 17-char strings walk the
    equality buckets 0 -> 8 -> 16 and finish on the terminated splitter."""
    from paper_1305_1157_b200 import arena_from_strings
    arena, h = arena_from_strings([b"q" * 17] * 100_000)
    ctr = Counters()
    _, lcp = sort_with_lcp(arena, h, cfg=SampleSortConfig(v=31), counters=ctr)
    assert ctr.get("parallel_steps") == 3
    assert np.all(lcp == 17)


@pytest.mark.parametrize("alphabet", [b"AB", b"ACGT"])
def test_second_key_words_carried_to_level1(alphabet):
    """Few distinct 8-byte prefixes (n > 16 x the root sample's estimate):
    the root gathers 16 bytes per string and level 1's equality buckets take
    their next key from the carried word instead of the arena.  Same output as
    the oracle and as the path with the carry disabled (flags bit8); fewer
    arena key fetches."""
    from paper_1305_1157_b200 import arena_from_strings
    rng = np.random.default_rng(21)
    n = 600_000 if len(alphabet) == 2 else 1_200_000
    lens = rng.integers(8, 40, n)
    sym = np.frombuffer(alphabet, np.uint8)[rng.integers(0, len(alphabet), int(lens.sum()))].tobytes()
    strs, at = [], 0
    for ln in lens.tolist():
        strs.append(sym[at:at + ln])
        at += ln
    arena, h0 = arena_from_strings(strs)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, O.max_threads())
    want_lcp = O.adjacent_lcps(arena, want)
    fetches = {}
    for flags in (0, 256):
        h = h0.copy()
        ctr = Counters()
        # (wide_v 63: the root's children are wide steps at these n)
        cfg = SampleSortConfig(flags=flags, wide_v=63)
        _, lcp = sort_with_lcp(arena, h, cfg=cfg, counters=ctr)
        _check_sorted(arena, h0, h, want, lcp, want_lcp, f"flags{flags}")
        fetches[flags] = ctr.get("fetches")
    assert fetches[0] < fetches[256]


@pytest.mark.parametrize("n_dup", [40, 100, 700])
def test_duplicate_short_strings_in_truncated_segments(n_dup):
    """A local segment with no common prefix (truncated sort words) holding
    long runs of identical short strings: the runs finish in the segment
    (terminator inside the compared bytes), next to longer strings that share
    those short strings as prefixes."""
    from paper_1305_1157_b200 import arena_from_strings
    rng = np.random.default_rng(n_dup)
    strs = []
    for w in (b"a", b"ab", b"abcdef", b"\x7f", b"zzzzz"):
        strs += [w] * n_dup
    for _ in range(1500):
        ln = int(rng.integers(1, 14))
        strs.append(bytes(rng.integers(33, 127, ln, dtype=np.uint8)))
    strs += [b"abcdefg", b"abcdefgh", b"abcdef\x01"] * 30
    order = rng.permutation(len(strs))
    arena, h0 = arena_from_strings([strs[i] for i in order])
    want = h0.copy()
    O.parallel_sample_sort(arena, want, 2)
    want_lcp = O.adjacent_lcps(arena, want)
    for cfg in (SampleSortConfig(), SampleSortConfig(local_max=256, narrow_max=256, small_max=8)):
        h = h0.copy()
        _, lcp = sort_with_lcp(arena, h, cfg=cfg)
        _check_sorted(arena, h0, h, want, lcp, want_lcp, f"dup{n_dup}")


# ---------------------------------------------------------------------------
# index mode (cfg flags bit13; always on for arenas >= 4 GiB): the offset
# arrays hold string indices and a position table maps them to the arena --
# the reference's handles are int64 offsets (strings.py:3-7)

INDEXED = 8192


@pytest.mark.parametrize("cfg_name", ["default", "equal", "tiny_tiers", "wide_everywhere",
                                      "wide_tma", "narrow_tier", "bitonic_gather"])
def test_index_mode_matches_reference_golden(sort_cases, cfg_name):
    import dataclasses
    base = CONFIGS[cfg_name]
    cfg = dataclasses.replace(base, flags=base.flags | INDEXED)
    for name, c in sort_cases.items():
        arena = StringArena(c["arena"])
        h = c["handles"].copy()
        _, lcp = sort_with_lcp(arena, h, cfg=cfg)
        _check_sorted(arena, c["handles"], h, c["sorted"], lcp, c["lcp"], f"idx/{cfg_name}/{name}")


@pytest.mark.parametrize("config,n", [(2, 1 << 20), (3, 1 << 19), (4, 1 << 19), (5, 1 << 20)])
def test_index_mode_configs_vs_oracle(config, n):
    import torch
    arena, h0 = datasets.generate(config, n)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, O.max_threads())
    want_lcp = O.adjacent_lcps(arena, want)
    # device-resident handles and the host path
    d = torch.from_numpy(h0.copy()).cuda()
    lcp = torch.empty(d.numel() - 1, dtype=torch.int64, device="cuda")
    parallel_sample_sort(arena, d, cfg=SampleSortConfig(flags=INDEXED), lcp_out=lcp)
    _check_sorted(arena, h0, d.cpu().numpy(), want, lcp.cpu().numpy(), want_lcp, f"idx/cfg{config}")
    h = h0.copy()
    _, hl = sort_with_lcp(arena, h, cfg=SampleSortConfig(flags=INDEXED, seed=4))
    _check_sorted(arena, h0, h, want, hl, want_lcp, f"idx/host/cfg{config}")


@pytest.mark.parametrize("shape", ["identical", "prefix1000", "nested"])
def test_index_mode_adversarial_shapes(shape):
    from paper_1305_1157_b200 import arena_from_strings
    rng = np.random.default_rng(23)
    n = 200_000
    if shape == "identical":
        strs = [b"the-same-string-repeated"] * n
    elif shape == "prefix1000":
        base = bytes(rng.integers(97, 123, 1000).tolist())
        strs = [base + bytes(rng.integers(97, 99, rng.integers(0, 12)).tolist()) for _ in range(n // 10)]
    else:
        strs = [b"a" * int(k) for k in rng.integers(0, 300, n // 3)]
    arena, h = arena_from_strings(strs)
    want = h.copy()
    O.parallel_sample_sort(arena, want, 8)
    got, lcp = sort_with_lcp(arena, h.copy(), cfg=SampleSortConfig(flags=INDEXED))
    _check_sorted(arena, h, got, want, lcp, O.adjacent_lcps(arena, want), "idx/" + shape)


@pytest.mark.slow
def test_arena_beyond_4gib():
    """A 4.25 GiB arena: handles above 2^32, duplicated handles (identical
    2 KB strings walked to their ends) and strings sharing long prefixes."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < 12 << 30:
        pytest.skip("needs 12 GiB of free device memory")
    rng = np.random.default_rng(41)
    L = 2048                       # bytes per string slot, terminator included
    n_slots = (17 << 28) // L      # 4.25 GiB
    data = rng.integers(33, 127, size=n_slots * L, dtype=np.uint8)
    data[L - 1::L] = 0
    # slots 1.. copy a long prefix of slot 0 in a few places (deep LCPs high up)
    for slot in (5, n_slots // 2, n_slots - 3, n_slots - 2):
        keep = int(rng.integers(500, 1900))
        data[slot * L: slot * L + keep] = data[:keep]
    arena = StringArena(data)
    h0 = np.arange(n_slots, dtype=np.int64) * L
    # suffix handles (strings starting inside a slot) and duplicates
    extra = h0[rng.integers(0, n_slots, 100_000)] + rng.integers(0, L - 1, 100_000)
    dups = h0[rng.integers(n_slots - 50_000, n_slots, 60_000)]
    h0 = np.concatenate([h0, extra, dups])
    rng.shuffle(h0)
    assert int(h0.max()) >= 1 << 32
    want = h0.copy()
    O.parallel_sample_sort(arena, want, O.max_threads())
    want_lcp = O.adjacent_lcps(arena, want)
    d = torch.from_numpy(h0.copy()).cuda()
    lcp = torch.empty(d.numel() - 1, dtype=torch.int64, device="cuda")
    parallel_sample_sort(arena, d, lcp_out=lcp)
    _check_sorted(arena, h0, d.cpu().numpy(), want, lcp.cpu().numpy(), want_lcp, "4gib/device")
    del d, lcp
    h = h0.copy()
    _, hl = sort_with_lcp(arena, h)     # host path: int64 handles both ways
    _check_sorted(arena, h0, h, want, hl, want_lcp, "4gib/host")
    from paper_1305_1157_b200 import samplesort as SS
    arena.drop_device()
    SS.release_workspace()


# ---------------------------------------------------------------------------
# root prefix skip (cfg flags bit14 turns it off): the root sample's common
# prefix is checked against every string; one mismatch redoes the sort

NO_SKIP = 16384


def _prefixed(prefix: bytes, n: int, seed: int, extra=()):
    from paper_1305_1157_b200 import arena_from_strings
    rng = np.random.default_rng(seed)
    body = rng.integers(97, 123, size=(n, 20), dtype=np.uint8)
    lens = rng.integers(0, 21, n)
    strs = [prefix + body[i, :lens[i]].tobytes() for i in range(n)]
    strs.extend(extra)
    order = rng.permutation(len(strs))
    return arena_from_strings([strs[i] for i in order])


@pytest.mark.parametrize("prefix", [b"ab", b"http://", b"/var/log/app/", b"\xff\xfe\xfd"])
def test_root_prefix_skip_matches_oracle(prefix):
    arena, h0 = _prefixed(prefix, 200_000, 5)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, 8)
    want_lcp = O.adjacent_lcps(arena, want)
    c_skip, c_plain = Counters(), Counters()
    h = h0.copy()
    lcp = np.empty(h.size - 1, np.int64)
    parallel_sample_sort(arena, h, cfg=SampleSortConfig(), counters=c_skip, lcp_out=lcp)
    _check_sorted(arena, h0, h, want, lcp, want_lcp, f"skip/{prefix!r}")
    h = h0.copy()
    parallel_sample_sort(arena, h, cfg=SampleSortConfig(flags=NO_SKIP), counters=c_plain, lcp_out=lcp)
    _check_sorted(arena, h0, h, want, lcp, want_lcp, f"noskip/{prefix!r}")
    # the skip never costs a level; behind a 7-byte prefix it saves one
    assert c_skip.get("parallel_steps") <= c_plain.get("parallel_steps")
    if prefix == b"http://":
        assert c_skip.get("parallel_steps") < c_plain.get("parallel_steps")


@pytest.mark.parametrize("odd", [[b"ftp://other"], [b"http:/"], [b""], [b"http://"],
                                 [b"http:/\x01zzz", b"h", b"i" * 40]])
def test_root_prefix_skip_falls_back_on_a_mismatch(odd):
    # the sample (a few thousand of 300 001+ strings) sees only "http://..."
    arena, h0 = _prefixed(b"http://", 300_000, 9, extra=odd)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, 8)
    for cfg in (SampleSortConfig(), SampleSortConfig(flags=INDEXED, seed=2)):
        h = h0.copy()
        _, lcp = sort_with_lcp(arena, h, cfg=cfg)
        _check_sorted(arena, h0, h, want, lcp, O.adjacent_lcps(arena, want), f"fallback/{odd!r}")


def test_root_prefix_skip_behind_a_caller_depth():
    # sample_sort(depth=6): every string starts with "prefix", and the bytes
    # behind it share "http://" -- the skip applies on top of the caller's depth
    from paper_1305_1157_b200 import arena_from_strings
    rng = np.random.default_rng(31)
    strs = [b"prefixhttp://" + bytes(rng.integers(97, 101, rng.integers(0, 14)).tolist())
            for _ in range(60_000)]
    arena, h = arena_from_strings(strs)
    want = h.copy()
    O.parallel_sample_sort(arena, want, 8)
    for flags in (0, NO_SKIP, INDEXED):
        got = h.copy()
        lcp = np.empty(h.size - 1, np.int64)
        sample_sort(arena, got, depth=6, cfg=SampleSortConfig(flags=flags), lcp_out=lcp)
        _check_sorted(arena, h, got, want, lcp, O.adjacent_lcps(arena, want), f"depth6/{flags}")


def test_long_shared_prefix_in_a_wide_segment():
    # 6000 strings (above the one-CTA limit) sharing 40 KB: a wide segment
    # moves 8 bytes per level, so after four whole-segment levels it goes to
    # the one-CTA step, whose in-place skip walks the prefix in one kernel
    from paper_1305_1157_b200 import arena_from_strings
    rng = np.random.default_rng(77)
    base = bytes(rng.integers(1, 256, 40_000).tolist())
    strs = [base + bytes(rng.integers(97, 100, rng.integers(0, 5)).tolist()) for _ in range(6000)]
    arena, h = arena_from_strings(strs)
    want = h.copy()
    O.parallel_sample_sort(arena, want, 8)
    ctr = Counters()
    got = h.copy()
    lcp = np.empty(h.size - 1, np.int64)
    parallel_sample_sort(arena, got, counters=ctr, lcp_out=lcp)
    _check_sorted(arena, h, got, want, lcp, O.adjacent_lcps(arena, want), "prefix40k")
    assert ctr.get("parallel_steps") < 64
    # the same through the wide tier only (narrow step off by size): every level counts
    big = [base[:4000] + bytes(rng.integers(97, 100, rng.integers(0, 5)).tolist()) for _ in range(6000)]
    arena, h = arena_from_strings(big)
    want = h.copy()
    O.parallel_sample_sort(arena, want, 8)
    got = h.copy()
    parallel_sample_sort(arena, got, cfg=SampleSortConfig(local_max=8192), counters=(c2 := Counters()),
                         lcp_out=lcp)
    _check_sorted(arena, h, got, want, lcp, O.adjacent_lcps(arena, want), "prefix4k")
