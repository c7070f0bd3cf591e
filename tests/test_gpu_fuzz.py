"""Seeded differential fuzz of the GPU sort against the CPU oracle: random
alphabets, length laws, shared prefixes, duplicates and tier configurations
(each case: sorted string sequence, LCP array, permutation -- exact)."""
import os

import numpy as np
import pytest

import oracle as O
from paper_1305_1157_b200 import SampleSortConfig, arena_from_strings, sort_with_lcp

pytestmark = pytest.mark.gpu


def _strings(rng):
    n = int(rng.choice([2, 3, 33, 257, 1000, 4097, 20_000, 70_000]))
    sigma = int(rng.choice([1, 2, 4, 26, 94, 255]))
    lo = int(rng.choice([0, 0, 1, 7]))
    hi = lo + int(rng.choice([0, 1, 8, 9, 24, 70]))
    base = int(rng.integers(1, 256 - sigma + 1)) if sigma < 255 else 1
    prefix = bytes(rng.integers(1, 256, int(rng.choice([0, 0, 2, 7, 8, 9, 40]))).tolist())
    pool = None
    if rng.random() < 0.4:  # many duplicates: draw from a small pool
        pool = int(rng.choice([1, 3, 50, 2000]))
    def one():
        m = int(rng.integers(lo, hi + 1))
        return prefix + bytes((rng.integers(0, sigma, m) + base).tolist())
    if pool is not None:
        bank = [one() for _ in range(pool)]
        strs = [bank[int(i)] for i in rng.integers(0, pool, n)]
    else:
        strs = [one() for _ in range(n)]
    if rng.random() < 0.3:  # a few strings off the common prefix
        for i in rng.integers(0, n, 3):
            strs[int(i)] = bytes(rng.integers(1, 256, int(rng.integers(0, 6))).tolist())
    return strs


def _config(rng):
    flags = 0
    for bit, p in ((8, .2), (16, .1), (32, .2), (64, .1), (128, .2), (256, .2), (2048, .2),
                   (8192, .25), (16384, .2)):
        if rng.random() < p:
            flags |= bit
    small = int(rng.choice([1, 8, 32]))
    local = int(rng.choice([32, 256, 1024, 4096]))
    narrow = int(rng.choice([local, 4096, 16384])) if local <= 4096 else local
    return SampleSortConfig(v=int(rng.choice([15, 63, 255, 1023, 8191])),
                            alpha=int(rng.choice([1, 2, 4, 8])),
                            classifier=str(rng.choice(["unroll", "equal"])),
                            small_max=small, local_max=max(local, small),
                            narrow_max=max(narrow, local, small), flags=flags,
                            seed=int(rng.integers(1, 1 << 30)))


@pytest.mark.parametrize("seed", range(int(os.environ.get("S5_FUZZ_CASES", "200"))))
def test_fuzz_against_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    strs = _strings(rng)
    cfg = _config(rng)
    arena, h0 = arena_from_strings(strs)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, 4)
    got = h0.copy()
    _, lcp = sort_with_lcp(arena, got, cfg=cfg)
    tag = f"seed {seed} n={len(strs)} cfg={cfg}"
    assert np.array_equal(np.sort(got), np.sort(h0)), tag
    assert O.contents_equal(arena, got, want), tag
    assert np.array_equal(lcp, O.adjacent_lcps(arena, want)), tag


@pytest.mark.parametrize("seed", range(int(os.environ.get("S5_FUZZ_BIG_CASES", "12"))))
def test_fuzz_large_against_oracle(seed):
    """Several wide levels, carried second key words, prefix skip, deep
    equality chains: 200 K - 600 K strings over tiny alphabets."""
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.choice([200_000, 600_000])) * int(os.environ.get("S5_FUZZ_BIG_SCALE", "1"))
    sigma = int(rng.choice([1, 2, 3, 4, 20]))
    lmax = int(rng.choice([6, 12, 30, 60]))
    prefix = bytes(rng.integers(1, 256, int(rng.choice([0, 3, 7, 16]))).tolist())
    body = (rng.integers(0, sigma, size=(n, lmax)) + 65).astype(np.uint8)
    lens = rng.integers(0, lmax + 1, n)
    if rng.random() < 0.5:  # long runs of equal leading characters
        body[:, : lmax // 2] = 65
    strs = [prefix + body[i, :lens[i]].tobytes() for i in range(n)]
    cfg = _config(rng)
    cfg.local_max = max(cfg.local_max, 256)  # keep the level count bounded
    cfg.narrow_max = max(cfg.narrow_max, cfg.local_max)
    arena, h0 = arena_from_strings(strs)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, O.max_threads())
    got = h0.copy()
    _, lcp = sort_with_lcp(arena, got, cfg=cfg)
    tag = f"seed {seed} n={n} sigma={sigma} lmax={lmax} cfg={cfg}"
    assert np.array_equal(np.sort(got), np.sort(h0)), tag
    assert O.contents_equal(arena, got, want), tag
    assert np.array_equal(lcp, O.adjacent_lcps(arena, want)), tag


@pytest.mark.parametrize("seed", range(int(os.environ.get("S5_FUZZ_MULTI_CASES", "40"))))
def test_fuzz_entry_points_against_oracle(seed):
    """The other doors into the same sort: device-resident handles, a caller
    depth behind a shared prefix, and workers = G shards on a repeated device
    list (partition kernel, exchange and boundary LCPs on one GPU)."""
    import torch
    from paper_1305_1157_b200 import parallel_sample_sort, sample_sort
    rng = np.random.default_rng(9000 + seed)
    strs = _strings(rng)
    cfg = _config(rng)
    arena, h0 = arena_from_strings(strs)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, 4)
    want_lcp = O.adjacent_lcps(arena, want)
    mode = seed % 3
    tag = f"seed {seed} mode {mode} n={len(strs)} cfg={cfg}"
    if mode == 0:    # CUDA tensors in and out
        d = torch.from_numpy(h0.copy()).cuda()
        dl = torch.empty(d.numel() - 1, dtype=torch.int64, device="cuda")
        parallel_sample_sort(arena, d, cfg=cfg, lcp_out=dl)
        got, lcp = d.cpu().numpy(), dl.cpu().numpy()
    elif mode == 1:  # sample_sort from the depth every string shares
        depth = int(O.adjacent_lcps(arena, want).min()) if h0.size > 1 else 0
        depth = int(rng.integers(0, depth + 1))
        got = h0.copy()
        lcp = np.empty(h0.size - 1, np.int64)
        sample_sort(arena, got, depth=depth, cfg=cfg, lcp_out=lcp)
    else:            # workers = G over one device
        G = int(rng.choice([2, 3, 5]))
        got = h0.copy()
        lcp = np.empty(h0.size - 1, np.int64)
        parallel_sample_sort(arena, got, workers=G, cfg=cfg, lcp_out=lcp, devices=[0] * G)
    assert np.array_equal(np.sort(got), np.sort(h0)), tag
    assert O.contents_equal(arena, got, want), tag
    assert np.array_equal(lcp, want_lcp), tag


@pytest.mark.parametrize("seed", range(int(os.environ.get("S5_FUZZ_AUX_CASES", "30"))))
def test_fuzz_auxiliary_surfaces(seed):
    """Line ingest, string lengths, materialisation, key packing, LCP and
    verification kernels on random inputs against numpy / Python."""
    from paper_1305_1157_b200 import (StringArena, adjacent_lcps, first_unsorted, ingest_lines,
                                      materialize, pack_keys, string_lengths,
                                      verify_sorted_permutation)
    rng = np.random.default_rng(20_000 + seed)
    n = int(rng.choice([1, 2, 31, 1000, 40_000]))
    lmax = int(rng.choice([0, 1, 7, 8, 9, 63, 300]))
    sigma = int(rng.choice([1, 3, 90]))
    lines = [bytes((rng.integers(0, sigma, int(rng.integers(0, lmax + 1))) + 33).tolist())
             for _ in range(n)]
    tail = [b"", b"\n", b"x", b"\n\n"][int(rng.integers(0, 4))]
    raw = b"\n".join(lines) + tail
    # ingest == harness.load_lines (newline -> terminator, one appended if missing)
    data = np.frombuffer(raw, np.uint8).copy()
    if data.size:
        data[data == 10] = 0
        if data[-1] != 0:
            data = np.append(data, np.uint8(0))
    ends = np.nonzero(data == 0)[0]
    want_h = np.zeros(ends.size, np.int64)
    want_h[1:] = ends[:-1] + 1
    arena, h = ingest_lines(raw)
    h = h.cpu().numpy()
    assert np.array_equal(arena.data, data) and np.array_equal(h, want_h)
    if h.size == 0:
        return
    strs = [data[a:e].tobytes() for a, e in zip(want_h, ends)]
    assert np.array_equal(np.asarray(string_lengths(arena, h)), np.array([len(s) for s in strs]))
    depth = int(rng.integers(0, 12))
    ok = (want_h + depth) < data.size
    keys = np.asarray(pack_keys(arena, h[ok], depth))
    ref = StringArena(data)
    assert np.array_equal(keys.astype(np.uint64), O.pack_keys(ref, h[ok], depth).astype(np.uint64))
    # sort, then LCP / verification / materialisation of the sorted order
    got = h.copy()
    _, lcp = sort_with_lcp(arena, got)
    order = sorted(range(len(strs)), key=lambda i: strs[i])
    want_sorted = [strs[i] for i in order]
    assert [strs[int(np.searchsorted(want_h, x))] for x in got] == want_sorted
    if h.size > 1:
        assert np.array_equal(np.asarray(adjacent_lcps(arena, got)), lcp)
        assert np.array_equal(lcp, O.adjacent_lcps(ref, got))
    assert first_unsorted(arena, got) == -1
    assert verify_sorted_permutation(arena, h, got).ok
    if h.size > 2 and want_sorted[0] != want_sorted[-1]:
        bad = got[::-1].copy()
        assert first_unsorted(arena, bad) >= 0
        assert not verify_sorted_permutation(arena, h, bad).ok
    out, oh = materialize(arena, got)
    oh = oh.cpu().numpy()
    blob = out.data.tobytes()
    assert [blob[a:blob.index(0, a)] for a in oh] == want_sorted


@pytest.mark.parametrize("seed", range(int(os.environ.get("S5_FUZZ_NATIVE_MULTI_CASES", "40"))))
def test_fuzz_s5_sort_multi_against_oracle(seed):
    """s5_sort_multi (the C-ABI multi-GPU entry) with ragged shard cuts --
    empty and one-string shards included -- over a repeated device list."""
    import torch
    from paper_1305_1157_b200.multi import sort_multi_device
    rng = np.random.default_rng(14000 + seed)
    strs = _strings(rng)
    cfg = _config(rng)
    arena, h0 = arena_from_strings(strs)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, 4)
    want_lcp = O.adjacent_lcps(arena, want)
    G = int(rng.choice([1, 2, 3, 4, 7, 9]))
    cuts = np.sort(rng.integers(0, h0.size + 1, G - 1)) if rng.random() < 0.7 else \
        np.array([h0.size * g // G for g in range(1, G)])
    cuts = [0] + [int(c) for c in cuts] + [int(h0.size)]
    shards = [torch.from_numpy(h0[a:b].copy()).cuda() for a, b in zip(cuts[:-1], cuts[1:])]
    slices, lcps = sort_multi_device(arena, shards, [0] * G, cfg)
    got = torch.cat(slices).cpu().numpy()
    lcp = torch.cat(lcps).cpu().numpy()
    tag = f"seed {seed} G={G} cuts={cuts} n={len(strs)} cfg={cfg}"
    assert np.array_equal(np.sort(got), np.sort(h0)), tag
    assert O.contents_equal(arena, got, want), tag
    assert np.array_equal(lcp, want_lcp), tag
