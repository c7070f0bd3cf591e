"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's inputs (URL crawl, GOV2, Wikipedia, Sinha sets)
are not available, so each configuration is a deterministic numpy recipe
 whose draw order is fixed.  Strings are laid out
back-to-back, each followed by one 0 byte, mirroring the reference generator
``generate_random`` (pkg/src/strsort/harness.py:45-56); config 5 is suffix
mode (one terminator after the text, one handle per position;
harness.py:97-102).

Every generator returns ``(StringArena, handles)`` like the reference's
generators.  Self-check values (N, D) are in ``EXPECTED``.
"""

from __future__ import annotations

import numpy as np

from .strings import StringArena

#: (n, N = arena bytes incl. terminators, D) per config, SURVEY.md 8 sizing table
EXPECTED = {
    1: (1 << 17, 1_966_333, 558_618),
    2: (1 << 25, 587_282_149, 141_001_734),
    3: (1 << 24, 1_053_323_519, 681_702_787),
    4: (1 << 25, 3_388_997_632, 1_025_719_795),
    5: (1 << 27, 134_217_729, 812_183_397),
}

#: sha256[:16] of the reference's sorted strings / LCP array
DIGESTS = {
    1: ("9f63d4cb347c8f3b", "39359fe05433b14b"),
    2: ("c52124844d1bf643", "8886a05ec8693487"),
    3: ("6693b4e40216e0a4", "2e1d9f4d1452ac7c"),
    4: ("fc15a779a317f83b", "715d398ee96e234b"),
    5: ("ad23b81651a34cef", "6fe7b06e97f0fc71"),
}

#: config 5 has no duplicates, so the sorted handle array itself is unique:
#: sha256[:16] of its int64 LE bytes and its first five entries
HANDLE_DIGESTS = {5: ("0f9c3331ca2ab3a2", [8554485, 128901439, 12150689, 619002, 15495257])}

DESCRIPTION = {
    1: "random a-z, length U[8,20], n=2^17, seed 1",
    2: "random printable ASCII 0x21-0x7E, length U[1,32], n=2^25, seed 2",
    3: "URL-like http://host/word/..., Zipf(1.1) hosts (2^12) and words (2^14), n=2^24, seed 3",
    4: "DNA reads of length 100 from a 2^28 ACGT genome, 5% exact duplicates, n=2^25, seed 4",
    5: "all 2^27 suffixes of an order-2 Markov text over 64 symbols, Dirichlet(0.3) rows, seed 5",
}


def _pack(lengths: np.ndarray, body: np.ndarray):
    """Back-to-back layout: handles[i] = sum_{j<i} (L_j + 1), one 0 after each."""
    n = lengths.size
    total = int(lengths.sum()) + n
    data = np.zeros(total, np.uint8)
    handles = np.zeros(n, np.int64)
    if n > 1:
        np.cumsum(lengths[:-1] + 1, out=handles[1:])
    mask = np.ones(total, bool)
    mask[handles + lengths] = False
    data[mask] = body
    return StringArena(data), handles


def gen_config1(n: int = 1 << 17, seed: int = 1):
    rng = np.random.default_rng(seed)
    lengths = rng.integers(8, 21, n)
    body = rng.integers(97, 123, int(lengths.sum()), dtype=np.uint8)
    return _pack(lengths, body)


def gen_config2(n: int = 1 << 25, seed: int = 2):
    rng = np.random.default_rng(seed)
    lengths = rng.integers(1, 33, n)
    body = rng.integers(0x21, 0x7F, int(lengths.sum()), dtype=np.uint8)
    return _pack(lengths, body)


def _zipf_inverse_cdf(k: int, s: float, u: np.ndarray) -> np.ndarray:
    w = np.arange(1, k + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return np.minimum(np.searchsorted(cdf, u, side="left"), k - 1)


def gen_config3(n: int = 1 << 24, seed: int = 3):
    rng = np.random.default_rng(seed)

    def word(lo, hi):
        ln = rng.integers(lo, hi + 1)
        return bytes(rng.integers(97, 123, ln).astype(np.uint8))

    tlds = (b".com", b".org", b".net")
    hosts = []
    for _ in range(4096):
        w = word(6, 15)
        hosts.append(w + tlds[int(rng.integers(0, 3))])
    vocab = [word(4, 16) for _ in range(16384)]
    host_idx = _zipf_inverse_cdf(4096, 1.1, rng.random(n))
    nseg = rng.integers(1, 7, n)
    word_idx = _zipf_inverse_cdf(16384, 1.1, rng.random(int(nseg.sum())))

    # vectorised assembly: string = "http://" + host + "/" + "/".join(words)
    host_len = np.array([len(h) for h in hosts], np.int64)
    voc_len = np.array([len(w) for w in vocab], np.int64)
    host_blob = np.frombuffer(b"".join(hosts), np.uint8)
    voc_blob = np.frombuffer(b"".join(vocab), np.uint8)
    host_off = np.concatenate(([0], np.cumsum(host_len)[:-1]))
    voc_off = np.concatenate(([0], np.cumsum(voc_len)[:-1]))

    seg_start = np.concatenate(([0], np.cumsum(nseg)[:-1]))
    words_len = np.add.reduceat(voc_len[word_idx], seg_start) + (nseg - 1)
    lengths = 7 + host_len[host_idx] + 1 + words_len
    total = int(lengths.sum()) + n
    data = np.zeros(total, np.uint8)
    handles = np.zeros(n, np.int64)
    np.cumsum(lengths[:-1] + 1, out=handles[1:])

    # "http://"
    prefix = np.frombuffer(b"http://", np.uint8)
    for j in range(7):
        data[handles + j] = prefix[j]
    # host bytes
    _scatter_pieces(data, handles + 7, host_off[host_idx], host_len[host_idx], host_blob)
    # "/" after host
    pos = handles + 7 + host_len[host_idx]
    data[pos] = ord("/")
    pos = pos + 1
    # words joined by "/"
    owner = np.repeat(np.arange(n), nseg)
    rank = np.arange(word_idx.size) - np.repeat(seg_start, nseg)
    wl = voc_len[word_idx]
    # start of each word inside its string: cumulative (len+1) within the string
    cum = np.cumsum(wl + 1)
    cum_before = cum - (wl + 1)
    base = np.repeat(cum_before[seg_start], nseg)
    wstart = pos[owner] + (cum_before - base)
    _scatter_pieces(data, wstart, voc_off[word_idx], wl, voc_blob)
    sep = rank > 0
    data[wstart[sep] - 1] = ord("/")
    return StringArena(data), handles


def _scatter_pieces(data, dst_start, src_start, lengths, blob, chunk=1 << 22):
    """data[dst_start[i] + j] = blob[src_start[i] + j] for j < lengths[i]."""
    try:
        from . import _native
        return _native.copy_pieces(data, dst_start, src_start, lengths, blob)
    except ImportError:  # library not built: the numpy restatement
        pass
    m = lengths.size
    for a in range(0, m, chunk):
        b = min(m, a + chunk)
        ln = lengths[a:b]
        tot = int(ln.sum())
        rep = np.repeat(np.arange(b - a), ln)
        within = np.arange(tot) - np.repeat(np.cumsum(ln) - ln, ln)
        data[dst_start[a:b][rep] + within] = blob[src_start[a:b][rep] + within]


def gen_config4(n: int = 1 << 25, seed: int = 4, read_len: int = 100,
                genome_len: int = 1 << 28, chunk: int = 1 << 20):
    rng = np.random.default_rng(seed)
    letters = np.frombuffer(b"ACGT", np.uint8)
    genome = letters[rng.integers(0, 4, genome_len)]
    off = rng.integers(0, genome_len - read_len + 1, n)
    dup = rng.random(n) < 0.05
    dup[0] = False
    di = np.nonzero(dup)[0]
    ru = rng.random(di.size)
    src = (ru * di).astype(np.int64)
    # ascending sequential assignment keeps duplicates of duplicates exact
    _assign_dups(off, di, src)
    stride = read_len + 1
    data = np.zeros(n * stride, np.uint8)
    win = np.lib.stride_tricks.sliding_window_view(genome, read_len)
    view = data.reshape(n, stride)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        view[a:b, :read_len] = win[off[a:b]]
    handles = np.arange(0, n * stride, stride, dtype=np.int64)
    return StringArena(data), handles


def _assign_dups(off: np.ndarray, di: np.ndarray, src: np.ndarray) -> None:
    """for i, s in zip(di, src) (ascending i): off[i] = off[s]; s < i always.

    Resolved with pointer jumping instead of a Python loop: each duplicate's
    final source is the first non-duplicate reached by following src links,
    which is exactly what the sequential assignment produces."""
    parent = np.arange(off.size, dtype=np.int64)
    parent[di] = src
    while True:
        nxt = parent[parent]
        if np.array_equal(nxt, parent):
            break
        parent = nxt
    off[di] = off[parent[di]]


def gen_config5(n: int = 1 << 27, seed: int = 5, sigma: int = 64, alpha: float = 0.3):
    from . import _native
    rng = np.random.default_rng(seed)
    P = rng.dirichlet(np.full(sigma, alpha), size=(sigma, sigma))
    u = rng.random(n)
    cdf = np.ascontiguousarray(np.cumsum(P, axis=2), np.float64)
    text = _native.markov_text(cdf, u, sigma)
    data = np.empty(n + 1, np.uint8)
    data[:n] = text
    data[n] = 0
    return StringArena(data), np.arange(n, dtype=np.int64)


GENERATORS = {1: gen_config1, 2: gen_config2, 3: gen_config3, 4: gen_config4, 5: gen_config5}


def generate(config: int, n: int | None = None):
    """Arena + handles for a BASELINE config; ``n`` shrinks it (same recipe)."""
    gen = GENERATORS[config]
    return gen() if n is None else gen(n)
