"""World-size-2 (and 3) CPU tests of the multi-GPU partitioning logic
(paper_1305_1157_b200.distributed) over gloo.  The string primitives are
injected from the CPU oracle (test-only backend); the production backend is
the GPU library."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1305_1157_b200 import datasets
from paper_1305_1157_b200.distributed import compare_strings, distributed_sample_sort
from paper_1305_1157_b200.strings import StringArena, arena_from_strings


class OracleBackend:
    def __init__(self, arena):
        self.arena = arena

    def pack_keys(self, handles, depth):
        k = O.pack_keys(self.arena, handles.numpy(), depth)
        return torch.from_numpy(k.view(np.int64).copy())

    def lengths(self, handles):
        return torch.from_numpy(O.string_lengths(self.arena, handles.numpy()))

    def ends_at(self, handles, pos):
        data = torch.from_numpy(self.arena.data)
        return data[(handles + pos).clamp(0, self.arena.size - 1)] == 0

    def partition(self, h, splitters):
        # binary search over the splitters with full-string comparison
        n, G = h.numel(), splitters.numel() + 1
        lo = torch.zeros(n, dtype=torch.int64)
        hi = torch.full((n,), G - 1, dtype=torch.int64)
        while True:
            idx = torch.nonzero(lo < hi).flatten()
            if not idx.numel():
                break
            mid = (lo[idx] + hi[idx]) // 2
            right = compare_strings(self, splitters[mid], h[idx]) < 0  # splitter < string
            lo[idx[right]] = mid[right] + 1
            hi[idx[~right]] = mid[~right]
        order = torch.argsort(lo, stable=True)
        return h[order], torch.bincount(lo, minlength=G).tolist()

    def lcp_pair(self, pair):
        return torch.from_numpy(O.adjacent_lcps(self.arena, pair.numpy()))

    def sort_u32(self, buf, n):
        h = buf.view(torch.int32)[:n].numpy().view(np.uint32).astype(np.int64)
        buf[:n] = torch.from_numpy(h)
        return self.sort(buf[:n])

    def sort(self, handles):
        h = handles.numpy().copy()
        O.parallel_sample_sort(self.arena, h, 1)
        return torch.from_numpy(h), torch.from_numpy(O.adjacent_lcps(self.arena, h))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, data, handles, shards, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    arena = StringArena(data)
    lo, hi = shards[rank]
    local = torch.from_numpy(handles[lo:hi].copy())
    res = distributed_sample_sort(arena, local, oversample=16, backend=OracleBackend(arena))
    np.save(os.path.join(out_dir, f"h{rank}.npy"), res.handles.numpy())
    np.save(os.path.join(out_dir, f"l{rank}.npy"), res.lcp.numpy())
    np.save(os.path.join(out_dir, f"o{rank}.npy"), np.asarray([res.offset]))
    dist.barrier()
    dist.destroy_process_group()


def _run(data, handles, shards, tmp_path):
    world = len(shards)
    mp.start_processes(_worker, args=(world, _free_port(), data, handles, shards, str(tmp_path)),
                       nprocs=world, join=True, start_method="fork")
    hs = [np.load(tmp_path / f"h{r}.npy") for r in range(world)]
    ls = [np.load(tmp_path / f"l{r}.npy") for r in range(world)]
    offs = [int(np.load(tmp_path / f"o{r}.npy")[0]) for r in range(world)]
    return hs, ls, offs


def _even(n, world):
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


CASES = {
    "random": lambda: arena_from_strings(
        [bytes(np.random.default_rng(i).integers(97, 101, i % 13).tolist()) for i in range(3000)]),
    "config1_small": lambda: datasets.generate(1, 1 << 12),
    "identical": lambda: arena_from_strings([b"same-string-of-twenty"] * 700 + [b"x"] * 5),
    "suffixes": lambda: datasets.generate(5, 1 << 12),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("world", [2, 3])
def test_distributed_matches_oracle(case, world, tmp_path):
    arena, handles = CASES[case]()
    hs, ls, offs = _run(arena.data, handles, _even(handles.size, world), tmp_path)
    got = np.concatenate(hs)
    lcp = np.concatenate(ls)
    want = handles.copy()
    O.parallel_sample_sort(arena, want, 1)
    assert np.array_equal(np.sort(got), np.sort(handles))
    assert O.contents_equal(arena, got, want)
    assert np.array_equal(lcp, O.adjacent_lcps(arena, want))
    assert offs == [sum(h.size for h in hs[:r]) for r in range(world)]


def test_distributed_uneven_and_empty_shard(tmp_path):
    arena, handles = datasets.generate(1, 2000)
    hs, ls, _ = _run(arena.data, handles, [(0, 0), (0, 2000)], tmp_path)
    got = np.concatenate(hs)
    want = handles.copy()
    O.parallel_sample_sort(arena, want, 1)
    assert O.contents_equal(arena, got, want)
    assert np.array_equal(np.concatenate(ls), O.adjacent_lcps(arena, want))


def test_compare_strings_tiebreak():
    arena, h = arena_from_strings([b"abc", b"abd", b"abc", b"ab", b"abcdefghijk", b"abcdefghijl"])
    be = OracleBackend(arena)
    a = torch.from_numpy(h[[0, 0, 0, 3, 4, 2]].copy())
    b = torch.from_numpy(h[[1, 2, 3, 0, 5, 0]].copy())
    assert compare_strings(be, a, b).tolist() == [-1, -1, 1, -1, -1, 1]
