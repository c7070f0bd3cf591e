"""GPU tests of the multi-GPU paths and of concurrent callers.

* ``parallel_sample_sort(..., workers=G)`` over several devices from one
  process (``multi.multi_gpu_sort``); a device may repeat, so the G > 1
  partition / exchange / boundary path runs on a one-GPU box too;
* ``distributed.distributed_sample_sort`` with the production ``GpuBackend``
  over a real NCCL process group (world 1 on one GPU; every visible GPU when
  there are several -- spawned ranks);
* several host threads sorting at once (shared per-device library state);
* the wide-pool overflow error path.

Every result is compared with the CPU oracle (pinned to the reference in
test_oracle_golden.py) or with the reference's digests.
"""
import os
import socket
import threading

import numpy as np
import pytest

import oracle as O
from paper_1305_1157_b200 import (SampleSortConfig, datasets, parallel_sample_sort,
                                  sort_with_lcp)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield


def _want(arena, h0):
    w = h0.copy()
    O.parallel_sample_sort(arena, w, 8)
    return w, O.adjacent_lcps(arena, w)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0, 0, 0, 0, 0]])
@pytest.mark.parametrize("config,n", [(1, None), (3, 1 << 16), (4, 1 << 15), (5, 1 << 16)])
def test_workers_over_devices_matches_oracle(devices, config, n):
    arena, h0 = datasets.generate(config, n)
    want, want_lcp = _want(arena, h0)
    h = h0.copy()
    lcp = np.full(h.size - 1, -7, np.int64)
    out = parallel_sample_sort(arena, h, workers=len(devices), lcp_out=lcp, devices=devices)
    assert out is h
    assert np.array_equal(np.sort(h), np.sort(h0))
    assert O.contents_equal(arena, h, want)
    assert np.array_equal(lcp, want_lcp)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0], [0] * 8])
@pytest.mark.parametrize("config,n", [(1, None), (2, 1 << 17), (3, 1 << 16), (4, 1 << 15),
                                      (5, 1 << 16)])
def test_s5_sort_multi_matches_oracle(devices, config, n):
    """The C-ABI multi-GPU entry (s5_sort_multi): slices in device order are
    the oracle's order, their LCP buffers its LCP array."""
    import torch
    from paper_1305_1157_b200.multi import sort_multi_device
    arena, h0 = datasets.generate(config, n)
    want, want_lcp = _want(arena, h0)
    G = len(devices)
    bounds = [(h0.size * g // G, h0.size * (g + 1) // G) for g in range(G)]
    shards = [torch.from_numpy(h0[a:b].copy()).cuda() for a, b in bounds]
    keep = [s.clone() for s in shards]
    slices, lcps = sort_multi_device(arena, shards, devices)
    for s, k in zip(shards, keep):
        assert torch.equal(s, k)  # inputs untouched
    h = torch.cat(slices).cpu().numpy()
    lcp = torch.cat(lcps).cpu().numpy()
    assert np.array_equal(np.sort(h), np.sort(h0))
    assert O.contents_equal(arena, h, want)
    assert np.array_equal(lcp, want_lcp)


def test_s5_sort_multi_ragged_empty_and_duplicates():
    """Empty shards, a one-string shard, heavy duplicates (identical strings
    must split consistently by handle) and a too-small output buffer."""
    import ctypes as C

    import torch
    from paper_1305_1157_b200 import _lib, arena_from_strings
    from paper_1305_1157_b200.multi import sort_multi_device
    strs = [b"same"] * 30000 + [b"dup-%d" % (i % 7) for i in range(20000)] + [b"", b"z"]
    arena, h0 = arena_from_strings(strs)
    rng = np.random.default_rng(5)
    h0 = h0[rng.permutation(h0.size)]
    want, want_lcp = _want(arena, h0)
    cuts = [0, 0, 1, 40000, 40000, h0.size]
    shards = [torch.from_numpy(h0[a:b].copy()).cuda() for a, b in zip(cuts[:-1], cuts[1:])]
    slices, lcps = sort_multi_device(arena, shards, [0] * 5)
    h = torch.cat(slices).cpu().numpy()
    assert np.array_equal(np.sort(h), np.sort(h0))
    assert O.contents_equal(arena, h, want)
    assert np.array_equal(torch.cat(lcps).cpu().numpy(), want_lcp)
    # the library's cached multi-GPU scratch can be released between calls
    assert _lib.lib().s5_release_caches() == 0
    slices2, _ = sort_multi_device(arena, shards, [0] * 5, want_lcp=False)
    assert O.contents_equal(arena, torch.cat(slices2).cpu().numpy(), want)
    # nothing to sort
    slices, lcps = sort_multi_device(arena, [shards[0], shards[0]], [0, 0])
    assert all(s.numel() == 0 for s in slices)
    # capacity too small -> S5_E_WORKSPACE, message names the slice
    G = 2
    d_ar = arena.device(torch.device("cuda", 0))
    sh = [shards[3], shards[5 - 1]]
    outs = [torch.empty(8, dtype=torch.int64, device="cuda") for _ in range(G)]
    P = lambda ts: (C.c_void_p * G)(*[t.data_ptr() for t in ts])
    rc = _lib.lib().s5_sort_multi(G, (C.c_int * G)(0, 0), P([d_ar, d_ar]), arena.size, P(sh),
                                  (C.c_uint64 * G)(*[s.numel() for s in sh]), P(outs), None,
                                  (C.c_uint64 * G)(8, 8), (C.c_uint64 * G)(), None, None)
    assert rc == -3 and b"slice" in _lib.lib().s5_last_error()


def test_workers_device_tensor_and_duplicates():
    import torch
    from paper_1305_1157_b200 import arena_from_strings
    rng = np.random.default_rng(3)
    strs = [b"dup-%d" % (i % 50) for i in range(20000)] + \
           [bytes(rng.integers(97, 100, rng.integers(0, 9)).tolist()) for _ in range(20000)]
    arena, h0 = arena_from_strings(strs)
    want, want_lcp = _want(arena, h0)
    d = torch.from_numpy(h0).cuda()
    dl = torch.empty(h0.size - 1, dtype=torch.int64, device="cuda")
    parallel_sample_sort(arena, d, workers=3, lcp_out=dl, devices=[0, 0, 0])
    got = d.cpu().numpy()
    assert O.contents_equal(arena, got, want)
    assert np.array_equal(dl.cpu().numpy(), want_lcp)


def test_workers_one_visible_device_is_single_gpu():
    import torch
    arena, h0 = datasets.generate(1, 5000)
    want, want_lcp = _want(arena, h0)
    h = h0.copy()
    lcp = np.empty(h.size - 1, np.int64)
    parallel_sample_sort(arena, h, workers=max(8, torch.cuda.device_count()), lcp_out=lcp)
    assert O.contents_equal(arena, h, want)
    assert np.array_equal(lcp, want_lcp)


@pytest.mark.slow
def test_workers_config5_handle_digest():
    import hashlib
    arena, h0 = datasets.generate(5)
    h = h0.copy()
    lcp = np.empty(h.size - 1, np.int64)
    parallel_sample_sort(arena, h, workers=2, lcp_out=lcp, devices=[0, 0])
    dig, first = datasets.HANDLE_DIGESTS[5]
    assert hashlib.sha256(h.tobytes()).hexdigest()[:16] == dig
    assert h[:5].tolist() == first
    assert O.digest_lcp(lcp)[:16] == datasets.DIGESTS[5][1]


def _nccl_world1(fn):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        return fn()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("config,n", [(1, None), (3, 1 << 17), (5, 1 << 18)])
def test_distributed_gpu_backend_nccl_world1(config, n):
    import torch
    from paper_1305_1157_b200.distributed import GpuBackend, distributed_sample_sort
    arena, h0 = datasets.generate(config, n)
    want, want_lcp = _want(arena, h0)

    def run():
        be = GpuBackend(arena)
        res = distributed_sample_sort(arena, torch.from_numpy(h0).cuda(), backend=be)
        return res.handles.cpu().numpy(), res.lcp.cpu().numpy(), res.offset, res.counts
    got, lcp, off, counts = _nccl_world1(run)
    assert off == 0 and counts == [h0.size]
    assert O.contents_equal(arena, got, want)
    assert np.array_equal(lcp, want_lcp)


@pytest.mark.slow
def test_distributed_nccl_world1_config5_digest():
    import hashlib

    import torch
    from paper_1305_1157_b200.distributed import GpuBackend, distributed_sample_sort
    arena, h0 = datasets.generate(5)

    def run():
        res = distributed_sample_sort(arena, torch.from_numpy(h0).cuda(), backend=GpuBackend(arena))
        return res.handles.cpu().numpy()
    got = _nccl_world1(run)
    dig, first = datasets.HANDLE_DIGESTS[5]
    assert hashlib.sha256(got.tobytes()).hexdigest()[:16] == dig
    assert got[:5].tolist() == first


def _rank_main(rank, world, port, config, n, out_dir):
    import torch
    import torch.distributed as dist
    from paper_1305_1157_b200.distributed import GpuBackend, distributed_sample_sort
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    arena, h0 = datasets.generate(config, n)
    lo, hi = h0.size * rank // world, h0.size * (rank + 1) // world
    res = distributed_sample_sort(arena, torch.from_numpy(h0[lo:hi].copy()).cuda(),
                                  backend=GpuBackend(arena))
    np.save(os.path.join(out_dir, f"h{rank}.npy"), res.handles.cpu().numpy())
    np.save(os.path.join(out_dir, f"l{rank}.npy"), res.lcp.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_nccl_all_visible_gpus(tmp_path):
    import torch
    import torch.multiprocessing as mp
    world = torch.cuda.device_count()
    if world < 2:
        pytest.skip("one visible GPU: the world-1 NCCL tests cover the path")
    arena, h0 = datasets.generate(3, 1 << 18)
    mp.start_processes(_rank_main, args=(world, _free_port(), 3, 1 << 18, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"h{r}.npy") for r in range(world)])
    lcp = np.concatenate([np.load(tmp_path / f"l{r}.npy") for r in range(world)])
    want, want_lcp = _want(arena, h0)
    assert O.contents_equal(arena, got, want)
    assert np.array_equal(lcp, want_lcp)


def test_concurrent_host_callers_one_device():
    # two host threads through the host-buffer path and two through the
    # device path on separate streams: the per-device library state (staging
    # pool, side streams, workspace) must keep them apart
    import torch
    cases = [datasets.generate(1, 60000), datasets.generate(2, 1 << 17),
             datasets.generate(3, 1 << 15), datasets.generate(4, 1 << 15)]
    wants = [_want(a, h) for a, h in cases]
    errors = []

    def host(i):
        try:
            for _ in range(3):
                a, h0 = cases[i]
                h = h0.copy()
                lcp = np.empty(h.size - 1, np.int64)
                parallel_sample_sort(a, h, lcp_out=lcp)
                assert O.contents_equal(a, h, wants[i][0]) and np.array_equal(lcp, wants[i][1])
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    def dev(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    a, h0 = cases[i]
                    d = torch.from_numpy(h0).cuda()
                    _, lcp = sort_with_lcp(a, d)
                    s.synchronize()
                    assert O.contents_equal(a, d.cpu().numpy(), wants[i][0])
                    assert np.array_equal(lcp.cpu().numpy(), wants[i][1])
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))
    ts = [threading.Thread(target=host, args=(0,)), threading.Thread(target=host, args=(1,)),
          threading.Thread(target=dev, args=(2,)), threading.Thread(target=dev, args=(3,))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_wide_pool_overflow_is_reported(monkeypatch):
    monkeypatch.setenv("S5_TEST_POOL_WORDS", "1000")
    arena, h0 = datasets.generate(2, 1 << 18)
    with pytest.raises(RuntimeError, match="wide pool overflow"):
        sort_with_lcp(arena, h0.copy(), cfg=SampleSortConfig(narrow_max=4096))
    monkeypatch.delenv("S5_TEST_POOL_WORDS")
    h, lcp = sort_with_lcp(arena, h0.copy())
    assert O.first_unsorted(arena, h) == -1
