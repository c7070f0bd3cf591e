"""The GPU names in the reference's own benchmark registry (SURVEY 8(f) #1,
pkg/src/strsort/harness.py:185-214, cli.py:27-89).

CPU: the adapter registered into the real reference harness (imported from
/root/reference in a subprocess, so its numba cache stays out of the
read-only tree) with the GPU call replaced by the oracle -- the reference's
run_benchmark then times, verifies and records the GPU names, and its CLI
accepts them.  GPU: the adapter's real sorter through a stand-in registry.
"""
import os
import subprocess
import sys
import types

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"

SCRIPT = r"""
import csv, io, sys
import numpy as np
import oracle as O
from paper_1305_1157_b200 import harness as A
import strsort.harness as H
from strsort.strings import compute_stats

calls = []
def stand_in(name, arena, handles, workers, cfg, counters):
    calls.append((name, workers, cfg.seed + 1))
    O.parallel_sample_sort(arena, handles, workers)   # the oracle as the GPU
    counters.add("parallel_steps", 1)

A.register(H, sorter=stand_in)
A.register(H, sorter=stand_in)          # idempotent
assert H.ALGORITHMS.count("gpu_samplesort") == 1
cfg = H.RunConfig(algorithms=["gpu_samplesort", "gpu_samplesort_equal", "samplesort"],
                  workers=[1, 2], dataset="random", n=3000, reps=2, csv_path=sys.argv[1])
recs = H.run_benchmark(cfg)
assert len(recs) == 3 * 2 * 2 and all(r.verified for r in recs)
assert {r.algorithm for r in recs} == {"gpu_samplesort", "gpu_samplesort_equal", "samplesort"}
arena, h0 = H.build_dataset(cfg)
D = compute_stats(arena, h0).D
w = h0.copy(); O.parallel_sample_sort(arena, w, 1)
assert all(r.D == D == O.distinguishing_prefix(arena, w) for r in recs)
assert calls.count(("gpu_samplesort", 2, 1)) == 2 and len(calls) == 8
rows = list(csv.reader(open(sys.argv[1])))
assert rows[0] == H.RunRecord.csv_header() and len(rows) == 1 + len(recs)
assert all(r.speedup is not None for r in recs)
# the reference CLI accepts the registered names (and still rejects others)
from strsort import cli
c = cli._config_from_args(cli.build_parser().parse_args(
    ["sort", "gpu_samplesort_equal,par_samplesort_unroll", "--random", "100", "--threads", "4"]))
assert c.algorithms == ["gpu_samplesort_equal", "par_samplesort_unroll"] and c.workers == [4]
try:
    cli._config_from_args(cli.build_parser().parse_args(["sort", "gpu_nope", "--random", "9"]))
    raise AssertionError("unknown name accepted")
except SystemExit:
    pass
print("harness adapter ok", D)
"""


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
def test_registered_in_reference_harness(tmp_path):
    env = dict(os.environ, PYTHONPATH=f"{REF_SRC}:{ROOT}", PYTHONDONTWRITEBYTECODE="1",
               NUMBA_CACHE_DIR=str(tmp_path / "numba"))
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(tmp_path / "runs.csv")], env=env,
                       capture_output=True, text=True, timeout=600, cwd=str(tmp_path))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "harness adapter ok" in r.stdout


def test_sorter_config_follows_reference_sample_cfg():
    from paper_1305_1157_b200 import harness as A
    rc = types.SimpleNamespace(v=255, alpha=2, seed=4)
    c = A.sorter_config(rc, "equal")
    assert (c.v, c.alpha, c.classifier, c.seed) == (255, 2, "equal", 5)


@pytest.mark.gpu
def test_gpu_sorter_through_a_registry():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1305_1157_b200 import Counters, datasets
    from paper_1305_1157_b200 import harness as A
    seen = []
    fake = types.SimpleNamespace(ALGORITHMS=["samplesort"],
                                 _run_algorithm=lambda *a: seen.append(a[0]))
    A.register(fake)
    arena, h0 = datasets.generate(1, 20000)
    ref_arena = types.SimpleNamespace(data=arena.data)  # the reference's arena: .data only
    rc = types.SimpleNamespace(v=8191, alpha=2, seed=0)
    want = h0.copy()
    O.parallel_sample_sort(arena, want, 4)
    for name in A.GPU_ALGORITHMS:
        h = h0.copy()
        cnt = Counters()
        fake._run_algorithm(name, ref_arena, h, 1, rc, cnt)
        assert O.contents_equal(arena, h, want), name
        assert cnt.get("parallel_steps") >= 1
    fake._run_algorithm("samplesort", ref_arena, h0.copy(), 1, rc, Counters())
    assert seen == ["samplesort"]
    assert [a for a in fake.ALGORITHMS if a.startswith("gpu_")] == list(A.GPU_ALGORITHMS)
    # the host array is sorted in place on the GPU: a second rep reuses the HBM arena
    h = h0.copy()
    fake._run_algorithm("gpu_samplesort", ref_arena, h, 1, rc, Counters())
    assert np.array_equal(np.sort(h), np.sort(h0))
