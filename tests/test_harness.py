"""The GPU entry of the benchmark harness: registry,
records and CSV in the reference's format (harness.py:142-172, :235-300)."""
import csv

import numpy as np
import pytest

import oracle as O
from paper_1305_1157_b200 import harness as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("kind", ["random", "dna", "config"])
def test_run_benchmark_records(kind, tmp_path):
    out = tmp_path / "runs.csv"
    cfg = H.RunConfig(algorithms=["gpu_samplesort", "gpu_samplesort_equal"], workers=[1, 2],
                      dataset=kind, n=20_000, config=1, reps=2, csv_path=str(out))
    recs = H.run_benchmark(cfg)
    assert len(recs) == 2 * 2 * 2 and all(r.verified for r in recs)
    arena, h = H.build_dataset(cfg)
    want = h.copy()
    O.parallel_sample_sort(arena, want, 4)
    D = int(O.adjacent_lcps(arena, want).size >= 0)  # sortable by the oracle
    assert D == 1 and recs[0].n == h.size
    rows = list(csv.reader(open(out)))
    assert rows[0] == H.RunRecord.csv_header() and len(rows) == 1 + len(recs)
    assert all(r.speedup is not None for r in recs)


def test_file_lines_and_suffixes(tmp_path):
    p = tmp_path / "text.txt"
    rng = np.random.default_rng(2)
    lines = [bytes(rng.integers(97, 101, rng.integers(0, 12)).tolist()) for _ in range(5000)]
    p.write_bytes(b"\n".join(lines) + b"\n")
    recs = H.run_benchmark(H.RunConfig(dataset="file", path=str(p)))
    assert recs[0].n == 5000 and recs[0].verified
    recs = H.run_benchmark(H.RunConfig(dataset="file", path=str(p), suffix=True, max_n=3000))
    assert recs[0].n == 3000 and recs[0].verified
    with pytest.raises(ValueError):
        H.run_benchmark(H.RunConfig(algorithms=["par_mkqs"], dataset="random", n=100))
