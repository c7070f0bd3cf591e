"""Benchmark harness entry for the GPU sorter.

Mirror of the reference's registry and record format for the S^5 path
(pkg/src/strsort/harness.py:108-214, :221-300): a ``RunConfig``, one
``RunRecord`` per (algorithm, workers, rep) with the same CSV columns, every
result verified before it is recorded (``VerificationFailed``), speed-ups
against the 1-worker median.  The algorithms are the GPU sorts:

* ``gpu_samplesort`` / ``gpu_samplesort_unroll`` -- table classifier (the
  count kernel's, same buckets as the unrolled descent);
* ``gpu_samplesort_equal`` -- equality-descent classifier.

``workers`` is recorded but one call sorts on one GPU (multi-GPU runs go
through ``distributed.distributed_sample_sort`` under torchrun).  Datasets:
``random`` / ``dna`` (seeded generators with the reference's parameter
meaning: lengths uniform in [0, 20) over bytes 33..126; fixed-length ACGT
reads), ``config`` (the BASELINE configurations, ``datasets.generate``) and
``file`` (lines ingested on the device, or every suffix of the file).

    python -m paper_1305_1157_b200.harness --dataset config --config 2 --reps 3 --csv out.csv
"""

from __future__ import annotations

import argparse
import csv
import io
import statistics
import sys
import time
from dataclasses import dataclass, field

import numpy as np

from .counters import Counters
from .samplesort import SampleSortConfig, parallel_sample_sort
from .strings import StringArena, compute_stats, verify_sorted_permutation


class VerificationFailed(RuntimeError):
    """harness.py:30-31."""


ALGORITHMS = ["gpu_samplesort", "gpu_samplesort_unroll", "gpu_samplesort_equal"]


@dataclass
class RunConfig:
    """harness.py:108-139 (the GPU subset of its knobs)."""
    algorithms: list[str] = field(default_factory=lambda: ["gpu_samplesort"])
    workers: list[int] = field(default_factory=lambda: [1])
    dataset: str = "random"        # random | dna | config | file
    n: int = 100_000
    config: int = 2
    path: str | None = None
    suffix: bool = False
    max_n: int | None = None
    dna_length: int = 9
    seed: int = 0
    reps: int = 1
    csv_path: str | None = None
    v: int = 8191
    alpha: int = 2

    def dataset_label(self) -> str:
        if self.dataset == "file":
            import os
            return f"file:{os.path.basename(str(self.path))}:{'suffix' if self.suffix else 'lines'}"
        if self.dataset == "dna":
            return f"dna:{self.n}x{self.dna_length}:seed{self.seed}"
        if self.dataset == "config":
            return f"config{self.config}"
        return f"random:{self.n}:seed{self.seed}"


@dataclass
class RunRecord:
    """harness.py:142-172: same fields and CSV columns."""
    algorithm: str
    workers: int
    dataset: str
    n: int
    N: int
    D: int
    rep: int
    time_ns: int
    speedup: float | None
    verified: bool
    counters: dict

    COUNTER_COLUMNS = ("fetches", "jobs", "shares", "share_requests", "max_queue",
                       "parallel_steps", "parallel_partitions")

    def csv_row(self) -> list:
        row = [self.algorithm, self.workers, self.dataset, self.n, self.N, self.D, self.rep,
               self.time_ns, "" if self.speedup is None else f"{self.speedup:.4f}",
               int(self.verified)]
        row.extend(self.counters.get(c, 0) for c in self.COUNTER_COLUMNS)
        return row

    @staticmethod
    def csv_header() -> list[str]:
        return ["algorithm", "workers", "dataset", "n", "N", "D", "rep", "time_ns", "speedup",
                "verified", *RunRecord.COUNTER_COLUMNS]


def _random_strings(n: int, seed: int):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 20, n)
    starts = np.concatenate([[0], np.cumsum(lens + 1)[:-1]]).astype(np.int64)
    data = np.zeros(int(lens.sum()) + n, np.uint8)
    body = np.repeat(starts, lens) + (np.arange(int(lens.sum())) -
                                      np.repeat(np.cumsum(lens) - lens, lens))
    data[body] = rng.integers(33, 127, body.size, dtype=np.uint8)
    return StringArena(data), starts


def _dna_reads(n: int, length: int, seed: int):
    rng = np.random.default_rng(seed)
    rows = np.zeros((n, length + 1), np.uint8)
    rows[:, :length] = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, (n, length))]
    return StringArena(rows.reshape(-1)), np.arange(0, n * (length + 1), length + 1, dtype=np.int64)


def build_dataset(cfg: RunConfig):
    """harness.py:221-232, plus the BASELINE configurations."""
    if cfg.dataset == "random":
        return _random_strings(cfg.n, cfg.seed)
    if cfg.dataset == "dna":
        return _dna_reads(cfg.n, cfg.dna_length, cfg.seed)
    if cfg.dataset == "config":
        from . import datasets
        return datasets.generate(cfg.config, None if cfg.n == RunConfig.n else cfg.n)
    if cfg.dataset == "file":
        if cfg.path is None:
            raise ValueError("file dataset needs a path")
        with open(cfg.path, "rb") as f:
            raw = f.read()
        if cfg.suffix:  # harness.py:98-102: one handle per byte, one terminator
            if b"\x00" in raw:
                from .strings import EmbeddedNul
                raise EmbeddedNul(raw.index(b"\x00"))
            n = len(raw) if cfg.max_n is None else min(cfg.max_n, len(raw))
            return StringArena(np.frombuffer(raw + b"\x00", np.uint8)), np.arange(n, dtype=np.int64)
        from .strings import ingest_lines
        arena, h = ingest_lines(raw)
        return arena, h.cpu().numpy()
    raise ValueError(f"unknown dataset kind {cfg.dataset!r}")


def _run_algorithm(name: str, arena, handles, workers: int, cfg: RunConfig, counters: Counters):
    """The registry entry (harness.py:185-214)."""
    if name not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {name!r}")
    classifier = "equal" if name == "gpu_samplesort_equal" else "unroll"
    parallel_sample_sort(arena, handles, workers,
                         cfg=SampleSortConfig(v=cfg.v, alpha=cfg.alpha, classifier=classifier,
                                              seed=cfg.seed + 1), counters=counters)


def run_benchmark(cfg: RunConfig, out=None) -> list[RunRecord]:
    """harness.py:235-265: every combination timed (wall, host buffers in and
    out) and verified on the device."""
    arena, handles0 = build_dataset(cfg)
    if handles0.size == 0:
        raise ValueError("dataset is empty")
    stats = compute_stats(arena, handles0)
    label = cfg.dataset_label()
    records = []
    for algo in cfg.algorithms:
        for workers in cfg.workers:
            for rep in range(cfg.reps):
                handles = handles0.copy()
                counters = Counters()
                t0 = time.perf_counter_ns()
                _run_algorithm(algo, arena, handles, workers, cfg, counters)
                elapsed = time.perf_counter_ns() - t0
                check = verify_sorted_permutation(arena, handles0, handles)
                if not check.ok:
                    raise VerificationFailed(f"{algo} with {workers} workers on {label}: "
                                             f"{check.message()}")
                records.append(RunRecord(algo, workers, label, stats.n, stats.N, stats.D, rep,
                                         elapsed, None, True, counters.as_dict()))
                if out is not None:
                    print(f"{algo:24s} p={workers:<3d} rep={rep} {elapsed / 1e6:10.2f} ms  verified",
                          file=out)
    base = {}
    for algo in {r.algorithm for r in records}:
        ts = [r.time_ns for r in records if r.algorithm == algo and r.workers == 1]
        if ts:
            base[algo] = statistics.median(ts)
    for r in records:
        if r.algorithm in base and r.time_ns > 0:
            r.speedup = base[r.algorithm] / r.time_ns
    if cfg.csv_path:
        write_csv(records, cfg.csv_path)
    return records


def write_csv(records: list[RunRecord], path) -> None:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(RunRecord.csv_header())
    for r in records:
        w.writerow(r.csv_row())
    with open(path, "w", newline="") as f:
        f.write(buf.getvalue())


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--algorithms", nargs="+", default=["gpu_samplesort"], choices=ALGORITHMS)
    ap.add_argument("--workers", nargs="+", type=int, default=[1])
    ap.add_argument("--dataset", default="random", choices=["random", "dna", "config", "file"])
    ap.add_argument("--n", type=int, default=RunConfig.n)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--path")
    ap.add_argument("--suffix", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--csv")
    a = ap.parse_args(argv)
    cfg = RunConfig(algorithms=a.algorithms, workers=a.workers, dataset=a.dataset, n=a.n,
                    config=a.config, path=a.path, suffix=a.suffix, seed=a.seed, reps=a.reps,
                    csv_path=a.csv)
    run_benchmark(cfg, out=sys.stdout)
    return 0


if __name__ == "__main__":
    sys.exit(main())
