"""Benchmark: S^5 string sample sort + LCP on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one sort (with LCP output) of one BASELINE configuration's synthetic
strings.  Default workload: config 2 (n = 2^25 random strings, the
configuration BASELINE.json's metric is quoted on that fits one GPU).

Our arm (default): inputs resident in HBM; before every step the unsorted
handle array is restored and L2 is flushed (untimed); each step is timed with
CUDA events on the sorting stream; the max over ranks is taken.  Extra keys:
``e2e`` (public API with host numpy buffers: H2D handles, sort, D2H handles +
LCP), ``roofline`` (dominant kernel, per-kernel CUDA events in a separate
profiled pass), ``roofline_sort`` (whole sort, SURVEY.md 8(d) B_alg), and
``cpu_baseline`` (the C port of the reference's parallel S^5, oracle/, on the
host cores).

``--impl reference``: the reference's CPU algorithm (C port of pS^5,
oracle/s5_oracle.c, all host threads) on the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback

METRIC = "strings/s sorted (S^5 string sample sort with LCP array)"


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(config: int, n: int | None):
    from paper_1305_1157_b200 import datasets
    t = time.time()
    arena, h0 = datasets.generate(config, n)
    return arena, h0, time.time() - t


def run_reference(args):
    """CPU reference arm: C port of pS^5 (oracle/), all host threads."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    from paper_1305_1157_b200 import datasets
    arena, h0, _ = workload(args.config, args.n)
    n = h0.size
    threads = O.max_threads()
    for _ in range(args.warmup):
        h = h0.copy()
        O.parallel_sample_sort(arena, h, threads)
    times = []
    for _ in range(args.steps):
        h = h0.copy()
        t0 = time.perf_counter()
        O.parallel_sample_sort(arena, h, threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = n * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "strings/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"config{args.config}: {datasets.DESCRIPTION[args.config]}",
                   "n": int(n), "arena_bytes": int(arena.data.size)},
        "cpu_baseline": {"value": value, "unit": "strings/s", "cores": threads, "kind": "port",
                         "sample": f"full config-{args.config} workload per step "
                                   f"(n={n}), C port of pS^5 (oracle/s5_oracle.c)"},
        "e2e": {"value": value, "unit": "strings/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "d_chars_per_s": None,
    }
    D = datasets.EXPECTED.get(args.config, (0, 0, 0))[2] if args.n is None else None
    if D:
        line["d_chars_per_s"] = D * args.steps / total
    print(json.dumps(line), flush=True)


def run_distributed(args):
    """N > 1 (torchrun): one global sort of the config's n strings across the
    ranks -- sample-sort partitioning + NCCL all-to-all + local S^5
    (paper_1305_1157_b200.distributed).  Strong scaling: n is fixed."""
    import torch
    import torch.distributed as dist

    from paper_1305_1157_b200 import datasets
    from paper_1305_1157_b200.distributed import GpuBackend, distributed_sample_sort
    from paper_1305_1157_b200.strings import first_unsorted

    if "RANK" not in os.environ:  # one-rank smoke run without torchrun
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    arena, h0, _ = workload(args.config, args.n)
    n = h0.size
    cfg = make_cfg(args)
    arena.device(dev)
    lo, hi = n * rank // world, n * (rank + 1) // world
    shard_host = np.ascontiguousarray(h0[lo:hi])
    shard = torch.from_numpy(shard_host).to(dev)
    be = GpuBackend(arena, cfg)
    l2_flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        distributed_sample_sort(arena, shard.clone(), backend=be)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    times = []
    res = None
    be.launches = 0
    for _ in range(args.steps):
        d = shard.clone()
        l2_flush.zero_()
        dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        res = distributed_sample_sort(arena, d, backend=be)
        ev1.record(stream)
        torch.cuda.synchronize()
        times.append(ev0.elapsed_time(ev1))
    clk = clocks.stop()
    launches = be.launches
    t = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    ok = torch.tensor([1 if first_unsorted(arena, res.handles) == -1 else 0], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    # e2e: host shard in, host slice + LCP out (host result buffers allocated
    # and touched once, as a caller reusing them would)
    e2e = []
    out_hb = np.full(n, -1, np.int64)
    out_lb = np.full(n, -1, np.int64)
    for it in range(1 + max(1, args.steps // 2)):  # first round untimed (staging set-up)
        dist.barrier()
        t0 = time.perf_counter()
        d = be.upload(shard_host)
        r = distributed_sample_sort(arena, d, backend=be)
        out_h, out_l = be.download(r.handles, r.lcp, out_hb, out_lb)
        if it:
            e2e.append(time.perf_counter() - t0)
    te = torch.tensor([sum(e2e) / len(e2e)], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    if rank == 0:
        D = datasets.EXPECTED.get(args.config, (0, 0, 0))[2] if args.n is None else None
        line = {
            "metric": METRIC, "value": n / (ms_per_step * 1e-3), "unit": "strings/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"config{args.config}: {datasets.DESCRIPTION[args.config]}",
                       "n": int(n), "arena_bytes": int(arena.data.size),
                       "parallelism": f"dp{world}: sample-sort partition, NCCL all-to-all, local S^5",
                       "l2": "256 MiB L2 flush before every step (untimed)"},
            "d_chars_per_s": D / (ms_per_step * 1e-3) if D else None,
            "e2e": {"value": n / float(te.item()), "unit": "strings/s",
                    "h2d_bytes_per_step": int(4 * n), "d2h_bytes_per_step": int(4 * n + (n - 1)),
                    "note": "host shards in, host slices + LCP out, all ranks; u32 handles and "
                            "narrow LCPs over PCIe (s5_upload_handles / s5_download)"},
            "sorted_ok": bool(ok.item()), "slice_sizes": res.counts, "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1305_1157_b200 import _lib, datasets
    from paper_1305_1157_b200.samplesort import SampleSortConfig, gpu_sort, parallel_sample_sort
    from paper_1305_1157_b200.strings import distinguishing_prefix

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    arena, h0, gen_s = workload(args.config, args.n)
    n = h0.size
    cfg = make_cfg(args)
    t_up = time.perf_counter()
    arena.device(dev)
    torch.cuda.synchronize()
    arena_upload_s = time.perf_counter() - t_up
    d_h0 = torch.from_numpy(h0).to(dev)
    d_h = torch.empty_like(d_h0)
    d_lcp = torch.empty(n - 1, dtype=torch.int64, device=dev)
    l2_flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # 256 MiB > L2
    stream = torch.cuda.current_stream()

    def one_step(stats=None, cfg_=cfg):
        d_h.copy_(d_h0)
        l2_flush.zero_()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        gpu_sort(arena, d_h, 0, cfg_, d_lcp, stats)
        ev1.record(stream)
        return ev0, ev1

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    events = []
    stats = _lib.S5Stats()
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        events.append(one_step(stats))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in events]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    st = stats.as_dict()
    launches_per_step = int(stats.launches)

    # correctness of the timed output (cheap device checks)
    from paper_1305_1157_b200.strings import first_unsorted
    assert first_unsorted(arena, d_h) == -1, "bench output not sorted"
    D = distinguishing_prefix(arena, d_h, d_lcp)

    # per-kernel device times: separate profiled steps (CUDA events per launch)
    pcfg = make_cfg(args)
    prof_stats = []
    for _ in range(max(1, min(args.steps, 3))):
        ps = _lib.S5Stats()
        c = pcfg.to_c()
        one_step_prof(arena, d_h, d_h0, d_lcp, pcfg, ps, l2_flush)
        prof_stats.append(ps.as_dict())
    kern = {}
    for ps in prof_stats:
        for name, rec in ps["kernels"].items():
            k = kern.setdefault(name, {"ms": 0.0, "launches": 0, "strings": 0})
            k["ms"] += rec["ms"] / len(prof_stats)
            k["launches"] += rec["launches"] / len(prof_stats)
            k["strings"] += rec["strings"] / len(prof_stats)
    peak, peak_src = hbm_peak()
    n_p = st["n_per_pass"]
    B_alg = 16 * sum(n_p) + D  # 16 B per string per S^5 level / base-case pass
    # dominant kernel and its algorithmic bytes: 16 B (8-B pointer read + write,
    # SURVEY 8(d)) per string it moves, strings counted by the library per launch
    dom = max(kern.items(), key=lambda kv: kv[1]["ms"]) if kern else \
        ("none", {"ms": 0, "launches": 1, "strings": 0})
    dom_name, dom_rec = dom
    strings = dom_rec["strings"]
    launches = max(dom_rec["launches"], 1)
    per_launch_bytes = 16.0 * strings / launches
    per_launch_ms = dom_rec["ms"] / launches
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"config{args.config}", {}).get(dom_name)
        except Exception:
            traffic = None

    # e2e through the public API with host buffers
    e2e_times = []
    h_host = np.empty_like(h0)
    lcp_host = np.empty(n - 1, np.int64)
    for i in range(args.warmup + args.steps):
        np.copyto(h_host, h0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        parallel_sample_sort(arena, h_host, cfg=cfg, lcp_out=lcp_host)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_times.append(dt)
    e2e_s = sum(e2e_times) / len(e2e_times)
    from paper_1305_1157_b200 import samplesort as _ss
    e2e_phases = dict(_ss.LAST_HOST_MS)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    value = world * n / (ms_per_step * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "strings/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"config{args.config}: {datasets.DESCRIPTION[args.config]}",
                   "n": int(n), "arena_bytes": int(arena.data.size), "D": int(D),
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": "256 MiB L2 flush + handle restore before every step (untimed)",
                   "classifier": args.classifier, "overrides": args.cfg},
        "d_chars_per_s": world * D / (ms_per_step * 1e-3),
        "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak if peak else None,
                     "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
                     "algorithmic_bytes": "16 B per string moved by the launch "
                                          "(8-B pointer read + write, SURVEY 8(d))"},
        "roofline_sort": {"B_alg": B_alg, "floor_bytes": 16 * n + D,
                          "achieved_gbs": B_alg / (ms_per_step * 1e-3) / 1e9,
                          "frac": B_alg / (ms_per_step * 1e-3) / 1e9 / peak,
                          "floor_frac": (16 * n + D) / (ms_per_step * 1e-3) / 1e9 / peak},
        "n_per_pass": n_p,
        "kernels_ms_per_step": {k: round(v["ms"], 4) for k, v in sorted(kern.items())},
        "kernels_strings_per_step": {k: int(v["strings"]) for k, v in sorted(kern.items())},
        "launch_recs": prof_stats[-1].get("launch_recs", []) if args.launch_recs else None,
        "e2e": {"value": world * n / e2e_s, "unit": "strings/s",
                "h2d_bytes_per_step": int(e2e_phases.get("h2d_bytes", 8 * n)),
                "d2h_bytes_per_step": int(e2e_phases.get("d2h_bytes", 16 * n - 8)),
                "ms_per_step": 1e3 * e2e_s,
                "note": "parallel_sample_sort(numpy int64 handles, lcp_out=numpy int64): "
                        "handles cross PCIe as u32 both ways, LCPs in the narrowest width "
                        "holding their maximum; H2D + sort + D2H + host widening",
                "phases_ms": e2e_phases},
        "arena_upload_s": arena_upload_s,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
        "wall_s_timed_region": wall,
        "step_ms": [round(x, 4) for x in step_ms],
        "levels": st["levels"],
        "tiers_per_level": {t: st[f"{t}_elems"] for t in ("wide", "narrow", "local", "small")},
        "key_fetches": st["key_fetches"], "boundary_lcps": st["boundary_lcps"],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(arena, h0, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def make_cfg(args):
    from paper_1305_1157_b200.samplesort import SampleSortConfig
    kw = {"classifier": args.classifier}
    for item in args.cfg:
        k, _, v = item.partition("=")
        kw[k] = int(v) if v.lstrip("-").isdigit() else v
    return SampleSortConfig(**kw)


def one_step_prof(arena, d_h, d_h0, d_lcp, cfg, stats, l2_flush):
    import ctypes as C
    import torch
    from paper_1305_1157_b200 import _lib
    from paper_1305_1157_b200.samplesort import _workspace
    d_h.copy_(d_h0)
    l2_flush.zero_()
    c = cfg.to_c()
    c.flags |= 2
    n = d_h.numel()
    need = int(_lib.lib().s5_workspace_bytes(n, arena.data.size, C.byref(c)))
    ws = _workspace(need, d_h.device)
    rc = _lib.lib().s5_sort(arena.device(d_h.device).data_ptr(), arena.data.size, d_h.data_ptr(),
                            n, 0, d_lcp.data_ptr(), C.byref(c), ws.data_ptr(), ws.numel(),
                            _lib.current_stream_ptr(), C.byref(stats))
    _lib.check(rc, "s5_sort (profiled)")
    torch.cuda.synchronize()


def cpu_baseline(arena, h0, args):
    import oracle as O
    threads = O.max_threads()
    h = h0.copy()
    t0 = time.perf_counter()
    O.parallel_sample_sort(arena, h, threads)
    dt = time.perf_counter() - t0
    return {"value": h0.size / dt, "unit": "strings/s", "cores": threads, "kind": "port",
            "sample": f"one sort of the full config-{args.config} workload (n={h0.size}) by the "
                      f"C port of pS^5 (oracle/s5_oracle.c), {threads} threads, {dt:.2f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--n", type=int, default=None, help="shrink the config (same recipe)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--classifier", default="unroll", choices=["unroll", "equal"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--launch-recs", action="store_true",
                    help="add per-launch (kernel, level, strings, ms) records")
    ap.add_argument("--cfg", action="append", default=[],
                    help="SampleSortConfig override key=value (tuning), repeatable")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif dist_env()[0] > 1 or os.environ.get("S5_BENCH_DISTRIBUTED") == "1":
        run_distributed(args)  # (the env switch runs the multi-GPU path on one rank: a smoke test)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
