"""Benchmark: S^5 string sample sort + LCP on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one sort (with LCP output) of one BASELINE configuration's synthetic
strings.  Default workload: config 2 (n = 2^25 random strings, the
configuration BASELINE.json's metric is quoted on that fits one GPU).

Our arm (default): inputs resident in HBM; before every step the unsorted
handle array is restored and a 256 MiB buffer (> the 126 MB L2) is written
(untimed); each step is timed with CUDA events on the sorting stream; the max
over ranks is taken.  Extra keys: ``e2e`` (public API with host numpy
buffers: H2D handles, sort, D2H handles + LCP), ``roofline`` (dominant
kernel, per-kernel CUDA events in a separate profiled pass), ``roofline_sort``
(whole sort, SURVEY.md 8(d) B_alg), ``per_config`` (configs 3/4/5 measured
the same way, default run only), and ``cpu_baseline`` (the C port of the
reference's parallel S^5, oracle/, at 1 worker and at every host thread).

``--gpus N`` (N > 1): one global sort of the config's n strings across N
ranks (sample-sort partitioning, NCCL all-to-all of u32 offsets, local S^5
per rank; strong scaling).  Without torchrun's environment the script
re-launches itself under ``torch.distributed.run`` with N processes.

``--impl reference``: the reference's CPU algorithm (C port of pS^5,
oracle/s5_oracle.c, all host threads) on the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
L2_NOTE = ("GPU arm: unsorted handles restored and a 256 MiB buffer (> 126 MB L2) written "
           "before every step, both untimed")


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


def common_config(args, config: int, n: int, arena_bytes: int, world: int) -> dict:
    """The ``config`` dict both arms print (identical keys and values)."""
    from paper_1305_1157_b200 import datasets
    par = "single GPU" if world == 1 else (
        f"dp{world}: sample-sort partition, NCCL all-to-all of u32 offsets, local S^5 per "
        f"rank (strong scaling: n fixed)")
    return {"workload": f"config{config}: {datasets.DESCRIPTION[config]}", "n": int(n),
            "arena_bytes": int(arena_bytes), "parallelism": par, "l2": L2_NOTE}


def host_info() -> dict:
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = None
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": aff}


def cpu_baseline(arena, h0, args) -> dict:
    """The reference's pS^5 (C port, oracle/) at workers=1 and workers=all on
    the full workload; value = all threads."""
    import oracle as O
    threads = O.max_threads()
    res = {}
    for w in (1, threads):
        h = h0.copy()
        t0 = time.perf_counter()
        O.parallel_sample_sort(arena, h, w)
        res[w] = time.perf_counter() - t0
    dt = res[threads]
    return {"value": h0.size / dt, "unit": "strings/s", "cores": threads, "kind": "port",
            "sample": f"one sort of the full config-{args.config} workload (n={h0.size}) by the C "
                      f"port of pS^5 (oracle/s5_oracle.c) at {threads} threads ({dt:.2f} s) and at "
                      f"1 thread ({res[1]:.2f} s)",
            "workers_1": {"value": h0.size / res[1], "seconds": res[1]},
            "workers_all": {"value": h0.size / dt, "seconds": dt, "workers": threads},
            **host_info()}


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
    h = h0.copy()
    t0 = time.perf_counter()
    O.parallel_sample_sort(arena, h, 1)
    t1 = time.perf_counter() - t0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "strings/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.gpus == 1 else "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": common_config(args, args.config, n, arena.data.size, args.gpus),
        "cpu_baseline": {"value": value, "unit": "strings/s", "cores": threads, "kind": "port",
                         "sample": f"full config-{args.config} workload per step (n={n}), C port "
                                   f"of pS^5 (oracle/s5_oracle.c), {threads} threads",
                         "workers_1": {"value": n / t1, "seconds": t1}, **host_info()},
        "e2e": {"value": value, "unit": "strings/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "d_chars_per_s": None,
    }
    D = datasets.EXPECTED.get(args.config, (0, 0, 0))[2] if args.n is None else None
    if D:
        line["d_chars_per_s"] = D * args.steps / total
    print(json.dumps(line), flush=True)


def make_cfg(args):
    from paper_1305_1157_b200.samplesort import SampleSortConfig
    kw = {"classifier": args.classifier}
    for item in args.cfg:
        k, _, v = item.partition("=")
        kw[k] = int(v) if v.lstrip("-").isdigit() else v
    return SampleSortConfig(**kw)


def one_step_prof(arena, d_h, d_h0, d_lcp, cfg, stats, l2_flush, extra_flags=0):
    """One sort with per-launch CUDA events (cfg flags bit1)."""
    import ctypes as C

    import torch
    from paper_1305_1157_b200 import _lib
    from paper_1305_1157_b200.samplesort import _workspace
    d_h.copy_(d_h0)
    l2_flush.zero_()
    c = cfg.to_c()
    c.flags |= 2 | extra_flags
    n = d_h.numel()
    need = int(_lib.lib().s5_workspace_bytes(n, arena.data.size, C.byref(c)))
    ws = _workspace(need, d_h.device)
    rc = _lib.lib().s5_sort(arena.device(d_h.device).data_ptr(), arena.data.size, d_h.data_ptr(),
                            n, 0, d_lcp.data_ptr(), C.byref(c), ws.data_ptr(), ws.numel(),
                            _lib.current_stream_ptr(), C.byref(stats))
    _lib.check(rc, "s5_sort (profiled)")
    torch.cuda.synchronize()


def kernel_roofline(prof_stats: list, config: int, peak: float, peak_src: str) -> tuple:
    """Per-kernel mean device times of the profiled sorts and the dominant
    kernel's roofline: 16 B (8-B pointer read + write) per
    string the launch moves, over its mean launch time."""
    kern = {}
    for ps in prof_stats:
        for name, rec in ps["kernels"].items():
            k = kern.setdefault(name, {"ms": 0.0, "launches": 0, "strings": 0})
            k["ms"] += rec["ms"] / len(prof_stats)
            k["launches"] += rec["launches"] / len(prof_stats)
            k["strings"] += rec["strings"] / len(prof_stats)
    dom_name, dom_rec = max(kern.items(), key=lambda kv: kv[1]["ms"]) if kern else \
        ("none", {"ms": 0, "launches": 1, "strings": 0})
    launches = max(dom_rec["launches"], 1)
    per_launch_bytes = 16.0 * dom_rec["strings"] / launches
    per_launch_ms = dom_rec["ms"] / launches
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"config{config}", {}).get(dom_name)
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak if peak else None, "traffic": traffic,
            "peak_source": peak_src, "bytes_per_launch": per_launch_bytes,
            "ms_per_launch": per_launch_ms,
            "algorithmic_bytes": "16 B per string moved by the launch "
                                 "(8-B pointer read + write, SURVEY 8(d))"}
    return kern, roof


def measure_device(arena, h0, cfg, steps, warmup, dev, config, clocks=None, world=1):
    """Device-resident sorts timed with CUDA events, then profiled sorts for
    the per-kernel times.  Returns the measured fields."""
    import torch
    from paper_1305_1157_b200 import _lib
    from paper_1305_1157_b200.samplesort import gpu_sort
    from paper_1305_1157_b200.strings import distinguishing_prefix, first_unsorted
    import torch.distributed as dist

    n = h0.size
    arena.device(dev)
    d_h0 = torch.from_numpy(h0).to(dev)
    d_h = torch.empty_like(d_h0)
    d_lcp = torch.empty(n - 1, dtype=torch.int64, device=dev)
    l2_flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # 256 MiB > L2
    stream = torch.cuda.current_stream()

    def one_step(stats=None):
        d_h.copy_(d_h0)
        l2_flush.zero_()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        gpu_sort(arena, d_h, 0, cfg, d_lcp, stats)
        ev1.record(stream)
        return ev0, ev1

    for _ in range(warmup):
        one_step()
    torch.cuda.synchronize()
    if clocks is not None:
        clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    events = []
    stats = _lib.S5Stats()
    t_wall = time.perf_counter()
    for _ in range(steps):
        events.append(one_step(stats))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks is not None else None
    step_ms = [a.elapsed_time(b) for a, b in events]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / steps
    st = stats.as_dict()
    assert first_unsorted(arena, d_h) == -1, "bench output not sorted"
    D = int(distinguishing_prefix(arena, d_h, d_lcp))
    prof = []
    for _ in range(max(1, min(steps, 3))):
        ps = _lib.S5Stats()
        one_step_prof(arena, d_h, d_h0, d_lcp, cfg, ps, l2_flush)
        prof.append(ps.as_dict())
    peak, peak_src = hbm_peak()
    kern, roof = kernel_roofline(prof, config, peak, peak_src)
    n_p = st["n_per_pass"]
    B_alg = 16 * sum(n_p) + D  # 16 B per string per S^5 level / base-case pass
    del l2_flush, d_h0
    return {
        "ms_per_step": ms, "step_ms": [round(x, 4) for x in step_ms], "wall": wall,
        "clocks": clk, "D": D, "stats": st, "launches_per_step": int(stats.launches),
        "kern": kern, "roofline": roof, "prof_last": prof[-1],
        "roofline_sort": {"B_alg": B_alg, "floor_bytes": 16 * n + D,
                          "achieved_gbs": B_alg / (ms * 1e-3) / 1e9,
                          "frac": B_alg / (ms * 1e-3) / 1e9 / peak,
                          "floor_frac": (16 * n + D) / (ms * 1e-3) / 1e9 / peak},
        "d_h": d_h, "d_lcp": d_lcp,
    }


def measure_e2e(arena, h0, cfg, steps, warmup):
    """The public API with numpy host buffers: H2D, sort, D2H, widening."""
    import torch
    from paper_1305_1157_b200 import samplesort as _ss
    n = h0.size
    e2e_times = []
    h_host = np.empty_like(h0)
    lcp_host = np.empty(n - 1, np.int64)
    for i in range(warmup + steps):
        np.copyto(h_host, h0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _ss.parallel_sample_sort(arena, h_host, cfg=cfg, lcp_out=lcp_host)
        dt = time.perf_counter() - t0
        if i >= warmup:
            e2e_times.append(dt)
    return sum(e2e_times) / len(e2e_times), dict(_ss.LAST_HOST_MS)


def per_config_block(args, cfg, dev):
    """Configs 3/4/5 measured like the headline (device-resident, L2 flushed,
    CUDA events; dominant kernel roofline with its ncu traffic)."""
    import torch
    from paper_1305_1157_b200.samplesort import release_workspace
    out = {}
    for c in (2, 3, 4, 5):
        if c == args.config:
            continue
        arena, h0, gen_s = workload(c, None)
        m = measure_device(arena, h0, cfg, max(3, min(args.steps, 5)), 3, dev, c)
        n = h0.size
        out[f"config{c}"] = {
            "n": int(n), "arena_bytes": int(arena.data.size), "D": m["D"],
            "ms_per_step": m["ms_per_step"], "strings_per_s": n / (m["ms_per_step"] * 1e-3),
            "d_chars_per_s": m["D"] / (m["ms_per_step"] * 1e-3),
            "levels": m["stats"]["levels"], "n_per_pass": m["stats"]["n_per_pass"],
            "roofline_sort": m["roofline_sort"], "roofline": m["roofline"],
            "kernels_ms_per_step": {k: round(v["ms"], 4) for k, v in sorted(m["kern"].items())},
            "step_ms": m["step_ms"], "generate_s": round(gen_s, 1)}
        del m, arena, h0
        release_workspace()
        torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch

    world, rank, local = dist_env()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    arena, h0, gen_s = workload(args.config, args.n)
    n = h0.size
    cfg = make_cfg(args)
    t_up = time.perf_counter()
    arena.device(dev)
    torch.cuda.synchronize()
    arena_upload_s = time.perf_counter() - t_up
    m = measure_device(arena, h0, cfg, args.steps, args.warmup, dev, args.config,
                       clocks=ClockSampler(local))
    ms_per_step = m["ms_per_step"]
    st = m["stats"]
    D = m["D"]
    e2e_s, e2e_phases = measure_e2e(arena, h0, cfg, args.steps, args.warmup)
    value = n / (ms_per_step * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "strings/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": common_config(args, args.config, n, arena.data.size, 1),
        "settings": {"classifier": args.classifier, "overrides": args.cfg, "D": D},
        "d_chars_per_s": D / (ms_per_step * 1e-3),
        "roofline": m["roofline"],
        "roofline_sort": m["roofline_sort"],
        "n_per_pass": st["n_per_pass"],
        "kernels_ms_per_step": {k: round(v["ms"], 4) for k, v in sorted(m["kern"].items())},
        "kernels_strings_per_step": {k: int(v["strings"]) for k, v in sorted(m["kern"].items())},
        "launch_recs": m["prof_last"].get("launch_recs", []) if args.launch_recs else None,
        "e2e": {"value": n / e2e_s, "unit": "strings/s",
                "h2d_bytes_per_step": int(e2e_phases.get("h2d_bytes", 8 * n)),
                "d2h_bytes_per_step": int(e2e_phases.get("d2h_bytes", 16 * n - 8)),
                "ms_per_step": 1e3 * e2e_s,
                "note": "parallel_sample_sort(numpy int64 handles, lcp_out=numpy int64): "
                        "handles cross PCIe as u32 both ways, LCPs in the narrowest width "
                        "holding their maximum; H2D + sort + D2H + host widening",
                "phases_ms": e2e_phases},
        "arena_upload_s": arena_upload_s,
        "generate_s": round(gen_s, 1),
        "gpu_launches": m["launches_per_step"] * args.steps,
        "clocks": m["clocks"],
        "wall_s_timed_region": m["wall"],
        "step_ms": m["step_ms"],
        "levels": st["levels"],
        "tiers_per_level": {t: st[f"{t}_elems"] for t in ("wide", "narrow", "local", "small")},
        "key_fetches": st["key_fetches"], "boundary_lcps": st["boundary_lcps"],
    }
    del m
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(arena, h0, args)
    if args.per_config and args.n is None:
        del arena, h0
        from paper_1305_1157_b200.samplesort import release_workspace
        release_workspace()
        torch.cuda.empty_cache()
        line["per_config"] = per_config_block(args, cfg, dev)
    print(json.dumps(line), flush=True)


def run_distributed(args):
    """N > 1 (torchrun): one global sort of the config's n strings across the
    ranks -- sample-sort partitioning + NCCL all-to-all + local S^5
    (paper_1305_1157_b200.distributed).  Strong scaling: n is fixed."""
    import torch
    import torch.distributed as dist

    from paper_1305_1157_b200 import _lib, datasets
    from paper_1305_1157_b200.distributed import GpuBackend, distributed_sample_sort
    from paper_1305_1157_b200.strings import first_unsorted

    if "RANK" not in os.environ:  # one-rank smoke run without torchrun
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
    world, rank, local = dist_env()
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but {torch.cuda.device_count()} GPUs")
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
    st = be.last_stats.as_dict() if getattr(be, "last_stats", None) is not None else \
        {"n_per_pass": []}
    t = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    ok = torch.tensor([1 if first_unsorted(arena, res.handles) == -1 else 0], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    # SURVEY 8(d) B_alg over all ranks: the partition pass (every local
    # string) + every level of every rank's local sort, 16 B per string, + D
    moved = torch.tensor([float((hi - lo) + sum(st["n_per_pass"]))], dtype=torch.float64,
                         device=dev)
    dist.all_reduce(moved)
    # the dominant kernel of this rank's local sort (profiled re-run)
    peak, peak_src = hbm_peak()
    ps = _lib.S5Stats()
    be.keep_input = True  # one more exchange keeps this rank's unsorted received handles
    distributed_sample_sort(arena, shard.clone(), backend=be)
    be.keep_input = False
    recv_h0 = be.last_input
    work = torch.empty_like(recv_h0)
    d_lcp = torch.empty(max(recv_h0.numel() - 1, 1), dtype=torch.int64, device=dev)
    if recv_h0.numel() > 1:
        one_step_prof(arena, work, recv_h0, d_lcp, cfg, ps, l2_flush)
    kern, roof = kernel_roofline([ps.as_dict()], args.config, peak, peak_src)
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
        be.download(r.handles, r.lcp, out_hb, out_lb)
        if it:
            e2e.append(time.perf_counter() - t0)
    te = torch.tensor([sum(e2e) / len(e2e)], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(arena, h0, args)
    dist.barrier()
    if rank == 0:
        D = datasets.EXPECTED.get(args.config, (0, 0, 0))[2] if args.n is None else None
        B_alg = 16 * float(moved.item()) + (D or 0)
        line = {
            "metric": METRIC, "value": n / (ms_per_step * 1e-3), "unit": "strings/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": common_config(args, args.config, n, arena.data.size, world),
            "settings": {"classifier": args.classifier, "overrides": args.cfg, "D": D},
            "d_chars_per_s": D / (ms_per_step * 1e-3) if D else None,
            "roofline": roof,
            "roofline_sort": {"B_alg": B_alg, "floor_bytes": 16 * n + (D or 0),
                              "achieved_gbs": B_alg / (ms_per_step * 1e-3) / 1e9,
                              "frac": B_alg / (ms_per_step * 1e-3) / 1e9 / (world * peak),
                              "note": "B_alg / (t * G * peak); passes: partition + local levels"},
            "e2e": {"value": n / float(te.item()), "unit": "strings/s",
                    "h2d_bytes_per_step": int(4 * n), "d2h_bytes_per_step": int(4 * n + (n - 1)),
                    "ms_per_step": 1e3 * float(te.item()),
                    "note": "host shards in, host slices + LCP out, all ranks; u32 handles and "
                            "narrow LCPs over PCIe (s5_upload_handles / s5_download)"},
            "sorted_ok": bool(ok.item()), "slice_sizes": res.counts, "clocks": clk,
            "gpu_launches": launches,
            "kernels_ms_rank0_local_sort": {k: round(v["ms"], 4) for k, v in sorted(kern.items())},
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args) -> int:
    """``--gpus N`` without torchrun's environment: run N ranks of this
    script under torch.distributed.run (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
    ap.add_argument("--per-config", dest="per_config", action="store_true", default=None,
                    help="add configs 3/4/5 (default: on for the default config-2 run)")
    ap.add_argument("--no-per-config", dest="per_config", action="store_false")
    ap.add_argument("--launch-recs", action="store_true",
                    help="add per-launch (kernel, level, strings, ms) records")
    ap.add_argument("--cfg", action="append", default=[],
                    help="SampleSortConfig override key=value (tuning), repeatable")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.per_config is None:
        args.per_config = args.config == 2 and args.n is None and not args.cfg
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    elif dist_env()[0] > 1 or os.environ.get("S5_BENCH_DISTRIBUTED") == "1":
        run_distributed(args)  # (the env switch runs the multi-GPU path on one rank: a smoke test)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
