#!/usr/bin/env python
"""bench.py -- MIS-2 on the BASELINE.json headline workload (27-point
Laplacian 100^3, BASELINE.json configs[1]) through the C ABI of libmis2.so.

One "step" = one whole MIS-2 call (Alg. 1): init, every
Refresh Column / Decide pass, worklist compaction, loop control, output.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  Timing rules: W untimed warm-up calls; K timed
calls, each bracketed by CUDA events on the launching stream; the L2 is
flushed (a 512 MiB memset) BETWEEN timed calls, outside the event pairs;
barrier + synchronize around the timed region; max over ranks.  SM clocks and
throttle reasons are sampled with NVML during the timed region.

`--impl reference` times the CPU oracle (oracle/, serial C, 1 thread) on the
same workload: this tier has no reference implementation, the oracle is the
reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "MIS-2 ms & GTEPS on 27-pt 100^3 Laplacian, %HBM peak, at 1/2/4/8 B200"
UNIT = "GTEPS"
WORKLOAD = "MIS-2 (Alg. 1) on the 27-point Laplacian 100^3 graph (BASELINE.json configs[1])"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def alg_bytes(stats: np.ndarray, n: int) -> int:
    """Compulsory HBM bytes of one MIS-2 call for this implementation's data
    layout: T uint64, M uint32 (id field),
    colinds int32, rowptr int64, worklists int32.  stats rows = iterations:
    |wl1| |wl2| E1 E2 |N[wl1]| |N[wl2]|."""
    total = 8 * n + 4 * n  # init: T, M
    it = stats.shape[0]
    for i in range(it):
        w1, w2, e1, e2, d1, d2 = (int(x) for x in stats[i])
        w1n = int(stats[i + 1, 0]) if i + 1 < it else 0
        w2n = int(stats[i + 1, 1]) if i + 1 < it else 0
        total += 4 * e2 + 8 * d2 + (8 + 4 + 4) * w2 + 4 * w2n          # Refresh Column
        total += 4 * e1 + 4 * d1 + (8 + 4 + 8 + 8) * w1 + 4 * w1n      # Decide (+ refresh)
    total += 8 * n + 1 * n  # output: read T, write in_set
    return total


def survey_bytes(stats: np.ndarray) -> int:
    """Algorithmic bytes of one MIS-2 call by SURVEY.md §8(d).3 (the paper's
    data structures, 8-byte words, 4-byte colinds and worklist entries,
    8-byte rowptr; each byte counted once per pass, gathers once per distinct
    vertex).  stats rows = iterations: |wl1| |wl2| E1 E2 |N[wl1]| |N[wl2]|:
      B_i = 4 E2 + 8 |N[wl2]| + (4+8+8) |wl2| + 4 |wl2'|        (Refresh Column)
          + 4 E1 + 8 |N[wl1]| + (4+8+16) |wl1| + 4 |wl1'|       (Decide)"""
    total = 0
    it = stats.shape[0]
    for i in range(it):
        w1, w2, e1, e2, d1, d2 = (int(x) for x in stats[i])
        w1n = int(stats[i + 1, 0]) if i + 1 < it else 0
        w2n = int(stats[i + 1, 1]) if i + 1 < it else 0
        total += 4 * e2 + 8 * d2 + 20 * w2 + 4 * w2n
        total += 4 * e1 + 8 * d1 + 28 * w1 + 4 * w1n
    return total


def agg_bytes(iter_stats, n: int, nnz: int) -> int:
    """Algorithmic bytes of one Alg. 3 call: the two MIS-2 calls
    by §8(d).3 (the second one masked, from its own worklist statistics) plus
    one CSR pass per labelling phase (phase 1 pull, phase 2 accept / label,
    phase 3): 3 x (4 nnz + 8 (n+1) + 4 n)."""
    return survey_bytes(iter_stats[0]) + survey_bytes(iter_stats[1]) + 3 * (4 * nnz + 8 * (n + 1) + 4 * n)


def host_cpu():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


def lib_build_id() -> str:
    """sha256 (16 hex) of the libmis2.so the bench loads: stamps the ncu numbers."""
    import hashlib
    import paper_2204_02934_b200 as m
    path = os.environ.get("MIS2_LIB_PATH") or m._build.LIB
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()[:16]


NCU_METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
               "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]


def ncu_capture(config: int, peak: float, timeout: float = 240.0):
    """One ncu replay of the persistent MIS-2 kernel of this build on the bench
    graph (a subprocess after the timed region; its time is never a bench
    value): DRAM bytes per launch, DRAM GB/s and fraction of the measured
    peak, sectors per global-load request, L2 hit rate.  ncu flushes the
    caches before the replay (--cache-control all) and leaves the clocks
    alone (--clock-control none).  None when ncu is not installed."""
    import shutil
    import subprocess
    exe = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if exe is None:
        return None
    cmd = [exe, "--metrics", ",".join(NCU_METRICS), "--clock-control", "none", "--cache-control", "all",
           "-k", "regex:mis2_persistent", "-s", "2", "-c", "1", "--csv",
           sys.executable, os.path.join(ROOT, "tools", "ncu_mis2.py"), str(config)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout).stdout
    except (subprocess.SubprocessError, OSError) as e:
        return {"error": str(e)[:200]}
    import csv
    vals = {}
    for row in csv.reader(line for line in out.splitlines() if line.startswith('"')):
        if len(row) >= 15 and row[12] in NCU_METRICS:
            unit, v = row[13], float(row[14].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                     "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3}.get(unit, 1)
            vals[row[12]] = v * scale
    if "gpu__time_duration.sum" not in vals or "dram__bytes_read.sum" not in vals:
        return {"error": "ncu produced no metrics", "tail": out[-300:]}
    t = vals["gpu__time_duration.sum"]
    dram = vals["dram__bytes_read.sum"] + vals.get("dram__bytes_write.sum", 0.0)
    req = vals.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", 0.0)
    return {"kernel": "mis2k::mis2_persistent", "launch_us": t * 1e6, "dram_bytes": dram,
            "dram_gbs": dram / t / 1e9, "dram_frac": dram / t / 1e9 / peak,
            "dram_pct_of_peak_sustained": vals.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "sectors_per_request": vals.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 0.0) / req if req else None,
            "l2_hit_pct": vals.get("lts__t_sector_hit_rate.pct"), "build": lib_build_id(),
            "how": "ncu --cache-control all --clock-control none, one replay (cold caches, serialised)"}


def time_calls(fn, steps: int, flush, stream, torch):
    """median / min ms of `steps` calls, each between CUDA events on `stream`,
    the L2 flushed before each (outside the event pair)."""
    per = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        per.append(a.elapsed_time(b))
    return statistics.median(per), min(per)


def sub_records(m, torch, flush, stream, peak, steps: int, c2=None):
    """Secondary configurations, timed like the headline (CUDA events, L2
    flushed between calls): MIS-2 on configs[2..4] and Alg. 3 on configs[1],
    each with its algorithmic bytes and fraction of the HBM peak."""
    import mis2gen as G
    out = []
    for cfg, name in ((2, "C3 7-pt 300^3 MIS-2"), (3, "C4 Kronecker scale 24 MIS-2"),
                      (4, "C5 3-dof 27-pt 150^3 MIS-2")):
        g = G.config_graph(cfg)
        rp, ci = torch.from_numpy(g.rowptr).cuda(), torch.from_numpy(g.colinds).cuda()
        st = m.mis2(rp, ci, stats=True)
        ref = m.mis2(rp, ci)
        res = torch.empty(g.n, dtype=torch.uint8, device="cuda")
        sc = torch.zeros(2, dtype=torch.int64, device="cuda")
        med, mn = time_calls(lambda: m.mis2_async(rp, ci, res, sc), steps, flush, stream, torch)
        assert int(sc[0].item()) == ref.count
        b = survey_bytes(st.stats)
        out.append({"config": name, "configs_index": cfg, "n": g.n, "nnz": g.nnz, "ms": med, "ms_min": mn,
                    "gteps": g.nnz / (med / 1e3) / 1e9, "iterations": ref.iterations, "mis2_size": ref.count,
                    "alg_bytes": b, "achieved_gbs": b / (med / 1e3) / 1e9, "frac": b / (med / 1e3) / 1e9 / peak})
        if cfg == 4:  # configs[4]'s workload: repeated aggregation + coarsening down to < 1000 vertices
            levels, _, _ = m.multilevel(rp, ci, threshold=1000)
            med, mn = time_calls(lambda: m.multilevel(rp, ci, threshold=1000), min(steps, 5), flush, stream, torch)
            out.append({"config": "C5 multilevel aggregation + coarsening to < 1000 vertices", "configs_index": 4,
                        "n": g.n, "nnz": g.nnz, "ms": med, "ms_min": mn,
                        "levels": [{"n": int(a), "nnz": int(b_), "num_aggs": int(c)} for a, b_, c in levels],
                        "note": "levels x (aggregate + coarsen) through the Python API (host reads of each level's "
                                "aggregate count and coarse size between levels)"})
        del rp, ci, res
        torch.cuda.empty_cache()
    if c2 is not None:
        g, rp, ci = c2
        a = m.aggregate(rp, ci, iter_stats=True)
        med, mn = time_calls(lambda: m.aggregate(rp, ci), steps, flush, stream, torch)
        b = agg_bytes(a.iter_stats, g.n, g.nnz)
        out.append({"config": "C2 27-pt 100^3 Alg. 3 aggregation", "configs_index": 1, "n": g.n, "nnz": g.nnz,
                    "ms": med, "ms_min": mn, "gteps": g.nnz / (med / 1e3) / 1e9, "num_aggs": a.num_aggs,
                    "alg_bytes": b, "achieved_gbs": b / (med / 1e3) / 1e9, "frac": b / (med / 1e3) / 1e9 / peak,
                    "note": "includes the host reads of the aggregate count (one synchronising ABI call)"})
    return out


class ClockSampler:
    """NVML sampling of SM clock + clock-event reasons during the timed region."""

    NAMES = {
        "nvmlClocksEventReasonHwSlowdown": "hw_slowdown",
        "nvmlClocksEventReasonHwThermalSlowdown": "hw_thermal_slowdown",
        "nvmlClocksEventReasonSwThermalSlowdown": "sw_thermal_slowdown",
        "nvmlClocksEventReasonSwPowerCap": "sw_power_cap",
        "nvmlClocksEventReasonHwPowerBrakeSlowdown": "hw_power_brake_slowdown",
        "nvmlClocksEventReasonApplicationsClocksSetting": "applications_clocks_setting",
        "nvmlClocksEventReasonSyncBoost": "sync_boost",
    }

    def __init__(self, dev_index: int):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for attr, name in self.NAMES.items():
                    if r & getattr(nv, attr, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def cpu_oracle_rate(g, seconds: float):
    """Serial C oracle (1 thread) on the same graph for about `seconds`."""
    import oracle as O
    runs, t0 = 0, time.perf_counter()
    while True:
        r = O.mis2(g.rowptr, g.colinds)
        runs += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return g.nnz * runs / el / 1e9, runs, el, r


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import mis2gen as G
    import oracle as O
    g = G.config_graph(args.config)
    for _ in range(args.warmup):
        O.mis2(g.rowptr, g.colinds)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = O.mis2(g.rowptr, g.colinds)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = g.nnz / (ms / 1e3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": g.n, "nnz": g.nnz, "seed": 0, "mis2_size": r.count,
                   "iterations": r.iterations},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} full serial MIS-2 calls (oracle/oracle.c, 1 thread) on the "
                                   f"full workload"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_partitioned(args, g, rank, world, torch, m):
    """N > 1: the C2 graph 1-D row-partitioned over the ranks,
    ghost halos over NCCL each half-round; strong scaling (the graph is fixed)."""
    import torch.distributed as dist
    obj = [m.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    c = m.Comm.nccl(obj[0], world, rank)
    n = g.n
    lo, hi = n * rank // world, n * (rank + 1) // world
    t0 = time.perf_counter()
    c.set_graph(n, g.rowptr[lo:hi + 1], g.colinds)
    plan_s = time.perf_counter() - t0
    out = torch.empty(max(hi - lo, 1), dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        cnt, its = c.mis2(out)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device())
    launches = 0
    with sampler:
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            cnt, its = c.mis2(out)
            launches += int(m.lib().mis2_last_launch_count())
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    per = [a.elapsed_time(b) for a, b in evs]
    t = torch.tensor([sum(per) / len(per)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # end to end through the public API: host CSR slice in (plan + upload), mask out
    e_ms = []
    for _ in range(3):
        dist.barrier()
        a = time.perf_counter()
        c.set_graph(n, g.rowptr[lo:hi + 1], g.colinds)
        c.mis2(out)
        host = out.cpu()
        e_ms.append(1e3 * (time.perf_counter() - a))
    te = torch.tensor([sum(e_ms) / len(e_ms)], device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    c.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": g.nnz / (ms / 1e3) / 1e9, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": g.n, "nnz": g.nnz, "seed": 0, "mis2_size": cnt, "iterations": its,
                       "parallelism": f"1-D row partition over {world} GPUs, NCCL halo exchange per half-round",
                       "l2": "flushed between timed steps (512 MiB memset outside the event pairs)",
                       "plan_s": plan_s},
            "roofline": None, "cpu_baseline": None,
            "e2e": {"value": g.nnz / (float(te.item()) / 1e3) / 1e9, "unit": UNIT, "ms_per_step": float(te.item()),
                    "h2d_bytes_per_step": int(g.rowptr.nbytes + g.colinds.nbytes) // world,
                    "d2h_bytes_per_step": int(hi - lo)},
            "gpu_launches": launches, "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_ours(args):
    import torch

    import mis2gen as G
    import paper_2204_02934_b200 as m

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()

    g = G.config_graph(args.config)
    if world > 1:
        return run_partitioned(args, g, rank, world, torch, m)
    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colinds).cuda()
    out = torch.empty(g.n, dtype=torch.uint8, device="cuda")
    sc = torch.zeros(2, dtype=torch.int64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()

    # instrumented (untimed) call: worklist statistics for the byte models
    st = m.mis2(rp, ci, stats=True)
    check = m.mis2(rp, ci)
    bytes_per_call = survey_bytes(st.stats)
    bytes_impl = alg_bytes(st.stats, g.n)          # this layout (M as 4-byte id fields)

    for _ in range(args.warmup):
        flush.zero_()
        m.mis2_async(rp, ci, out, sc)
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev)
    wall0 = time.perf_counter()
    with sampler:
        for k in range(args.steps):
            flush.zero_()                          # L2 flush, outside the timed pair
            evs[k][0].record(stream)
            launches += m.mis2_async(rp, ci, out, sc)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        torch.distributed.barrier()
    per = [a.elapsed_time(b) for a, b in evs]  # ms
    ms = sum(per) / len(per)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = world * g.nnz / (ms / 1e3) / 1e9  # replicas: every rank solves the full graph
    scal = sc.cpu().tolist()
    assert scal[0] == check.count, "timed calls disagree with the checked call"

    peak, peak_src = peaks()
    achieved = bytes_per_call / (ms / 1e3) / 1e9

    # end-to-end through mis2_host(): pinned host CSR in, in_set out
    e2e = None
    if not args.no_e2e:
        rph = torch.from_numpy(g.rowptr).pin_memory()
        cih = torch.from_numpy(g.colinds).pin_memory()
        outh = torch.empty(g.n, dtype=torch.uint8).pin_memory()
        ws = m.workspace(m.OP_MIS2_HOST, g.n, g.nnz)
        for _ in range(2):
            m.mis2_host(rph, cih, outh, ws=ws)
        e_ms = []
        for _ in range(max(3, min(args.steps, 20))):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            m.mis2_host(rph, cih, outh, ws=ws)
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
        ems = sum(e_ms) / len(e_ms)
        assert int(outh.sum()) == check.count
        e2e = {"value": world * g.nnz / (ems / 1e3) / 1e9, "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": int(g.rowptr.nbytes + g.colinds.nbytes), "d2h_bytes_per_step": int(g.n + 16)}

    subs = None
    if rank == 0 and world == 1 and not args.no_subs:
        subs = sub_records(m, torch, flush, stream, peak, args.sub_steps, c2=(g, rp, ci))

    # ncu (a subprocess, after every timed region): DRAM traffic of one
    # launch of this build's kernel, sectors per request
    ncu = None
    if rank == 0 and world == 1 and not args.no_ncu:
        ncu = ncu_capture(args.config, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, runs, el, _ = cpu_oracle_rate(g, args.cpu_seconds)
        model, nproc = host_cpu()
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{runs} full serial MIS-2 calls of the oracle (oracle/oracle.c, 1 thread) on the same "
                         f"graph, {el:.1f} s", "cpu_model": model, "nproc": nproc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": g.n, "nnz": g.nnz, "seed": 0, "generator":
                       "mis2gen.laplace3d_27pt(100)", "mis2_size": check.count, "iterations": check.iterations,
                       "l2": "flushed between timed steps (512 MiB memset outside the event pairs)",
                       "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
                       "ms_min": min(per), "ms_median": statistics.median(per), "wall_s": wall},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": ncu.get("dram_bytes") if isinstance(ncu, dict) else None,
                         "kernel": "mis2k::mis2_persistent",
                         "alg_bytes_per_launch": bytes_per_call, "alg_bytes_model": "SURVEY.md 8(d).3",
                         "alg_bytes_impl_layout": bytes_impl, "peak_source": peak_src, "ncu": ncu},
            "configs": subs,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1, help="BASELINE.json configs index (bench workload: 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-ncu", action="store_true", help="skip the ncu DRAM-traffic capture")
    ap.add_argument("--no-subs", action="store_true", help="skip the secondary configuration records")
    ap.add_argument("--sub-steps", type=int, default=5)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
