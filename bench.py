#!/usr/bin/env python
"""Benchmark: GPU S^5 string sort with LCP array (BASELINE.json metric).

One "step" = one full sort (handles + LCP array) of the workload, inputs
resident in HBM.  Default workload: BASELINE.json configs[4] (C5, 2^28
unique strings of 32-200 characters, 31.4 GB -- the configuration the metric
is quoted on "at 1/2/4/8 B200", and the largest that fits one GPU), generated
on the device by the counter-based generator (csrc/s5g_gen.cu; the host copy
for the e2e and CPU legs is read back once).  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5_nodup]
  python bench.py --impl reference ...   # CPU S^5 (oracle port), all host cores

The arena (31.4 GB at C5, 1.69 GB at C2) is larger than the 126 MB L2, so no
explicit L2 flush is needed between timed steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "strings/sec (+ D-bytes/sec) of S^5 sort with LCP array"
UNIT = "strings/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback


TRAFFIC = ROOT / "profiles" / "r01i_traffic.json"  # replaced per config in main()


def traffic_file(config: str):
    """The committed ncu per-kernel traffic of this workload (full size)."""
    p = ROOT / "profiles" / f"r02_{config}_traffic.json"
    return p if p.exists() else (ROOT / "profiles" / "r01i_traffic.json" if config == "c2_dna" else None)
PASS_BYTES = 24  # algorithmic bytes per string per distribution pass


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full
    capture (profiles/r01i_traffic.json), or None."""
    try:
        d = json.loads(TRAFFIC.read_text())["kernels"]
    except Exception:
        return None
    k = d.get(kernel)
    if k is None:  # ncu names templates with their argument values
        k = next((v for n, v in d.items() if n.split("<")[0] == kernel.split("<")[0]), None)
    return k["dram_bytes_per_launch"] if k else None


def ncu_warp_inst(kernel: str):
    """warp instructions per launch of `kernel` from the committed ncu
    capture, or None."""
    try:
        d = json.loads(TRAFFIC.read_text())["kernels"]
    except Exception:
        return None
    k = d.get(kernel)
    if k is None and "<" not in kernel:  # bench names omit ncu's template arguments
        k = next((v for n, v in d.items() if n.split("<")[0] == kernel), None)
    return k.get("warp_inst_per_launch") if k else None


def ncu_share(kernel: str):
    """The kernel's share of the summed launch durations in the committed
    full-size ncu launch list (serialized, cold caches), or None."""
    try:
        d = json.loads(TRAFFIC.read_text())["kernels"]
    except Exception:
        return None
    tot = sum(v["ms"] for v in d.values())
    ms = sum(v["ms"] for n, v in d.items()
             if n == kernel or ("<" not in kernel and n.split("<")[0] == kernel))
    return ms / tot if tot > 0 and ms > 0 else None


def dominant_kernel(kernels: dict) -> str:
    """The kernel with the largest summed live time.  The profiled pass runs
    every kernel on one stream (s5g_profile_enable(2)), so a launch's event
    time is its own and the per-kernel sums add up to the step."""
    return max(kernels, key=lambda k: kernels[k]["ms"])


def issue_roofline(kernel: str, avg_ms: float, sm_mhz: float, sms: int):
    """Instruction-issue roofline of an integer / latency-bound kernel: warp
    instructions per launch (ncu) over the live launch time, against
    SMs x 4 schedulers x 1 warp-instruction per clock."""
    wi = ncu_warp_inst(kernel)
    if not wi or avg_ms <= 0 or not sm_mhz:
        return None
    ach = wi / (avg_ms / 1000.0) / 1e9
    peak = sms * 4 * sm_mhz * 1e6 / 1e9
    return {"bound": "issue", "achieved": ach, "peak": peak, "unit": "G warp-inst/s",
            "frac": ach / peak, "warp_inst_per_launch": wi,
            "source": "smsp__inst_executed.sum from the committed ncu capture"}


def hbm_peak():
    try:
        d = json.loads(PEAKS.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def b_alg(n: int, D: int) -> int:
    """Algorithmic bytes of a sort: 24*(floor(D/8) + n) + 8n."""
    return 24 * (D // 8 + n) + 8 * n


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        busy = [s for s in sm if mx and s > 0.3 * max(mx)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def cpu_reference(buf, hnd, sample_n: int, reps: int, threads: int):
    """The reference's CPU S^5 (oracle port of parallel_s5, parallel.py:468-492)
    on a bounded prefix sample.  Returns (strings/s, seconds list)."""
    import oracle

    if sample_n < len(hnd):
        end = int(hnd[sample_n])  # packed configs: the prefix is a self-contained set
        sbuf, shnd = buf[:end], hnd[:sample_n]
    else:
        sbuf, shnd = buf, hnd
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.parallel_s5(sbuf, shnd, p=threads, want_lcps=True)
        times.append(time.perf_counter() - t0)
    return len(shnd) / statistics.median(times), times


def config_n(name: str, scale: float) -> int:
    base = {"c1_random": 1_000_000, "c2_dna": 1 << 24, "c3_urls": 1 << 23,
            "c4_suffixes": 1 << 24, "c5_nodup": 1 << 28}[name]
    return int(base * scale)


def load_config(name: str, scale: float, pinned: bool = False):
    """Host copy (buffer, handles) of the workload; C5 is generated on all
    host cores (optionally straight into pinned memory)."""
    from paper_1403_2056_b200 import corpora

    if name == "c5_nodup":
        n = config_n(name, scale)
        out = None
        if pinned:
            import torch

            out = torch.empty(corpora.nodup_bytes(n), dtype=torch.uint8,
                              pin_memory=True).numpy()
        return corpora.gen_nodup(n, 4, out=out)
    return corpora.CONFIGS[name](scale)


def load_device(name: str, scale: float, dev):
    """(DeviceStrings, host buffer, host handles, buffer pinned?): C5 is generated in HBM
    and read back once into pinned host memory (the e2e and CPU legs' copy);
    the other configs are generated on the host and uploaded."""
    import torch

    from paper_1403_2056_b200 import corpora
    from paper_1403_2056_b200 import device as DV

    if name == "c5_nodup":
        arena, alen, h = corpora.gen_nodup_device(config_n(name, scale), 4, dev)
        buf = torch.empty(alen, dtype=torch.uint8, pin_memory=True)
        buf.copy_(arena[:alen])
        hnd = h.cpu().numpy()
        return DV.DeviceStrings(arena, alen, h), buf.numpy(), hnd, True
    buf, hnd = corpora.CONFIGS[name](scale)
    return DV.upload(buf, hnd, dev), buf, hnd, False


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    buf, hnd = load_config(args.config, args.scale)
    n = len(hnd)
    sample = min(n, args.cpu_sample) if args.cpu_sample > 0 else n
    # the CPU needs no clock / cache warm-up beyond one pass (a full C5 sort
    # takes ~10 s on 16 threads): min(W, 1) untimed passes keep the run at a
    # few minutes
    cpu_warm = min(args.warmup, 1)
    for _ in range(cpu_warm):
        cpu_reference(buf, hnd, sample, 1, threads)
    rate, times = cpu_reference(buf, hnd, sample, args.steps, threads)
    total = sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": args.config, "n": n, "scale": args.scale,
                   "sample_strings": sample, "parallelism": f"cpu{threads}",
                   "cpu_warmup_passes": cpu_warm},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": (f"all {n} strings" if sample == n else
                                    f"first {sample} strings") + f" of {args.config} "
                                   f"(oracle/s5_oracle.c parallel_s5, {threads} OpenMP threads, "
                                   f"{cpu_model()})"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def dist_stats_device(ds, out_h, lcps):
    """(D, L) of the sorted set on the GPU (s5g_dist_stats, strset.py:290-309)."""
    from paper_1403_2056_b200 import device as DV

    return DV.dist_stats(lcps)


def load_slice(name: str, scale: float, lo: int, hi: int, dev):
    """Strings [lo, hi) of the workload as one rank's shard: (DeviceStrings,
    host buffer, host handles relative to the slice).  C5 is generated
    straight into HBM from its counter-based definition (the slice only);
    the other configs are generated on the host and cut."""
    import torch

    from paper_1403_2056_b200 import corpora
    from paper_1403_2056_b200 import device as DV

    if name == "c5_nodup":
        arena, alen, h = corpora.gen_nodup_device(hi - lo, 4, dev, n0=lo)
        buf = torch.empty(max(alen, 1), dtype=torch.uint8, pin_memory=True)[:alen]
        buf.copy_(arena[:alen])
        return DV.DeviceStrings(arena, alen, h), buf.numpy(), h.cpu().numpy()
    buf, hnd = corpora.CONFIGS[name](scale)
    end = int(hnd[hi]) if hi < len(hnd) else len(buf)
    b0 = int(hnd[lo]) if lo < len(hnd) else end
    sb, sh = buf[b0:end], hnd[lo:hi] - b0
    return DV.upload(sb, sh, dev), sb, sh


def run_dist(args):
    """N > 1 (torchrun): STRONG scaling of one global corpus -- rank r owns
    the contiguous slice [r n / N, (r+1) n / N) of the workload (C5: generated
    on its own GPU); one step is the whole multi-GPU sort (sample, partition,
    NCCL all-to-all of bytes + global indices over NVLink, local S^5,
    boundary LCP), timed on the device and reported as the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1403_2056_b200 import _lib
    from paper_1403_2056_b200 import device as DV
    from paper_1403_2056_b200.dist import GpuBackend, Shard, distributed_merge_sort, distributed_sort

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    n_total = config_n(args.config, args.scale)
    lo, hi = rank * n_total // world, (rank + 1) * n_total // world
    ds, hbuf, hhnd = load_slice(args.config, args.scale, lo, hi, dev)
    be = GpuBackend(dev)
    xstats: dict = {}

    def step(shard):
        if args.strategy == "merge":  # partitioned_merge_sort across ranks
            return distributed_merge_sort(shard, be)
        return distributed_sort(shard, be, want_lcps=True, stats=xstats)

    shard = Shard(ds, hhnd, lo)
    for _ in range(args.warmup):
        res = step(shard)
    torch.cuda.synchronize()
    # D of the whole job from the ranks' exact LCP arrays (strset.py:290-309)
    D_loc, L_loc = DV.dist_stats(res.lcps.clamp(min=0)) if res.lcps is not None and res.lcps.numel() else (0, 0)
    red = torch.tensor([D_loc, L_loc, xstats.get("sent_bytes", 0)], dtype=torch.int64, device=dev)
    dist.all_reduce(red)
    D_all, L_all, sent_all = (int(x) for x in red.tolist())
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            res = step(shard)
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_step = float(ms.item()) / args.steps
    launches = _lib.launch_count() - l0
    peak, peak_src = hbm_peak()
    t = ms_step / 1000.0
    sort_gbs = b_alg(n_total, D_all) / t / 1e9

    # end to end through the public API on host buffers: every step uploads
    # each rank's slice from pinned memory, sorts across the ranks and reads
    # back the sorted global indices and LCPs
    e2e = None
    if not args.no_e2e:
        pin_h = torch.empty(max(len(hhnd), 1), dtype=torch.int64, pin_memory=True)[:len(hhnd)]
        pin_h.numpy()[:] = hhnd
        ts = []
        for it in range(max(1, min(args.steps, 3)) + 1):
            dist.barrier()
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            dsh = DV.upload(hbuf, pin_h.numpy(), dev)
            r2 = step(Shard(dsh, hhnd, lo))
            g_host, l_host = r2.gidx.cpu(), r2.lcps.cpu()
            s1.record()
            torch.cuda.synchronize()
            tt = torch.tensor([s0.elapsed_time(s1)], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            if it:
                ts.append(float(tt.item()))
            del dsh, r2
        e2e = {"value": n_total / (statistics.median(ts) / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(len(hbuf) + 8 * len(hhnd)),
               "d2h_bytes_per_step": int(16 * res.gidx.numel()),
               "ms_per_step": statistics.median(ts), "per": "rank 0's bytes; time = max over ranks",
               "call": "dist.distributed_sort on each rank's uploaded shard (NCCL)"}
    cpu_line = None
    if rank == 0 and not args.no_cpu_baseline:
        # the same CPU leg as at N = 1 (the oracle port on all host cores)
        threads = os.cpu_count() or 1
        buf_all, hnd_all = load_config(args.config, args.scale)
        rate, times = cpu_reference(buf_all, hnd_all, len(hnd_all), 1, threads)
        cpu_line = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                    "sample": f"all {len(hnd_all)} strings of {args.config}, 1 rep, {times[0]:.2f} s "
                              f"(oracle/s5_oracle.c parallel_s5, {threads} OpenMP threads)"}
        del buf_all, hnd_all
    line = {
        "metric": METRIC, "value": n_total / t, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": args.config, "n": n_total, "n_per_rank": hi - lo, "scale": args.scale,
                   "D": D_all, "L": L_all,
                   "parallelism": f"dp{world} (" + ("local S^5 + sampled cuts + NCCL all-to-all of "
                                                     "sorted pieces + K-way LCP merge"
                                                     if args.strategy == "merge" else
                                                     "sample-sort partition + NCCL all-to-all") + ")",
                   "l2": "inputs larger than L2 (arena > 126 MB), no flush"},
        "roofline": {"bound": "hbm", "kernel": "whole multi-GPU sort",
                     "achieved": sort_gbs / world, "peak": peak, "unit": "GB/s per GPU",
                     "frac": sort_gbs / world / peak, "traffic": None, "peak_source": peak_src,
                     "bytes_model": "B_alg = 24 (floor(D/8) + n) + 8 n over all ranks (SURVEY 8d)"},
        "nvlink": {"sent_bytes_per_step": sent_all, "peak_gbs_per_gpu": 900.0,
                   "frac": (sent_all / world / 900e9) / t if t > 0 else None,
                   "model": "X = bytes each rank sends to the others (strings + 24 B/string); "
                            "frac = X / (N * 900 GB/s) / step time"},
        "gpu_launches": int(launches), "clocks": clk.summary(), "cpu_baseline": cpu_line,
        "e2e": e2e,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1403_2056_b200 import _lib
    from paper_1403_2056_b200 import device as DV

    rank, world, local = dist_env()
    _lib.lib().s5g_set_l2_fetch_granularity(args.l2_fetch)
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", torch.cuda.current_device())
    ds, buf, hnd, pinned = load_device(args.config, args.scale, dev)
    n = len(hnd)
    threads = os.cpu_count() or 1

    cpu_line = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(n, args.cpu_sample) if args.cpu_sample > 0 else n
        cpu_reference(buf, hnd, sample, 1, threads)  # one untimed pass, as the reference arm
        rate, times = cpu_reference(buf, hnd, sample, 1, threads)
        cpu_line = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                    "sample": (f"all {n} strings" if sample == n else f"first {sample} strings")
                              + f" of {args.config}, 1 rep after 1 untimed, "
                              f"{times[0]:.2f} s (oracle/s5_oracle.c parallel_s5, "
                              f"{threads} OpenMP threads, {cpu_model()})"}

    ws = torch.empty(DV.workspace_bytes(n, 1 << 20), dtype=torch.uint8, device=dev)
    out = (torch.empty(n, dtype=torch.int64, device=dev),
           torch.empty(n, dtype=torch.int64, device=dev))

    def step():
        return DV.sort(ds, want_lcps=True, out=out, workspace=ws)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    D, L = dist_stats_device(ds, out[0], out[1])

    stream = torch.cuda.current_stream()
    l0 = _lib.launch_count()
    with ClockSampler(dev.index) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = _lib.launch_count() - l0
    ms = e0.elapsed_time(e1)
    # per-kernel CUDA events in a second pass of the same steps: the event
    # records and their read-back between sorts would otherwise add ~10 % to
    # the timed region above
    _lib.profile(enable=True, reset=True, serial=True)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    prof = _lib.profile(enable=False)
    profiled_ms = p0.elapsed_time(p1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    total_strings = n * world
    value = total_strings / (ms_step / 1000.0)

    # end to end through the reference-facing call: s5_sort(sset, want_lcps=True)
    # on a string set whose buffer and handles sit in pinned host memory; the
    # library copies them in (s5g_sort_host), sorts, and copies the handles
    # and LCPs back into new host arrays -- all inside the timed region
    e2e = None
    if not args.no_e2e:
        from paper_1403_2056_b200 import ssss
        from paper_1403_2056_b200.strset import StringSet

        ref_h = out[0].cpu().numpy()
        del ds, ws, out
        torch.cuda.empty_cache()
        if not pinned:
            pin_buf = torch.empty(len(buf), dtype=torch.uint8, pin_memory=True)
            pin_buf.numpy()[:] = buf
            buf = pin_buf.numpy()
        pin_h = torch.empty(n, dtype=torch.int64, pin_memory=True)
        pin_h.numpy()[:] = hnd
        sset = StringSet(buf, pin_h.numpy())
        res = ssss.s5_sort(sset, want_lcps=True)  # warm-up (device pool, staging ring)
        ts = []
        for _ in range(max(1, min(args.steps, 3))):
            t0 = time.perf_counter()
            res = ssss.s5_sort(sset, want_lcps=True)
            ts.append(time.perf_counter() - t0)
        assert np.array_equal(res.set.handles, ref_h)
        del res
        _lib.lib().s5g_release_cached_memory()
        e2e = {"value": n / statistics.median(ts), "unit": UNIT,
               "h2d_bytes_per_step": int(len(buf) + 8 * n),
               "d2h_bytes_per_step": int(16 * n), "ms_per_step": 1000 * statistics.median(ts),
               "call": "paper_1403_2056_b200.s5_sort(sset, want_lcps=True) -> s5g_sort_host, "
                       "buffer + handles in pinned host memory, outputs to new numpy arrays"}

    peak, peak_src = hbm_peak()
    kernels = {k: v for k, v in prof.items() if v["launches"]}
    top = dominant_kernel(kernels)
    kt = kernels[top]
    # 24 algorithmic bytes per string per distribution pass (the
    # 8-byte word plus the 8-byte handle read and written); the kernel's own
    # record model (DESIGN.md kernel table) is reported beside it
    alg_bytes = PASS_BYTES * kt["units"]
    ach = alg_bytes / (kt["ms"] / 1000.0) / 1e9 if kt["ms"] > 0 else 0.0
    ach_rec = kt["bytes"] / (kt["ms"] / 1000.0) / 1e9 if kt["ms"] > 0 else 0.0
    sort_gbs = b_alg(n, D) / (ms_step / 1000.0) / 1e9
    step_ms_sum = sum(v["ms"] for v in kernels.values()) / args.steps
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": args.config, "n": n, "N_bytes": int(len(buf)), "scale": args.scale,
                   "D": D, "L": L, "parallelism": f"dp{world}" if world > 1 else "1gpu",
                   "l2": "inputs larger than L2 (arena > 126 MB), no flush",
                   "kernel_timing": "per-kernel CUDA events in a second pass of the same steps with "
                                    "every kernel on one stream (exclusive launch times; value: the "
                                    "unprofiled timed region with the finishers on side streams)"},
        "d_bytes_per_s": D * world / (ms_step / 1000.0),
        "roofline": {"bound": "hbm", "kernel": top, "achieved": ach, "peak": peak,
                     "unit": "GB/s", "frac": ach / peak, "traffic": ncu_traffic(top),
                     "algorithmic_bytes_per_launch": alg_bytes / max(1, kt["launches"]),
                     "bytes_model": f"{PASS_BYTES} B per string (SURVEY 8d)",
                     "peak_source": peak_src,
                     "share_of_step": kt["ms"] / args.steps / profiled_ms,
                     "ncu_share_of_step": ncu_share(top),
                     "record_model": {"achieved": ach_rec, "frac": ach_rec / peak,
                                      "bytes_per_launch": kt["bytes"] / max(1, kt["launches"]),
                                      "model": "the kernel's own record traffic model "
                                               "(DESIGN.md kernel table)"}},
        "issue_roofline": issue_roofline(
            top, kt["ms"] / max(1, kt["launches"]), (clk.summary() or {}).get("sm_mhz") or 0,
            torch.cuda.get_device_properties(dev).multi_processor_count),
        "sort_roofline": {"b_alg_bytes": b_alg(n, D), "achieved": sort_gbs,
                          "frac": sort_gbs / peak, "unit": "GB/s"},
        "kernels": {k: {"ms_per_step": v["ms"] / args.steps,
                        "launches_per_step": v["launches"] / args.steps,
                        "units_per_step": v["units"] / args.steps,
                        "GBps": v["bytes"] / (v["ms"] / 1000) / 1e9 if v["ms"] else None}
                    for k, v in kernels.items()},
        "kernel_ms_per_step": step_ms_sum,
        "profiled_ms_per_step": profiled_ms,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu_line,
        "e2e": e2e,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c5_nodup")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="strings the CPU legs sort (prefix; 0 = the whole workload)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--l2-fetch", type=int, default=32)
    ap.add_argument("--strategy", choices=["sample", "merge"], default="sample",
                    help="N > 1: sample-sort exchange (default) or local sort + LCP merge")
    ap.add_argument("--dist", action="store_true",
                    help="run the multi-GPU (torchrun) code path even at N = 1 (checks)")
    args = ap.parse_args(argv)
    global TRAFFIC
    TRAFFIC = traffic_file(args.config)
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.dist:
        return run_dist(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
