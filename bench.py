"""Benchmark: StencilFFT-P periodic solve on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl reference]

A step is one full periodic solve a_T = IFFT(FFT(s)^T . FFT(a_0)) of the
configured synthetic grid.  The default workload is BASELINE configs[2]
(cfg3: 2D 9-point box, 8192^2 fp64, T = 1e5), one of the configs the
metric is quoted on at 1/2/4/8 GPUs and the largest 2D one that fits a B200;
`--impl reference` times the reference's CPU path on the same full grid.

`value`  cell-updates/s (cells * T / device time) with a_0 resident in HBM,
         the step timed with CUDA events on the solve's stream, L2 flushed
         (256 MiB write) before every step; max over ranks; whole-job sum.
`e2e`    the same metric through the public host API: the K steps as one
         fsx_solve_periodic_batch call (pinned host input and output; every
         step's H2D and D2H inside the timed region, overlapped across steps
         by the library's two lanes); `single_call_value` = one synchronous
         fsx_solve_periodic per step.
`roofline` the fused spectral kernel (k_cols_tma for plan 1): its
         algorithmic bytes / its CUDA-event duration (separate steps with the
         library's stage events on the solve stream).
`cpu_baseline` the reference's CPU path timed on this host, rank 0 at N = 1
         only: oracle/_ref (the reference's own sources compiled against a
         stand-in for the absent Eigen3, kind "reference") when built, else
         the oracle restatement (kind "port"); both are test infrastructure.

Multi-GPU (torchrun, one rank per GPU): 2D/3D configs are slab-decomposed
over the ranks (strong scaling; two NCCL all-to-alls per step, reported
against NVLink's 900 GB/s); 1D configs (cfg1, cfg5) run independent replicas
per rank (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/sec (N·T/wall) and FFT-pipeline HBM GB/s vs peak, 1/2/4/8 GPUs"
UNIT = "cell-updates/s"
FLUSH_BYTES = 256 << 20


NOMINAL_HBM_GBS = 8000.0  # the north star's "~8 TB/s" denominator, reported beside the measured copy peak


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_fp64(cfg_name, kernel_ms, kernel=""):
    """FP64 roofline of the dominant kernel: its per-launch FP64 pipe
    instructions (committed ncu count) over its live CUDA-event time, against
    the measured DFMA instruction rate (profiles/fp64_peak.json)."""
    try:
        cnt = json.load(open(os.path.join(ROOT, "profiles", "ncu_fp64.json"))).get(cfg_name)
        peak = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
    except Exception:
        return None
    if not cnt or not kernel_ms:
        return None
    if kernel and kernel.split()[0].split("<")[0] not in cnt.get("kernel", ""):
        return None  # the committed count is of another kernel than this build's
    peak_ops = peak["fp64_fma_tflops"] / 2.0  # DFMA instructions (tera) per second
    ach = cnt["pipe_ops"] / (kernel_ms * 1e-3) / 1e12
    return {"bound": "fp64 pipe", "achieved_tops": ach, "peak_tops": peak_ops, "frac": ach / peak_ops,
            "achieved_tflops": cnt["flops"] / (kernel_ms * 1e-3) / 1e12, "peak_tflops": peak["fp64_fma_tflops"],
            "pipe_ops_per_launch": cnt["pipe_ops"],
            "source": "ncu DADD+DMUL+DFMA thread instructions (profiles/ncu_fp64.json); peak measured by "
                      "scripts/micro/fp64_peak.cu (profiles/fp64_peak.json)"}


def load_traffic(cfg_name, kernel):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/ncu_traffic.json, stamped with the kernel it measured and
    the commit it was taken at).  None when the capture is of another kernel
    than the one this build launches (a stale count is not reported)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
    except Exception:
        return None, None
    name = t.get(cfg_name + "_kernel", "")
    if t.get(cfg_name) is None or not kernel.startswith(name.split("<")[0]) or name.split("<")[0] == "":
        return None, f"no capture of {kernel} in profiles/ncu_traffic.json"
    return t.get(cfg_name), f"ncu dram__bytes_read.sum + dram__bytes_write.sum of {name} at {t.get(cfg_name + '_head', 'round-1 HEAD')}"


def dominant_kernel(info, cfg):
    """The kernel bench.py's roofline times (the plan's fused spectral pass)."""
    if info["path"] == 1:
        n0 = cfg.dims[0]
        if n0 == 8192 and len(cfg.dims) == 2:
            return "k_fused8192c (8192-point columns, 2-CTA cluster)"
        return f"k_cols_tma<{n0}, 2>"
    if info["path"] == 2:
        n = cfg.dims[0]
        mc = n // 2 if cfg.fields == 1 else n  # complex points of the 1D row-pair plan
        b = mc.bit_length() - 1
        n2 = mc if mc <= 256 else 1 << min(12, (b + 1) // 2)
        n1 = mc // n2
        # 4096-point rows run on a CTA pair (k_rowpair_c), the others one row pair per CTA
        return f"k_rowpair_c<{n2}>" if (n2 == 4096 and n1 >= 4) else f"k_rowpair<{n2}>"
    return "k_spectral_general"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx.append(float(s[1]))
            except ValueError:
                continue
            for n, v in zip(names, s[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def mem_available_bytes():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def oracle_peak_bytes(cells, m):
    """Peak host RAM of the reference pipeline (~96 N bytes
    for m = 1, ~(32 m^2 + 80 m) N for m > 1)."""
    return cells * (96 if m == 1 else 32 * m * m + 80 * m)


def cpu_impl():
    """The CPU implementation the baseline legs time: oracle/_ref (the
    reference's own periodic-path sources compiled against oracle/eigen_shim,
    `kind` "reference") when it was built, else the oracle restatement
    ("port").  Returns (binding module, kind, one-line description)."""
    from oracle import ref as refmod

    if refmod.available() or refmod.build():
        return (refmod.module(), "reference",
                "oracle/_ref: the reference's own fft/spectrum/periodic/parallel/grid/kernel sources, unmodified, "
                "built with its flags (-O3 -DNDEBUG, C++20) against a stand-in for the absent Eigen3")
    from oracle import oracle as orc

    orc.build()
    return (orc, "port", "oracle (CPU restatement of the reference solve_periodic; radix-2/Bluestein FFT, "
            "FFT-of-generator spectrum, std::thread chunks)")


def cpu_sample(cfg, budget_s=None):
    """The CPU reference's workload: the FULL configured grid whenever the
    host has the RAM for the reference pipeline (and, if `budget_s` is given,
    one solve fits that budget by an N log N estimate); otherwise the largest
    halved grid that does.  Returns (sample config, offsets, blocks, a0)."""
    dims = list(cfg.dims)
    avail = mem_available_bytes()

    def fits(d):
        return oracle_peak_bytes(math.prod(d), cfg.fields) < 0.8 * avail if avail else True

    use = dims
    est = None
    if budget_s is not None:
        orc = cpu_impl()[0]
        small = [max(8, d // (16 if len(dims) > 1 else 64)) for d in dims]
        sc = cfg.scaled(small)
        off, blk = sc.kernel().arrays()
        a = sc.initial()
        t0 = time.perf_counter()
        orc.solve_periodic(a, small, cfg.fields, off, blk, cfg.T, vector=cfg.fields > 1)
        t_small, n_s = max(time.perf_counter() - t0, 1e-4), sc.cells()

        def est(d):
            n = math.prod(d)
            return t_small * (n / n_s) * (math.log2(n) / max(math.log2(n_s), 1.0))
    while math.prod(use) > 4096 and (not fits(use) or (est is not None and est(use) > budget_s)):
        use = [max(8, d // 2) for d in use]
    sample = cfg.scaled(use) if use != dims else cfg
    off, blk = sample.kernel().arrays()
    return sample, off, blk, sample.initial()


def run_reference(args, cfg):
    """--impl reference: the reference's CPU path (cpu_impl(): its own sources
    from oracle/_ref when built, else the restatement) on all host threads, on
    the SAME grid as our arm (no sample shrink unless the host lacks the RAM),
    K timed solves after W warm-ups."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    orc, kind, what = cpu_impl()
    cores = orc.thread_count()
    sample, off, blk, a = cpu_sample(cfg)
    for _ in range(args.warmup):
        orc.solve_periodic(a, sample.dims, sample.fields, off, blk, sample.T, vector=sample.fields > 1)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out = orc.solve_periodic(a, sample.dims, sample.fields, off, blk, sample.T, vector=sample.fields > 1)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = sample.cells() * sample.T / t
    desc = (f"{what} on grid {sample.dims} x{sample.fields}, T={sample.T}, "
            f"{cores} threads on {cpu_model()}; mean of {args.steps} solves (best {min(times):.3f} s)"
            + ("" if sample.dims == cfg.dims else f" (bounded sample of {cfg.dims}: host RAM)"))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SplitMix64, reference init)",
        "config": {"workload": cfg.name + ": " + cfg.description, "grid": cfg.dims, "fields": cfg.fields,
                   "T": cfg.T, "sample_grid": sample.dims, "same_grid": sample.dims == cfg.dims},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc,
                         "cpu_model": cpu_model(), "best_s": min(times), "mean_s": t},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "checksum": float(np.abs(out).sum()),
    }
    print(json.dumps(line), flush=True)


def run_gpu_slab(args, cfg, ws, rank, local):
    """N > 1 for a 2D/3D config: one global grid slab-decomposed over the ranks
    (strong scaling), two NCCL all-to-alls per step (distributed.SlabSolver)."""
    import torch
    import torch.distributed as dist

    import paper_2105_06676_b200 as fs
    from paper_2105_06676_b200.distributed import SlabSolver

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    shape, kern = cfg.shape(), cfg.kernel()
    exchange = args.exchange
    if exchange == "auto":
        exchange = "p2p" if len(cfg.dims) == 2 else "nccl"
    exchange_note = None
    try:
        solver = SlabSolver(shape, kern, cfg.T, exchange=exchange)
    except Exception as e:  # symmetric memory unavailable: the NCCL all-to-all path
        if args.exchange != "auto":
            raise
        exchange_note = f"p2p unavailable ({type(e).__name__}: {e}); NCCL all-to-all used"
        exchange = "nccl"
        solver = SlabSolver(shape, kern, cfg.T, exchange="nccl")
    nloc = solver.local_cells()
    start = rank * nloc
    host = cfg.initial(start, nloc)
    d_in = torch.from_numpy(host).cuda()
    d_out = torch.empty_like(d_in)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    for _ in range(args.warmup):
        flush.fill_(1)
        solver.solve(d_in, d_out)
    torch.cuda.synchronize()
    fs.device_check(stream=torch.cuda.current_stream().cuda_stream, device=dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    sampler = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.fill_(i)
        solver.solve(d_in, d_out, events=ev[i])
    torch.cuda.synchronize()
    dist.barrier()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    fs.device_check(stream=torch.cuda.current_stream().cuda_stream, device=dev)
    step = sum(e[0].elapsed_time(e[5]) for e in ev) / args.steps
    a2a = sum(e[1].elapsed_time(e[2]) + e[3].elapsed_time(e[4]) for e in ev) / args.steps
    fused = sum(e[2].elapsed_time(e[3]) for e in ev) / args.steps
    rowsx = sum(e[0].elapsed_time(e[1]) + e[4].elapsed_time(e[5]) for e in ev) / args.steps
    t = torch.tensor([step, a2a, fused, rowsx], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step, a2a, fused, rowsx = (float(x) for x in t)
    cells_T = cfg.cells() * cfg.T
    value = cells_T / (step * 1e-3)
    sent = 2 * solver.a2a_bytes()
    # nccl: the two all-to-alls; p2p: the NVLink traffic rides inside the row
    # kernels, so the row passes' time is the transfer window
    xfer_ms = a2a if exchange == "nccl" else rowsx
    nvl_gbs = sent / (xfer_ms * 1e-3) / 1e9 if xfer_ms > 0 else None
    # e2e: every rank's slab H2D from pinned memory + solve + D2H, max over ranks
    pin_in = torch.from_numpy(host).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        d_in.copy_(pin_in, non_blocking=True)
        solver.solve(d_in, d_out)
        pin_out.copy_(d_out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    et = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_val = cells_T / float(et[0])
    fs.device_check(stream=torch.cuda.current_stream().cuda_stream, device=dev)
    peak, peak_src = load_peaks()
    fused_bytes = 2 * solver.info["xbuf_bytes"]  # the rank's column tile in and out
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SplitMix64 stream of the reference's random init; " + cfg.init + f", seed {cfg.seed})",
        "config": {"workload": cfg.name + ": " + cfg.description, "grid": cfg.dims, "fields": cfg.fields,
                   "T": cfg.T, "parallelism": f"slab{ws} (axis 0)", "wall_s_timed_region": wall,
                   "l2": f"flushed before every step ({FLUSH_BYTES >> 20} MiB write)"},
        # nccl: the all-to-alls are their own window (frac = bytes / window / 900 GB/s);
        # p2p: the transfer rides inside the row kernels, so no window holds it
        # alone -- only a lower bound over the row passes is reported
        "nvlink": {"exchange": exchange, "exchange_note": exchange_note,
                   "transfer_ms_per_step": xfer_ms, "barrier_or_a2a_ms_per_step": a2a,
                   "bytes_sent_per_rank_per_step": sent, "achieved_gbs": nvl_gbs if exchange == "nccl" else None,
                   "peak_gbs": 900.0,
                   "frac": (nvl_gbs / 900.0) if (nvl_gbs and exchange == "nccl") else None,
                   "frac_lower_bound": (nvl_gbs / 900.0) if (nvl_gbs and exchange != "nccl") else None,
                   "window": "the two all-to-alls" if exchange == "nccl" else
                             "none separable: stores/loads inside the R2C/C2R row kernels (lower bound over those passes)"},
        "roofline": {"bound": "hbm", "kernel": "k_cols_tma (fused spectral pass, per rank)", "kernel_ms": fused,
                     "achieved": fused_bytes / (fused * 1e-3) / 1e9 if fused > 0 else None, "peak": peak,
                     "unit": "GB/s", "frac": (fused_bytes / (fused * 1e-3) / 1e9 / peak) if fused > 0 else None,
                     "traffic": None, "alg_bytes_per_launch": fused_bytes, "peak_source": peak_src},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": nloc * 8 * ws, "d2h_bytes_per_step": nloc * 8 * ws,
                "mode": "per rank: pinned slab H2D + SlabSolver.solve + D2H, max over ranks"},
        "gpu_launches": 3 * args.steps, "clocks": clocks,
    }
    # parity self-check of the decomposed solve: the slabs gathered on rank 0
    # against rank 0's own single-GPU solve of the whole grid
    gathered = [torch.empty_like(d_out) for _ in range(ws)] if rank == 0 else None
    dist.gather(d_out, gathered, dst=0)
    if rank == 0:
        full_in = torch.from_numpy(cfg.initial()).cuda()
        full_out = torch.empty_like(full_in)
        fs.solve_periodic_device(shape, full_in.data_ptr(), kern, cfg.T, full_out.data_ptr(), stream=0, device=dev)
        fs.device_check(stream=0, device=dev)
        slab = torch.cat(gathered)
        line["parity_vs_single_gpu_rel_l2"] = float(torch.linalg.vector_norm(slab - full_out) /
                                                    torch.linalg.vector_norm(full_out))
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def cpu_baseline(cfg):
    """The reference CPU path timed on this host (rank 0, N = 1): best of 3
    solves of the configured grid on all host threads (
    a halved-grid sample only when the host lacks the RAM or one solve would
    exceed ~30 s by an N log N estimate), plus a 1-thread solve of a bounded sample."""
    orc, kind, what = cpu_impl()
    cores = orc.thread_count()
    sample, off, blk, a = cpu_sample(cfg, budget_s=30.0)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        orc.solve_periodic(a, sample.dims, sample.fields, off, blk, sample.T, vector=sample.fields > 1)
        ts.append(time.perf_counter() - t0)
    tc = min(ts)
    # 1 thread on a bounded sample (the reference's 1D FFTs are serial anyway)
    s1, off1, blk1, a1 = cpu_sample(cfg, budget_s=4.0)
    orc.set_threads(1)
    try:
        t0 = time.perf_counter()
        orc.solve_periodic(a1, s1.dims, s1.fields, off1, blk1, s1.T, vector=s1.fields > 1)
        t1 = time.perf_counter() - t0
    finally:
        orc.set_threads(0)
    return {
        "value": sample.cells() * sample.T / tc, "unit": UNIT, "cores": cores, "kind": kind,
        "cpu_model": cpu_model(), "impl": what,
        "sample": f"best of 3 solve_periodic on grid {sample.dims} x{sample.fields}, T={sample.T}, "
                  f"{cores} threads ({', '.join(f'{x:.2f}' for x in ts)} s)"
                  + ("" if sample.dims == cfg.dims else f" (bounded sample of {cfg.dims})"),
        "one_thread": {"value": s1.cells() * s1.T / t1, "unit": UNIT, "cores": 1, "grid": s1.dims,
                       "seconds": t1},
    }


def run_gpu(args, cfg):
    import numpy as np
    import torch

    import paper_2105_06676_b200 as fs

    ws, rank, local = dist_env()
    if (ws > 1 or args.slab) and len(cfg.dims) in (2, 3) and cfg.fields == 1 and not args.replicas:
        return run_gpu_slab(args, cfg, ws, rank, local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    stream = torch.cuda.Stream()
    sptr = stream.cuda_stream
    shape, kern = cfg.shape(), cfg.kernel()
    info = fs.plan_describe(shape, kern)
    f32 = args.precision == 32  # fp32 storage mode: float grids in and out, fp64 arithmetic
    host = cfg.initial().astype(np.float32 if f32 else np.float64)
    n = host.size
    esz = host.itemsize
    d_a0 = torch.from_numpy(host).to(f"cuda:{dev}")
    d_out = torch.empty_like(d_a0)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device=f"cuda:{dev}")
    torch.cuda.synchronize()

    solve_dev = fs.solve_periodic_device_f32 if f32 else fs.solve_periodic_device

    def solve(stage=0):
        solve_dev(shape, d_a0.data_ptr(), kern, cfg.T, d_out.data_ptr(), stream=sptr, device=dev, stage_events=stage)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.fill_(1)
            solve()
    stream.synchronize()
    fs.device_check(stream=sptr, device=dev)

    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sampler = ClockSampler(dev if ws == 1 else local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    step_ms, fused_ms, host_us = [], [], []
    wall0 = time.perf_counter()
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.fill_(i)
            ev0[i].record(stream)
            h0 = time.perf_counter()
            solve()
            host_us.append((time.perf_counter() - h0) * 1e6)
            ev1[i].record(stream)
            ev1[i].synchronize()
            step_ms.append(ev0[i].elapsed_time(ev1[i]))
    torch.cuda.synchronize()
    # the fused kernel's own time: the same steps again with the library's
    # stage events (events between the passes would serialize the launches
    # that overlap through PDL in the timed steps above)
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.fill_(i)
            solve(stage=1)
            stream.synchronize()
            fused_ms.append(fs.last_stage_ms(device=dev)[1])
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    fs.device_check(stream=sptr, device=dev)
    ms = sum(step_ms) / len(step_ms)
    fms = sum(fused_ms) / len(fused_ms)
    if dist is not None:
        t = torch.tensor([ms, fms], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, fms = float(t[0]), float(t[1])
    cells_T = cfg.cells() * cfg.T
    value = cells_T * ws / (ms * 1e-3)

    # disclosure: in the default 2D fused path the multipliers of half-spectrum columns the host
    # proved to be exactly 0 are taken as 0 without evaluating the symbol (DESIGN 4b'); every
    # column is still loaded, transformed both ways and stored
    symbol_shortcut = None
    if info["path"] == 1 and len(cfg.dims) == 2 and not f32 and max(cfg.dims[0], 0) >= 4096:
        zc_on = os.environ.get("FSX_ZEROCOL", "1") != "0"
        kept0, total0 = fs.spectral_cut_columns(shape, kern, cfg.T)
        symbol_shortcut = {
            "enabled": zc_on, "columns_proved_zero": (total0 - kept0) if zc_on else 0, "columns": total0,
            "what": "multiplier 0 taken for host-proved zero columns without evaluating the symbol there; all "
                    "columns still loaded, transformed forward and back, and stored; bit-identical result; "
                    "FSX_ZEROCOL=0 evaluates every column"}

    # exact spectral cut (opt-in, fsx_options.spectral_cut): reported beside the
    # headline, which keeps the reference's full work.  Same steps, same flush;
    # the result must equal the full solve bit for bit.
    cut_line = None
    if info["path"] == 1 and len(cfg.dims) == 2 and not f32 and ws == 1 and not args.no_cut:
        kept, total = fs.spectral_cut_columns(shape, kern, cfg.T)
        full_out = d_out.clone()
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                flush.fill_(1)
                fs.solve_periodic_device(shape, d_a0.data_ptr(), kern, cfg.T, d_out.data_ptr(), stream=sptr,
                                         device=dev, spectral_cut=1)
            cut_ms = []
            for i in range(args.steps):
                flush.fill_(i)
                ev0[i].record(stream)
                fs.solve_periodic_device(shape, d_a0.data_ptr(), kern, cfg.T, d_out.data_ptr(), stream=sptr,
                                         device=dev, spectral_cut=1)
                ev1[i].record(stream)
                ev1[i].synchronize()
                cut_ms.append(ev0[i].elapsed_time(ev1[i]))
        torch.cuda.synchronize()
        fs.device_check(stream=sptr, device=dev)
        cms = sum(cut_ms) / len(cut_ms)
        R_b, H_b = n * 8, (info["alg_bytes"] - 2 * n * 8) // 4
        cut_line = {"value": cells_T / (cms * 1e-3), "unit": UNIT, "ms_per_step": cms,
                    "columns_kept": kept, "columns": total,
                    "bytes_per_step": int(2 * R_b + 4 * H_b * kept / total),
                    "bitwise_equal_to_full": bool(torch.equal(d_out, full_out)),
                    "what": "columns whose multipliers lam^T all underflow to 0 (|lam|^T < 2^-1100, bounded per "
                            "column) are neither stored, transformed nor read; opt-in, not the headline"}

    # e2e through the public host API: pinned host in/out, H2D + solve + D2H per step
    e2e_val = e2e_single = None
    if not args.no_e2e:
        tdt = torch.float32 if f32 else torch.float64
        pin_in = torch.from_numpy(host).pin_memory()
        pin_out = torch.empty(n, dtype=tdt).pin_memory()
        out_np = pin_out.numpy()
        if f32:
            def host_solve(out):
                fs.solve_periodic_f32(shape, pin_in.numpy(), kern, cfg.T, out=out)

            def host_batch(k, outs):
                fs.solve_periodic_batch_f32(shape, [pin_in.numpy()] * k, kern, cfg.T, outs)
        else:
            grid = fs.FieldGrid(shape, pin_in.numpy())

            def host_solve(out):
                fs.solve_periodic(grid, kern, cfg.T, out=out)

            def host_batch(k, outs):
                fs.solve_periodic_batch([grid] * k, kern, cfg.T, outs)
        for _ in range(max(1, args.warmup)):
            host_solve(out_np)
        # (a) one synchronous host call per step
        e2e_t = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            host_solve(out_np)
            e2e_t.append(time.perf_counter() - t0)
        et1 = sum(e2e_t) / len(e2e_t)
        # parity sanity: host result equals the device result
        assert np.array_equal(out_np, d_out.cpu().numpy())
        # (b) the K steps as one pipelined batch call (every step still moves its
        # input H2D and its result D2H; the lanes overlap them across steps)
        pin_out2 = torch.empty(n, dtype=tdt).pin_memory()
        outs = [out_np, pin_out2.numpy()]
        host_batch(max(2, args.warmup), [outs[i & 1] for i in range(max(2, args.warmup))])
        t0 = time.perf_counter()
        host_batch(args.steps, [outs[i & 1] for i in range(args.steps)])
        etb = (time.perf_counter() - t0) / args.steps
        assert np.array_equal(outs[(args.steps - 1) & 1], d_out.cpu().numpy())
        t = torch.tensor([et1, etb], dtype=torch.float64, device=f"cuda:{dev}")
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        et1, etb = float(t[0]), float(t[1])
        e2e_val = cells_T * ws / etb
        e2e_single = cells_T * ws / et1

    peak, peak_src = load_peaks()
    fused_gbs = info["fused_bytes"] / (fms * 1e-3) / 1e9 if fms > 0 else None
    alg_step = info["alg_bytes"]
    if f32:  # plan 1 reads / writes the grid as floats; the others widen (R/2 + R) and narrow (R + R/2)
        alg_step += -n * 8 if info["path"] == 1 else 3 * n * 8
    sched_step = alg_step + (info.get("sched_bytes", info["alg_bytes"]) - info["alg_bytes"])  # bytes the launched passes move
    pipe_gbs = alg_step / (ms * 1e-3) / 1e9
    kernel_name = dominant_kernel(info, cfg)
    traffic, traffic_src = load_traffic(cfg.name, kernel_name)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (SplitMix64 stream of the reference's random init; " + cfg.init + f", seed {cfg.seed})",
        "config": {
            "workload": cfg.name + ": " + cfg.description,
            "grid": cfg.dims, "fields": cfg.fields, "T": cfg.T,
            "parallelism": "replicas" if ws > 1 else "single",
            "l2": f"flushed before every step ({FLUSH_BYTES >> 20} MiB write), grid {n * esz >> 20} MiB",
            "storage": "f32 (fp32 storage mode: float grids in and out, fp64 arithmetic)" if f32 else "f64",
            "plan": info["path"],
            "wall_s_timed_region": wall,
            "symbol_shortcut": symbol_shortcut,
        },
        "roofline": {
            "bound": "hbm",
            "kernel": kernel_name,
            "achieved": fused_gbs,
            "peak": peak,
            "unit": "GB/s",
            "frac": (fused_gbs / peak) if fused_gbs else None,
            "frac_vs_nominal_8tbs": (fused_gbs / NOMINAL_HBM_GBS) if fused_gbs else None,
            "traffic": traffic,
            "traffic_source": traffic_src,
            "alg_bytes_per_launch": info["fused_bytes"],
            "kernel_ms": fms,
            "peak_source": peak_src,
            "fp64": None if f32 else load_fp64(cfg.name, fms, kernel_name),  # the fp32 mode's fused pass has its own counts
        },
        "pipeline": {"alg_bytes_per_step": alg_step, "achieved_gbs": pipe_gbs, "frac": pipe_gbs / peak,
                     "frac_vs_nominal_8tbs": pipe_gbs / NOMINAL_HBM_GBS,
                     "alg_bytes_source": "SURVEY.md 8(d) minimal schedule (2D 2R+4H, 3D 2R+8H, 1D 6R)",
                     "schedule_bytes_per_step": sched_step,
                     "schedule_frac": sched_step / (ms * 1e-3) / 1e9 / peak},
        "gpu_launches": info["launches"] * args.steps,
        "host_enqueue_us": sorted(host_us)[len(host_us) // 2],
        "clocks": clocks,
    }
    if cut_line is not None:
        line["spectral_cut"] = cut_line
    if e2e_val is not None:
        sfx = "_f32" if f32 else ""
        line["e2e"] = {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": n * esz, "d2h_bytes_per_step": n * esz,
                       "mode": f"fsx_solve_periodic_batch{sfx} of the {args.steps} steps (pinned host in/out; two lanes "
                               "overlap one step's D2H with the next step's H2D and kernels)",
                       "single_call_value": e2e_single,
                       "single_call_mode": f"one synchronous fsx_solve_periodic{sfx} per step"}
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def spawn_ranks(n):
    """`python bench.py --gpus N` without torchrun: relaunch this command as N
    ranks (one process per GPU) through torch.distributed.run on 127.0.0.1.
    Exits non-zero when fewer than N GPUs are visible."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} requested but {have} CUDA device(s) visible"}), flush=True)
        sys.exit(3)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3",
                    help="BASELINE config (default cfg3: 8192^2, T=1e5, one of the metric's 1/2/4/8-GPU configs)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", choices=["auto", "nccl", "p2p"], default="auto",
                    help="slab exchange for N > 1: p2p = fused into the row kernels over NVLink peer memory "
                         "(2D; auto falls back to nccl if symmetric memory is unavailable)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cut", action="store_true", help="skip the spectral_cut measurement (profiling runs)")
    ap.add_argument("--precision", type=int, choices=[64, 32], default=64,
                    help="32: the fp32 storage mode (float grids in/out, fp64 arithmetic; single GPU)")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of slabs")
    ap.add_argument("--slab", action="store_true", help="use the slab-decomposed path even at N=1 (under torchrun)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    from paper_2105_06676_b200.synthetic import configs

    cfg = configs()[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
