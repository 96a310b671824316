"""Benchmark of the batched split-format DFT (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

A step is one pass of the hot path -- one batched forward transform of the
whole config batch (one kernel launch for N <= 4096) -- over inputs already
resident in HBM.  Default workload: BASELINE.json configs[2] in its fp64
variant (N=1024, B=2^18, seed 2, uniform[-1,1)) -- the largest single-GPU
configuration and the reference's own arithmetic (fp64 only,
layout.py:29-30); the other configs via --config.  With N GPUs
(``--gpus N``: spawned here with torchrun when WORLD_SIZE is unset) the
batch is split into N contiguous row blocks (``--scaling strong``, the
default, BASELINE configs[2] / SURVEY 8e) or every rank transforms its own
B rows (``--scaling weak``); no collective on the data path.  Config 5 (one
N = 2^28 transform) runs the sharded four-step.  The timed region is
bracketed by barrier + synchronize, timed with CUDA events on the launching
stream, and the max over ranks is reported.

Rank 0 prints ONE JSON line with the driver contract keys plus
``roofline`` (HBM-bound: algorithmic bytes 4*N*sizeof(real) per transform /
the measured kernel duration, against MEASURED_PEAKS.json hbm_gbs),
``cpu_baseline`` (the oracle's numpy restatement of the reference executor,
timed on this host's cores on a bounded sample of the same workload, plus
its one-process rate) and ``parity`` (relative L2 / bitwise agreement of
sampled rows of the timed output with the C oracle -- the checker, run
after the timed region),
``e2e`` (the same metric through the public ``fft_split`` on pinned HOST
buffers, H2D + D2H inside the timed region), ``gpu_launches`` and
``clocks`` (NVML samples taken during the timed region).

``--impl reference`` times the reference algorithm's CPU implementation
(the oracle's numpy port of transform.py, all host cores) on the same
config and prints the same line with ``"impl": "reference"``.
"""

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

BASELINE_METRIC = "batched split-DFT transforms/s and achieved HBM GB/s vs peak at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0
SPINUP_S = 0.5   # extra untimed warm-up time after the W warm-up steps (power/clock state settles)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg3_n1024_f64", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1 GPUs, batch configs: split the config's B rows across the ranks (strong) "
                         "or give every rank B rows (weak)")
    ap.add_argument("--parity-rows", type=int, default=64,
                    help="rows of the timed output checked against the C oracle after the timed region")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algorithm", default="dit", choices=["dit", "dif"])
    ap.add_argument("--radix-log", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="config 5 on N>1 GPUs: NCCL all-to-all, or phase 0 storing into the peers' "
                         "symmetric-memory receive buffers (fused exchange)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


KERNEL_SRC_DIR = os.path.join(ROOT, "paper_2504_07264_b200", "csrc")


def src_hash():
    """Hash of the kernel sources (hand-written .cu/.cuh/.h and the
    instantiation generator; the generated units follow from them)."""
    h = hashlib.sha256()
    for name in sorted(os.listdir(KERNEL_SRC_DIR)):
        if name.startswith("sfft_inst_") or name == "sfft_small_tw.h":
            continue
        if name.endswith((".cu", ".cuh", ".h", ".py")) or name == "Makefile":
            with open(os.path.join(KERNEL_SRC_DIR, name), "rb") as f:
                h.update(name.encode() + b"\0" + f.read())
    return h.hexdigest()[:16]


def ncu_traffic(cfg_name, algorithm="dit"):
    """(dram bytes per launch, note) from the committed ncu --set full capture
    of this config -- None unless the capture was taken from the kernel
    sources this run is built from (same src_hash) with the same algorithm."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None, "no committed ncu capture"
    with open(path) as f:
        d = json.load(f)
    v = d.get(cfg_name)
    if v is None:
        return None, "no committed ncu capture for this config"
    if v.get("src_hash") != src_hash():
        return None, f"stale: capture {v.get('source')} is of kernel sources {v.get('src_hash')}, not {src_hash()}"
    if v.get("algorithm", "dit") != algorithm:
        return None, f"capture is of the {v.get('algorithm', 'dit')} schedule"
    return float(v["dram_bytes_per_launch"]), f"{v.get('source')} (kernel sources {v.get('src_hash')})"


# ---------------------------------------------------------------- clocks ---
class ClockSampler:
    """NVML SM clock + clock-event reasons sampled every ~5 ms in a thread."""

    REASONS = {
        "hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
        "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
        "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
        "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
        "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown",
        "gpu_idle": "nvmlClocksEventReasonGpuIdle",
        "applications_clocks_setting": "nvmlClocksEventReasonApplicationsClocksSetting",
        "sync_boost": "nvmlClocksEventReasonSyncBoost",
    }

    def __init__(self, torch_device):
        self.samples = []
        self.ok = False
        self._stop = threading.Event()
        self.window = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            idx = torch.cuda._get_nvml_device_index(torch_device)
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # NVML missing: report it instead of guessing
            self.err = repr(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": f"nvml unavailable: {self.err}"}
        t0, t1 = self.window
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        note = "samples inside the timed region"
        if not inside:   # region shorter than one sample period: nearest samples
            inside = sorted(self.samples, key=lambda s: min(abs(s[0] - t0), abs(s[0] - t1)))[:3]
            note = "timed region shorter than the 5 ms sampling period; nearest samples"
        mask = 0
        for s in inside:
            mask |= s[2]
        reasons = [k for k, attr in self.REASONS.items() if mask & getattr(self.nv, attr, 0)]
        return {"sm_mhz": float(np.median([s[1] for s in inside])) if inside else None,
                "sm_max_mhz": float(self.max_mhz), "reasons": reasons,
                "samples": len(inside), "note": note}


# ------------------------------------------------------------ CPU side ---
def _cpu_worker(args):
    cfg_name, rows, algorithm = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    sys.path.insert(0, ROOT)
    from oracle import oracle
    cfg = workloads.CONFIGS[cfg_name]
    re, im = workloads.generate(cfg, rows=rows)
    plan = oracle.NumpyPlan(cfg.log2n, algorithm)
    t0 = time.perf_counter()
    for b in range(rows):
        oracle.split_to_split_numpy(plan, re[b], im[b])
    return time.perf_counter() - t0


def _cpu_one_signal(args):
    m, algorithm = args
    sys.path.insert(0, ROOT)
    from oracle import oracle
    rng = np.random.default_rng(4)
    re, im = rng.standard_normal(1 << m), rng.standard_normal(1 << m)
    plan = oracle.NumpyPlan(m, algorithm)
    t0 = time.perf_counter()
    oracle.split_to_split_numpy(plan, re, im)
    return time.perf_counter() - t0


def cpu_port_rate_long(cfg, algorithm, sample_m=20):
    """A single very long transform cannot be split across processes in the
    reference (no internal parallelism): time the numpy port on one
    2^sample_m-point signal and extrapolate by N log2 N."""
    t = _cpu_one_signal((sample_m, algorithm))
    scale = (cfg.n * cfg.log2n) / ((1 << sample_m) * sample_m)
    per = t * scale
    sample = (f"one 2^{sample_m}-point transform of the numpy port (transform.py:208-238) in "
              f"{t:.3f} s, extrapolated to N=2^{cfg.log2n} by N*log2N ({per:.1f} s per transform); "
              f"1 process (a single transform does not split)")
    return 1.0 / per, 1, sample, per


def cpu_port_rate(cfg, algorithm, target_s, procs=None):
    """Transforms/s of the numpy port of the reference executor over all host
    cores (one process per core, the reference has no internal parallelism).
    Sample: every worker transforms the first r rows of the config stream,
    with r sized so that one worker computes for about target_s seconds."""
    import multiprocessing as mp
    if cfg.log2n > 16:
        return cpu_port_rate_long(cfg, algorithm)
    procs = procs or os.cpu_count() or 1
    # size the sample with a 1-process probe
    probe_rows = max(1, min(cfg.batch, 64 if cfg.log2n <= 12 else 1))
    t = _cpu_worker((cfg.name, probe_rows, algorithm))
    per_row = t / probe_rows
    rows = int(max(1, min(cfg.batch, target_s / max(per_row, 1e-9))))
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        times = pool.map(_cpu_worker, [(cfg.name, rows, algorithm)] * procs)
    rate = rows * procs / max(times)
    sample = (f"first {rows} rows of the {cfg.name} stream in each of {procs} worker processes "
              f"(SplitSignal -> interleave -> fft -> deinterleave per row, numpy port of "
              f"transform.py:123-270); throughput = rows / max worker time")
    return rate, procs, sample, per_row


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------ reference ---
def run_reference(args):
    world, rank, _ = dist_env()
    cfg = workloads.CONFIGS[args.config]
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    if cfg.log2n > 16:
        rate, procs, sample, per = cpu_port_rate_long(cfg, args.algorithm)
        line = {
            "impl": "reference", "metric": BASELINE_METRIC, "value": rate, "unit": "transforms/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg.name, "n": cfg.n, "batch": cfg.batch},
            "cpu_baseline": {"value": rate, "unit": "transforms/s", "cores": procs, "kind": "port",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": rate, "unit": "transforms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return
    per_step_target = 1.0
    rate, procs, sample, per_row = cpu_port_rate(cfg, args.algorithm, min(2.0, per_step_target), procs)
    # steps: each a bounded sample (the same row prefix) on all cores
    import multiprocessing as mp
    rows = int(max(1, min(cfg.batch, per_step_target / max(per_row, 1e-9))))
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        for _ in range(args.warmup):
            pool.map(_cpu_worker, [(cfg.name, rows, args.algorithm)] * procs)
        t_steps = []
        for _ in range(args.steps):
            t_steps.append(max(pool.map(_cpu_worker, [(cfg.name, rows, args.algorithm)] * procs)))
    ms = 1e3 * float(np.mean(t_steps))
    value = rows * procs / (ms / 1e3)
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": value, "unit": "transforms/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "n": cfg.n, "batch": cfg.batch, "input_dtype": cfg.dtype,
                   "seed": cfg.seed, "step_rows": rows * procs},
        "cpu_baseline": {"value": value, "unit": "transforms/s", "cores": procs, "kind": "port",
                         "sample": f"each step: {sample.replace(f'first {rows}', f'first {rows}')}",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "transforms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours ---
def parity_check(cfg, algorithm, xr, xi, yr, yi, row0, rows):
    """The checker (after the timed region): sampled rows of the timed
    output against the C oracle (a bit-exact restatement of the reference
    executor, transform.py:123-270, pinned to reference-generated vectors)
    on the same inputs.  fp64: bitwise; fp32: relative L2 against the fp64
    oracle on the same fp32 inputs (north_star: <= 1e-5 * log2 N)."""
    from oracle import oracle
    b = xr.shape[0]
    idx = np.unique(np.linspace(0, b - 1, num=min(rows, b)).astype(np.int64))
    import torch
    ti = torch.from_numpy(idx).to(xr.device)
    xr_s, xi_s = xr.index_select(0, ti).cpu().numpy(), xi.index_select(0, ti).cpu().numpy()
    gr, gi = yr.index_select(0, ti).cpu().numpy(), yi.index_select(0, ti).cpu().numpy()
    t0 = time.perf_counter()
    wr, wi = oracle.fft_split_c(xr_s.astype(np.float64), xi_s.astype(np.float64), algorithm, False)
    t_oracle = time.perf_counter() - t0
    d = (gr.astype(np.float64) - wr) ** 2 + (gi.astype(np.float64) - wi) ** 2
    ref = wr ** 2 + wi ** 2
    per_row = np.sqrt(d.sum(1) / np.maximum(ref.sum(1), 1e-300))
    out = {"rows_checked": int(len(idx)), "row_indices": f"{len(idx)} rows evenly spaced over rows "
           f"[{row0}, {row0 + b}) of the {cfg.name} stream",
           "oracle": "oracle/liboracle.so (C restatement of transform.py:123-270, bitwise the reference)",
           "rel_l2_global": float(np.sqrt(d.sum() / ref.sum())), "rel_l2_max_row": float(per_row.max()),
           "oracle_s": t_oracle}
    if cfg.dtype == "f64":
        out["bitwise"] = bool(np.array_equal(gr.view(np.int64), wr.view(np.int64)) and
                              np.array_equal(gi.view(np.int64), wi.view(np.int64)))
        out["tolerance"] = "1e-12 (north_star, fp64); bitwise expected"
        out["pass"] = out["bitwise"] or out["rel_l2_max_row"] <= 1e-12
    else:
        tol = 1e-5 * cfg.log2n
        out["tolerance"] = f"{tol:g} (north_star 1e-5*log2N, fp32)"
        out["pass"] = out["rel_l2_max_row"] <= tol
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # SFFT_BENCH_BACKEND=gloo (test hook): ranks may share a GPU (index
    # local % device_count) and the barrier / max-over-ranks go over gloo
    backend = os.environ.get("SFFT_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        from paper_2504_07264_b200 import dist as sdist
        sdist.init_process_group(backend, device=torch.device("cuda", local) if backend == "nccl" else None)
    device = torch.device("cuda", local if world > 1 else torch.cuda.current_device())
    torch.cuda.set_device(device)

    import paper_2504_07264_b200 as sf
    from paper_2504_07264_b200 import _ffi
    from paper_2504_07264_b200.dist import shard_rows

    cfg = workloads.CONFIGS[args.config]
    dt = torch.float32 if cfg.dtype == "f32" else torch.float64
    # this rank's rows.  strong: rows [r0, r1) of the config's canonical
    # stream (the B rows split into `world` contiguous blocks); weak: B rows
    # per rank -- rank 0 the canonical stream, others a seeded variant of
    # the same distribution
    if args.scaling == "strong" or world == 1:
        r0, r1 = shard_rows(cfg.batch, world, rank)
        re, im = workloads.generate(cfg, rows=r1 - r0, start=r0)
    else:
        r0, r1 = 0, cfg.batch
        c2 = cfg if rank == 0 else workloads.Config(cfg.name, cfg.log2n, cfg.batch, cfg.dtype,
                                                    cfg.seed * 1000 + rank, cfg.dist)
        re, im = workloads.generate(c2)
    x_re = torch.from_numpy(re).to(device)
    x_im = torch.from_numpy(im).to(device)
    del re, im
    y_re = torch.empty_like(x_re)
    y_im = torch.empty_like(x_im)
    plan = sf.make_plan(cfg.log2n, args.algorithm, dtype=dt, device=device, radix_log=args.radix_log)
    stream = torch.cuda.current_stream(device)
    b, n = x_re.shape[0], cfg.n
    ws_bytes = plan.workspace_bytes(b)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=device)
    sp = stream.cuda_stream

    def step():
        _ffi.check(_ffi.lib.sfft_exec_split(plan._handle, x_re.data_ptr(), x_im.data_ptr(),
                                            y_re.data_ptr(), y_im.data_ptr(), b, n, n,
                                            _ffi.SFFT_FORWARD, ws.data_ptr() if ws_bytes else None, sp))

    # The clock sampler and the events exist before the warm-up so that nothing
    # but a synchronize (and the rank barrier) sits between the last warm-up
    # step and the timed region: an idle gap of even ~20 ms lets the power
    # controller re-boost the SM clock, and the first ~100 ms after that run
    # 5-9% slower than the settled state while it pulls the clock back under
    # the power cap (tools/spread_probe.py, profiles/r02aj_spread_probe.txt:
    # 1.47 -> 1.34 ms per step over 150 back-to-back steps of the headline).
    clocks = ClockSampler(device)
    clocks.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(device)
    # the W warm-up steps of a short step are over before the clocks settle:
    # keep stepping (untimed) for SPINUP_S, then go straight into the timed steps
    spin0 = time.perf_counter()
    while time.perf_counter() - spin0 < SPINUP_S:
        for _ in range(20):
            step()
        torch.cuda.synchronize(device)
    if world > 1:
        # the ranks leave their spin-up up to one burst apart: align them, settle
        # again together for 0.1 s (short bursts), and align once more -- the
        # second barrier then idles nobody for longer than a few steps
        dist.barrier()
        spin0 = time.perf_counter()
        while time.perf_counter() - spin0 < 0.1:
            for _ in range(5):
                step()
            torch.cuda.synchronize(device)
        dist.barrier()
    torch.cuda.synchronize(device)
    launches0 = _ffi.launch_count()
    # one event pair around the K steps: nothing sits between consecutive
    # launches of the stream (per-step events cost ~2% on the 0.17 ms cfg2
    # step and block the TMA kernel's dependent launch); SFFT_BENCH_STEP_EVENTS=1
    # records one per step for the step-time spread
    step_events = os.environ.get("SFFT_BENCH_STEP_EVENTS", "0") != "0"
    t_wall0 = time.perf_counter()
    ev[0].record(stream)
    for k in range(args.steps):
        step()
        if step_events or k == args.steps - 1:
            ev[k + 1].record(stream)
    torch.cuda.synchronize(device)
    t_wall1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    launches = _ffi.launch_count() - launches0
    clocks.mark(t_wall0, t_wall1)
    time.sleep(0.01)
    clocks.stop()
    total_ms = ev[0].elapsed_time(ev[-1])
    per_step = ([ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)] if step_events
                else [total_ms / args.steps] * args.steps)
    ms_local = total_ms / args.steps
    # roofline unit: one HBM sweep (a launch that reads and writes the whole
    # batch once); N > 4096 runs one launch per stage group
    n_launch, n_sweep = plan.schedule(b)
    kern_local = float(np.mean(per_step)) / n_sweep

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=device if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=device if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    ms = max_over_ranks(ms_local)
    kern_ms = max_over_ranks(kern_local)
    total_rows = int(sum_over_ranks(b))
    value = total_rows / (ms / 1e3)

    # ---------------- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        hr = torch.empty((b, n), dtype=dt, pin_memory=True)
        hi = torch.empty((b, n), dtype=dt, pin_memory=True)
        hr.copy_(x_re)
        hi.copy_(x_im)
        ho_r = torch.empty((b, n), dtype=dt, pin_memory=True)
        ho_i = torch.empty((b, n), dtype=dt, pin_memory=True)
        sf.fft_split(hr, hi, out=(ho_r, ho_i), plan=plan)   # warm the allocator
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(device)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            sf.fft_split(hr, hi, out=(ho_r, ho_i), plan=plan)
        e1.record(stream)
        torch.cuda.synchronize(device)
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps)
        ok = torch.equal(ho_r.to(device), y_re) and torch.equal(ho_i.to(device), y_im)
        e2e = {"value": total_rows / (e2e_ms / 1e3), "unit": "transforms/s",
               "h2d_bytes_per_step": int(hr.numel() * hr.element_size() * 2),
               "d2h_bytes_per_step": int(ho_r.numel() * ho_r.element_size() * 2),
               "ms_per_step": e2e_ms, "api": "paper_2504_07264_b200.fft_split(host pinned re, im, out=host)",
               "matches_device_result": bool(ok)}
        del hr, hi, ho_r, ho_i

    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    import dataclasses
    census = dataclasses.asdict(sf.count_flops(cfg.log2n))
    # every launch reads and writes both planes of the rank's rows once: the
    # fused kernel is the whole transform, each pass-group launch of the
    # multi-launch schedule (N > 4096) moves the same 4*N*sizeof(real) bytes
    bytes_per_launch = 4 * n * cfg.elem_bytes * b
    achieved = bytes_per_launch / (kern_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(cfg.name, args.algorithm)
    _, k_lr, kname = plan.exec_kernel(b)
    line = {
        "metric": BASELINE_METRIC,
        "value": value,
        "unit": "transforms/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "strong",
        "vs_baseline": None,
        "dtype": "f32" if cfg.dtype == "f32" else "f64",
        "data": "synthetic (seeded, BASELINE.json config shapes/distributions; workloads.py)",
        "config": {"workload": cfg.name, "n": n, "batch_per_gpu": b, "global_batch": total_rows,
                   "input_dtype": cfg.dtype, "seed": cfg.seed, "algorithm": args.algorithm,
                   "radix_log": k_lr,
                   "parallelism": (f"batch split into {world} contiguous row blocks (strong), no collective"
                                   if args.scaling == "strong" or world == 1 else
                                   f"batch-sharded x{world}, B rows per GPU (weak), no collective"),
                   "l2": f"inputs {2 * n * cfg.elem_bytes * b / 2**20:.0f} MiB per GPU "
                         f"{'>' if 2 * n * cfg.elem_bytes * b > 126e6 else '<='} 126 MB L2 (no flush)",
                   "extra_warmup_s": SPINUP_S},
        "gbs_algorithmic": 4 * n * cfg.elem_bytes * total_rows / (ms / 1e3) / 1e9,
        "gflops_5nlogn": 5 * n * cfg.log2n * total_rows / (ms / 1e3) / 1e9,
        # the reference's own census (count_flops, transform.py:312-335) next to 5N log2N
        "census": census,
        "gflops_census": (census["real_mults"] + census["real_adds"]) * total_rows / (ms / 1e3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": kname + f"<{cfg.dtype}, log2N={cfg.log2n}, radix=2^{k_lr}>",
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "unit_of_work": "launch" if n_launch == 1 else "sweep (one pass-group launch)",
                     "sweeps_per_step": n_sweep,
                     "launches_per_step": n_launch,
                     "kernel_ms": kern_ms, "peak_source": peak_src,
                     "frac_of_datasheet_8tbs": achieved / 8000.0,
                     "step_frac": bytes_per_launch / (ms / 1e3) / 1e9 / peak,
                     "kernel_src_hash": src_hash()},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        # cpu_baseline leg: the reference's CPU path (numpy port) on a
        # bounded sample, and the checker on sampled rows of the timed output
        rate, procs, sample, per_row = cpu_port_rate(cfg, args.algorithm, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": "transforms/s", "cores": procs, "kind": "port",
                                "sample": sample, "cpu_model": cpu_model(),
                                "one_process": {"value": 1.0 / per_row, "unit": "transforms/s", "cores": 1,
                                                "sample": "the sizing probe of the same stream, 1 process"}}
    if args.parity_rows > 0:
        line["parity"] = parity_check(cfg, args.algorithm, x_re, x_im, y_re, y_im, r0, args.parity_rows)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args):
    """Config 5 on N > 1 GPUs: one N = 2^28 transform, sharded four-step
    (phase 0, all-to-all of both planes over NCCL, phase 1); strong scaling."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    from paper_2504_07264_b200 import _ffi
    from paper_2504_07264_b200 import dist as sdist
    sdist.init_process_group("nccl", device=torch.device("cuda", local))
    device = torch.device("cuda", local)

    cfg = workloads.CONFIGS[args.config]
    dt = torch.float32 if cfg.dtype == "f32" else torch.float64
    plan = sdist.DistPlan(cfg.log2n, world, rank, dtype=dt, device=device)
    nl = plan.local_elems
    g = torch.Generator(device=device).manual_seed(cfg.seed * 1000 + rank)
    xr = torch.randn(nl, generator=g, device=device, dtype=torch.float64).to(dt)
    xi = torch.randn(nl, generator=g, device=device, dtype=torch.float64).to(dt)
    sr, si, rr, ri, yr, yi = (torch.empty_like(xr) for _ in range(6))
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=device)

    if args.transport == "p2p":
        xch = sdist.P2PExchange(plan)

        def step():
            xch.run(xr, xi, yr, yi, workspace=ws)
    else:
        def step():
            plan.phase(0, xr, xi, sr, si, workspace=ws)
            dist.all_to_all_single(rr, sr)
            dist.all_to_all_single(ri, si)
            plan.phase(1, rr, ri, yr, yi, workspace=ws)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(device)
    clocks = ClockSampler(device)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize(device)
    l0 = _ffi.launch_count()
    stream = torch.cuda.current_stream(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(device)
    t1 = time.perf_counter()
    dist.barrier()
    launches = _ffi.launch_count() - l0
    clocks.mark(t0, t1)
    clocks.stop()
    ms_t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=device)
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    if rank == 0:
        peak, src = peaks()
        # per-rank HBM bytes: every pass launch of the C dist plan reads and
        # writes the rank's N/G elements of both planes once
        sweeps = sum(plan.launches)
        moved = sweeps * 2 * 2 * nl * (4 if cfg.dtype == "f32" else 8)
        line = {
            "metric": BASELINE_METRIC, "value": 1.0 / (ms / 1e3), "unit": "transforms/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic (seeded per rank)",
            "config": {"workload": cfg.name, "n": cfg.n, "batch": 1,
                       "parallelism": f"sharded four-step x{world}, " + (
                           "NCCL all-to-all of both planes" if args.transport == "nccl"
                           else "phase 0 stores into peers' symmetric-memory receive buffers (P2P)")},
            "gbs_algorithmic": 4 * cfg.n * (4 if cfg.dtype == "f32" else 8) / (ms / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": moved / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": moved / (ms / 1e3) / 1e9 / peak, "traffic": None,
                         "sweeps_per_step": sweeps, "launches_per_phase": list(plan.launches),
                         "note": "per-rank HBM bytes of all pass launches (C dist plan) / step time "
                                 "(includes the all-to-all)",
                         "peak_source": src},
            "gpu_launches": int(launches), "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args):
    """--gpus N without a launcher: re-run this script under torchrun with N
    ranks (one per GPU) and pass rank 0's line through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
    cmd += [a for a in sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    world, _, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    elif world > 1 and workloads.CONFIGS[args.config].batch == 1:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
