#!/usr/bin/env python3
"""ES-RNN training throughput on B200 (BASELINE.json metric: train series/sec, M4-Quarterly shape).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1|cfg2|cfg3|q24k|sweep<B>]
                    [--impl b200|reference] [--precision fp32|fp64]

A "step" is one pass of the hot path over the workload: one training epoch (every window
once, reference Trainer::train_epoch, trainer.hpp:234-243) followed by one validation
forecast (Trainer::validate, :292-305) — BASELINE configs[0] "one training epoch +
forecast".  Default workload (cfg1): M4-Quarterly-shaped synthetic data, 1,000 series
per GPU (weak scaling), length 88 (C=72 + 2*8), S=4, O=8, I=12, H=40, dilations
(1,2),(4,8), batch 1,000 per GPU, data seed 41, train seed 7, fp32.

value      series/s over all ranks, from CUDA-event device time of each step (max over
           ranks); the L2 is flushed (512 MiB write) between timed steps, outside the events.
e2e        the same metric through the public Python API with host buffers: every step
           constructs the Trainer from host arrays (H2D of the series), trains one epoch
           (H2D of the shuffled window plan), validates and reads back the losses,
           forecasts and sMAPE (D2H); wall clock, synchronised.
roofline   dominant kernel by device-time share of the timed configuration (the epoch's CUDA
           graph, programmatic dependent launch on): every CTA stamps the device global timer
           after its dependency wait and at its end, a kernel's time per step is its latest
           end minus its earliest start (esrnn_trainer_profile_kernels(t, 2)).  achieved =
           algorithmic work per launch (k_tile does the stack forward and the
           input adjoints = 2 x fwd FLOPs; k_grad_finish the weight-gradient contraction =
           1 x fwd FLOPs; k_adam / k_forecast_scan bytes) over that time.  `kernels` lists
           every kernel's share, time and roofline fraction.
cpu_baseline  the reference (oracle/_ref, the reference's own headers) timed on this host,
           1 core pinned with sched_setaffinity (it is single-threaded); CPU model and build
           flags recorded.  The reference arm also reports all_cores_upper_bound: one
           reference process per usable core, each on its own N/P-series shard (P separate
           models, so not the same training problem).

--gpus N without a torchrun environment re-launches itself under torch.distributed.run
with N ranks (127.0.0.1 rendezvous), one GPU per rank.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_1907_03329_b200 import _native as N  # noqa: E402
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer  # noqa: E402

REF_LIB = ROOT / "oracle" / "_ref" / "libesrnn_ref.so"
PORT_LIB = ROOT / "oracle" / "liboracle_esrnn.so"

CONFIGS = {
    # name: (frequency, series per GPU or total, length, season, batch per GPU, scaling)
    "cfg1": (Frequency.Quarterly, 1000, 88, 4, 1000, "weak"),
    "cfg2": (Frequency.Yearly, 23000, 25, 1, 2048, "strong"),
    "cfg3": (Frequency.Monthly, 48000, 108, 12, 2048, "strong"),
    "q24k": (Frequency.Quarterly, 24000, 88, 4, 2048, "strong"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def workload(name: str, world: int):
    if name.startswith("sweep"):
        B = int(name[5:])
        freq, n, length, s, scaling = Frequency.Quarterly, 24000, 88, 4, "strong"
        return freq, n, length, s, B, scaling
    freq, n, length, s, B, scaling = CONFIGS[name]
    if scaling == "weak":
        n, B = n * world, B * world
    return freq, n, length, s, B, scaling


def lstm_fwd_flops(prof: FrequencyProfile, B: int) -> float:
    """live-gate LSTM forward FLOPs, fwd = sum_l 2*B*in_l*3H + 2BH^2 + 2BHO.
    The step's FLOPs are 3 x fwd: k_tile does the forward and the input adjoints (2 x fwd),
    k_grad_finish the weight-gradient contraction (1 x fwd)."""
    H, O = prof.hidden_size, prof.horizon
    in0 = prof.input_window + 6
    layers = sum(len(b) for b in prof.dilation_blocks)
    return sum(2.0 * B * (in0 if l == 0 else H) * 3 * H for l in range(layers)) + 2.0 * B * H * H + 2.0 * B * H * O


def live_params(prof: FrequencyProfile) -> int:
    """Live shared parameters: W_in and bias over the i, g, o gates, head."""
    H, O = prof.hidden_size, prof.horizon
    in0 = prof.input_window + 6
    layers = sum(len(b) for b in prof.dilation_blocks)
    return sum(((in0 if l == 0 else H) + 1) * 3 * H for l in range(layers)) + H * H + H + H * O + O


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


REF_BUILD_FLAGS = "g++ -std=gnu++20 -O3 -march=x86-64-v4 (oracle/Makefile; the reference's Release flags, ISA pinned)"


def scan_bytes(prof: FrequencyProfile, k: int, T: int) -> float:
    """K1 algorithmic bytes (fp32): y (k*T) + params k(2+S) + levels k*T + seasonalities k(T+S)."""
    S = prof.seasonality_length
    return 4.0 * (k * T + k * (2 + S) + k * T + k * (T + S))


class ClockSampler:
    def __init__(self, path: Path):
        self.path, self.proc = path, None

    def _lines(self) -> int:
        try:
            return self.path.read_text().count("\n")
        except OSError:
            return 0

    def __enter__(self):
        # nvidia-smi takes ~100 ms to start: wait for its first sample so the (short) timed
        # region is covered, then sample every 20 ms
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
            return self
        t0 = time.time()
        while self._lines() < 1 and time.time() - t0 < 5.0:
            time.sleep(0.01)
        self.start_lines = self._lines()
        return self

    def __exit__(self, *a):
        if self.proc:
            # at least one sample taken after the timed region began
            t0 = time.time()
            while self._lines() <= self.start_lines and time.time() - t0 < 2.0:
                time.sleep(0.01)
            self.proc.terminate()
            self.proc.wait()

    def summary(self, device: int):
        try:
            rows = [r.split(", ") for r in self.path.read_text().strip().splitlines()]
        except Exception:
            return None
        rows = [r for r in rows if len(r) >= 9 and r[0].strip() == str(device)]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for i, nm in enumerate(names):
                if r[5 + i].strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]), "reasons": sorted(reasons),
                "samples": len(rows)}


def dist_setup(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def flush_l2(local: int):
    import torch
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = flush_l2.buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    buf.fill_(1.0)
    torch.cuda.synchronize()


def make_data(api, n, length, s, seed=41, sigma=0.05):
    return api.make_synthetic(seed, n, length, s, sigma)


# ----------------------------------------------------------------------------- CPU legs
def time_cpu(lib_path: Path, prof, cfg: TrainConfig, vals, cats, budget_s: float, warmup: int = 1):
    """Reference / port on this host, pinned to one core (the reference is single-threaded).
    `warmup` untimed epochs (or batches) first; then full epochs (+ validate) when an epoch
    fits the budget, else a bounded sample of training batches through run_batch(update)
    extrapolated to the epoch."""
    core = None
    old = None
    if hasattr(os, "sched_setaffinity"):
        old = os.sched_getaffinity(0)
        core = max(old)
        os.sched_setaffinity(0, {core})
    try:
        r = _time_cpu(lib_path, prof, cfg, vals, cats, budget_s, warmup)
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    r.update({"pinned_core": core, "cpu_model": cpu_model(), "build": REF_BUILD_FLAGS if lib_path == REF_LIB else
              "gcc -std=c11 -O2 (oracle/Makefile)"})
    return r


def _time_cpu(lib_path: Path, prof, cfg: TrainConfig, vals, cats, budget_s: float, warmup: int):
    api = N.NativeApi(lib_path)
    n = vals.shape[0]
    cfg_c = TrainConfig(**{**cfg.__dict__, "precision": "fp64", "max_batch_size": 0,
                           "batch_size": min(cfg.batch_size, 2048)})
    tr = Trainer((vals, cats), prof, cfg_c, api=api)
    T = vals.shape[1] - 2 * prof.horizon
    per = T - prof.horizon - prof.input_window + 1
    nw = n * per
    steps = -(-nw // cfg_c.batch_size)
    from paper_1907_03329_b200.trainer import WindowBatch
    t0 = time.perf_counter()
    tr.step(WindowBatch([0], [prof.input_window - 1]), update=False)
    probe = time.perf_counter() - t0
    # estimate one epoch: probe a single full batch
    w = tr.all_windows()
    rng = np.random.default_rng(0)
    idx = rng.integers(0, len(w), size=cfg_c.batch_size)
    b = WindowBatch([w[i][0] for i in idx], [w[i][1] for i in idx])
    t0 = time.perf_counter()
    tr.step(b, update=True)
    per_batch = time.perf_counter() - t0
    est_epoch = per_batch * steps
    times = []
    if est_epoch <= budget_s / 2:
        kind = "epochs"
        for _ in range(warmup):
            tr.train_epoch()
            tr.validate()
        t_start = time.perf_counter()
        while time.perf_counter() - t_start < budget_s or not times:
            t0 = time.perf_counter()
            tr.train_epoch()
            tr.validate()
            times.append(time.perf_counter() - t0)
        step_s = statistics.median(times)
        sample = f"{len(times)} full epochs (+validate) of {n} series after {warmup} untimed, median"
    else:
        kind = "batches"
        for _ in range(warmup):
            idx = rng.integers(0, len(w), size=cfg_c.batch_size)
            tr.step(WindowBatch([w[i][0] for i in idx], [w[i][1] for i in idx]), update=True)
        t_start = time.perf_counter()
        nb = 0
        while time.perf_counter() - t_start < budget_s or nb == 0:
            idx = rng.integers(0, len(w), size=cfg_c.batch_size)
            b = WindowBatch([w[i][0] for i in idx], [w[i][1] for i in idx])
            tr.step(b, update=True)
            nb += 1
        per_batch = (time.perf_counter() - t_start) / nb
        t0 = time.perf_counter()
        tr.validate()
        val_s = time.perf_counter() - t0
        step_s = per_batch * steps + val_s
        sample = (f"{nb} training batches of {cfg_c.batch_size} windows (+1 validate), extrapolated to "
                  f"{steps} batches/epoch")
    del probe, kind
    return {"value": n / step_s, "unit": "series/s", "cores": 1, "epoch_s": step_s, "sample": sample,
            "host_cores": os.cpu_count()}


def _shard_worker(args):
    """One process of the all-host-cores bound: the reference trainer on one shard of the
    series, full epochs (+ validate) for `budget_s`; returns series/s of this shard."""
    lib, freq_name, vals, cats, cfg_d, budget_s = args
    api = N.NativeApi(Path(lib))
    prof = FrequencyProfile.defaults(Frequency[freq_name])
    tr = Trainer((vals, cats), prof, TrainConfig(**cfg_d), api=api)
    tr.train_epoch()  # warm-up
    n_ep, t_start = 0, time.perf_counter()
    while time.perf_counter() - t_start < budget_s or n_ep == 0:
        tr.train_epoch()
        tr.validate()
        n_ep += 1
    return vals.shape[0] * n_ep / (time.perf_counter() - t_start)


def time_cpu_all_cores(lib_path: Path, prof, cfg: TrainConfig, vals, cats, budget_s: float):
    """SURVEY §8(d) optional upper bound: P = usable host cores independent reference
    processes, each training its own contiguous N/P-series shard concurrently; aggregate
    series/s.  NOT the same training problem (P separate models) -- reported beside the
    1-core number, never instead of it."""
    import multiprocessing as mp
    n = vals.shape[0]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    P = max(1, min(cores, 128, n // 4))
    cfg_d = {**cfg.__dict__, "precision": "fp64", "max_batch_size": 0, "batch_size": min(cfg.batch_size, 2048)}
    bounds = [n * p // P for p in range(P + 1)]
    jobs = [(str(lib_path), prof.frequency.name, np.ascontiguousarray(vals[bounds[p]:bounds[p + 1]]),
             np.ascontiguousarray(cats[bounds[p]:bounds[p + 1]]), cfg_d, budget_s) for p in range(P)]
    with mp.get_context("spawn").Pool(P) as pool:
        rates = pool.map(_shard_worker, jobs, chunksize=1)
    return {"value": float(sum(rates)), "unit": "series/s", "cores": P, "host_cores": os.cpu_count(),
            "sample": f"{P} concurrent processes x {n // P}-{-(-n // P)} series each, full epochs (+validate) "
                      f"for ~{budget_s:.0f} s after one warm-up epoch",
            "note": "P independent models on series shards: not the same training problem (upper bound)"}


# ----------------------------------------------------------------------------- main
def spawn_ranks(a) -> int:
    """--gpus N outside torchrun: run this script under torch.distributed.run with N ranks."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a))
    world, rank, local = dist_setup(a.gpus)
    freq, n_total, length, s, B, scaling = workload(a.config, world)
    prof = FrequencyProfile.defaults(freq)
    metric = "train series/sec (M4-Quarterly shape) at 1/2/4/8 B200 vs CPU ref; sMAPE parity"
    cfg_desc = {"workload": f"{a.config}: {freq.name}-shaped synthetic, {n_total} series x length {length}, "
                            f"S={s}, O={prof.horizon}, I={prof.input_window}, H={prof.hidden_size}, "
                            f"dilations {prof.dilation_blocks}, batch {B}; step = 1 train epoch + validate",
                "series": n_total, "global_batch": B, "length": length, "parallelism": f"series-sharded dp{world}",
                "l2": "flushed between timed steps (512 MiB write)", "data_seed": 41, "train_seed": 7}

    if a.impl == "reference":
        if rank != 0:
            return
        lib = REF_LIB if REF_LIB.exists() else PORT_LIB
        kind = "reference" if lib == REF_LIB else "port"
        api = N.NativeApi(PORT_LIB if kind == "port" else REF_LIB)
        vals, cats = make_data(api, n_total, length, s)
        cfg = TrainConfig(batch_size=min(B, 2048), seed=7, precision="fp64")
        # W untimed epochs (or batches) before the first timed step, in the same process
        res = [time_cpu(lib, prof, cfg, vals, cats, budget_s=max(3.0, 60.0 / max(a.steps, 1)),
                        warmup=max(a.warmup, 0) if i == 0 else 0)
               for i in range(max(a.steps, 1))]
        v = statistics.median(r["value"] for r in res)
        allc = None
        if not a.no_cpu_baseline:
            allc = time_cpu_all_cores(lib, prof, cfg, vals, cats, budget_s=10.0)
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": v, "unit": "series/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000.0 * n_total / v, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg_desc,
            "cpu_baseline": {"value": v, "unit": "series/s", "cores": 1, "kind": kind, "sample": res[0]["sample"],
                             "cpu_model": res[0]["cpu_model"], "pinned_core": res[0]["pinned_core"],
                             "host_cores": os.cpu_count(), "build": res[0]["build"],
                             "all_cores_upper_bound": allc},
            "e2e": {"value": v, "unit": "series/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    api = N.product_api()
    vals, cats = make_data(api, n_total, length, s)
    cfg = TrainConfig(batch_size=B, seed=7, precision=a.precision, device=local,
                      max_batch_size=max(B, 2048))
    def new_dist():
        # every NCCL communicator needs its own unique id (rank 0 draws it, all ranks get it)
        if world == 1:
            return None
        import torch.distributed as dist
        uid = [api.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        return (rank, world, uid[0])

    tr = Trainer((vals, cats), prof, cfg, api=api, dist=new_dist())
    n_local = tr.row_end - tr.row_begin

    for _ in range(a.warmup):
        tr.train_epoch()
        tr.validate()
    losses = []
    dev_ms = []
    wall = []
    launches0 = tr.kernel_launches()
    clock = ClockSampler(ROOT / "gpurun_out" / f"clocks_r{rank}.csv") if (ROOT / "gpurun_out").exists() else \
        ClockSampler(Path(f"/tmp/esrnn_clocks_r{rank}.csv"))
    import torch
    torch.cuda.synchronize()
    barrier(world)
    with clock:
        for _ in range(a.steps):
            flush_l2(local)
            barrier(world)
            t0 = time.perf_counter()
            losses.append(tr.train_epoch())
            m_train = tr.last_device_ms()
            v = tr.validate()
            m_val = tr.last_device_ms()
            wall.append(time.perf_counter() - t0)
            dev_ms.append(m_train + m_val)
    torch.cuda.synchronize()
    barrier(world)
    launches = tr.kernel_launches() - launches0
    total_ms = allreduce_max(sum(dev_ms), world)
    value = n_total * a.steps / (total_ms / 1000.0)
    clocks = clock.summary(local)

    # Per-kernel time in the timed configuration (outside the timed region): the epoch graph
    # with in-kernel global-timer spans; the forecast kernels (no graph) by CUDA events
    tr.profile_kernels(2)
    tr.train_epoch()  # captures the span-instrumented graph
    tr.profile_kernels(2)  # reset
    n_span_epochs = 3
    for _ in range(n_span_epochs):
        tr.train_epoch()
    kt = tr.kernel_times()
    tr.profile_kernels(1)
    tr.validate()
    kt_fc = tr.kernel_times()
    tr.profile_kernels(0)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12
    fma_peak = fp32_peak if a.precision == "fp32" else fp32_peak / 2
    hbm_peak = peaks.get("hbm_gbs", 6553.9)
    T = length - 2 * prof.horizon
    per = T - prof.horizon - prof.input_window + 1
    steps_per_epoch = -(-n_total * per // B)
    B_local = B // world
    S = prof.seasonality_length
    rb = 4 if a.precision == "fp32" else 8
    # DRAM traffic per launch, from the committed ncu --set full capture of this workload
    traffic = {}
    tf = ROOT / "profiles" / f"ncu_traffic_{a.config}.json"
    if tf.exists():
        doc = json.loads(tf.read_text())
        if doc.get("config") == a.config and doc.get("precision", "fp32") == a.precision:
            traffic = doc.get("kernels", {})
    windows_local = n_local * per  # every window once per epoch
    P_live = live_params(prof)
    k_slots = min(n_local, B_local)
    kern = {}

    def add(name, cls, ms_tot, launches, work, unit, peak, note):
        if not launches:
            return
        avg_s = ms_tot / launches / 1e3
        ach = work / avg_s / (1e12 if unit == "TFLOP/s" else 1e9)
        kern[name] = {"class": cls, "ms_per_step": ms_tot / (n_span_epochs if cls != "forecast" else 1),
                      "launches_per_step": launches / (n_span_epochs if cls != "forecast" else 1),
                      "avg_us": avg_s * 1e6, "algorithmic_per_launch": work, "achieved": ach, "unit": unit,
                      "peak": peak, "frac": ach / peak, "work": note,
                      "traffic": traffic.get(name, traffic.get(name + "_sc"))}

    fwd_epoch = lstm_fwd_flops(prof, windows_local)
    ms, n = kt["tile"]
    add("k_tile", "train", ms, n, 2.0 * fwd_epoch / max(n / n_span_epochs, 1), "TFLOP/s", fma_peak,
        "stack forward + input adjoints = 2 x fwd FLOPs of the step's windows (SURVEY §8(d))")
    ms, n = kt["finish"]
    add("k_grad_finish", "train", ms, n, fwd_epoch / max(n / n_span_epochs, 1), "TFLOP/s", fma_peak,
        "weight-gradient contraction = 1 x fwd FLOPs (its ES reverse-scan blocks run beside it)")
    ms, n = kt["adam"]
    add("k_adam", "train", ms, n, rb * (7.0 * P_live + 7.0 * k_slots * (2 + S)) + 8.0 * k_slots, "GB/s", hbm_peak,
        "SURVEY K5 bytes: 7 x (P_live + k(2+S)) Real + 8k")
    if "finalize" in kt:
        ms, n = kt["finalize"]
        add("k_finalize/k_group_reduce", "train", ms, n, rb * 2.0 * P_live, "GB/s", hbm_peak, "reduced buffer in+out")
    fmsn = kt_fc.get("forecast_scan")
    if fmsn:
        add("k_forecast_scan", "forecast", fmsn[0], fmsn[1], rb * (n_local * (length - 2 * prof.horizon) + n_local * (2 + S)
                                                               + n_local * (prof.input_window + 6) + n_local * (1 + prof.horizon)),
            "GB/s", hbm_peak, "SURVEY K6 bytes: observations to t_ins + params + window/level/seasonality outputs")
    fmsn = kt_fc.get("forecast_tile")
    if fmsn:
        add("k_tile<forecast>", "forecast", fmsn[0], fmsn[1], lstm_fwd_flops(prof, n_local), "TFLOP/s", fma_peak,
            "stack forward over every series (1 x fwd FLOPs)")
    step_ms = sum(kv["ms_per_step"] for kv in kern.values())
    for kv in kern.values():
        kv["share"] = kv["ms_per_step"] / step_ms if step_ms else None
    dom = max(kern, key=lambda k: kern[k]["ms_per_step"])
    d = kern[dom]
    roof = {"kernel": dom, "bound": "fp32-fma" if d["unit"] == "TFLOP/s" else "hbm", "achieved": d["achieved"],
            "peak": d["peak"], "unit": d["unit"], "frac": d["frac"], "traffic": d["traffic"],
            "algorithmic_per_launch": d["algorithmic_per_launch"], "work": d["work"],
            "timing": "in-graph global-timer spans (PDL on), mean over 3 epochs",
            "peak_source": (f"derived CUDA-core FP32 FMA peak: 148 SM x 128 lanes x 2 x {sm_max:.0f} MHz "
                            f"(MEASURED_PEAKS sm_max_mhz){'; fp64 = half' if a.precision == 'fp64' else ''}; "
                            "no tensor-core path at these batch sizes (fp32 contract)")
            if d["unit"] == "TFLOP/s" else "MEASURED_PEAKS hbm_gbs (measured)"}
    shares = kern

    # e2e through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        e2e_t = []
        h2d = d2h = 0
        n_e2e = max(1, a.warmup) + max(1, a.steps)
        dists = [new_dist() for _ in range(n_e2e + 1)]  # drawn outside the timed region
        for it in range(n_e2e):
            barrier(world)
            t0 = time.perf_counter()
            t2 = Trainer((vals, cats), prof, cfg, api=api, dist=dists[it])
            t2.train_epoch()
            v2 = t2.validate()
            t2.close()
            if it >= max(1, a.warmup):
                e2e_t.append(time.perf_counter() - t0)
            # the series go up once as fp64 (laid out on the device); the epoch plan is 8
            # int32 arrays per window (w_row/anchor/slot/first/csr, csr_anchor, slot_win, slot_row)
            h2d = n_local * length * 8 + n_local * per * 8 * 4
            d2h = steps_per_epoch * 8 + v2.forecasts.nbytes + v2.smape_per_series.nbytes
        e2e_s = allreduce_max(sum(e2e_t), world)
        # the same through a trainer built once (the reference arm's usage: construct, then
        # epochs): per step the epoch's window plan goes H2D from pinned memory and the
        # losses, forecasts and sMAPE come back D2H
        t3 = Trainer((vals, cats), prof, cfg, api=api, dist=dists[n_e2e])
        res_t = []
        for it in range(max(1, a.warmup) + max(1, a.steps)):
            barrier(world)
            t0 = time.perf_counter()
            t3.train_epoch()
            t3.validate()
            if it >= max(1, a.warmup):
                res_t.append(time.perf_counter() - t0)
        t3.close()
        res_s = allreduce_max(sum(res_t), world)
        e2e = {"value": n_total * len(e2e_t) / e2e_s, "unit": "series/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": [1000 * x for x in e2e_t],
               "what": "Trainer(series) construction + train_epoch + validate + destroy per step, wall clock",
               "resident": {"value": n_total * len(res_t) / res_s, "unit": "series/s",
                            "h2d_bytes_per_step": int(n_local * per * 8 * 4),
                            "d2h_bytes_per_step": int(steps_per_epoch * 8 + v2.forecasts.nbytes
                                                      + v2.smape_per_series.nbytes),
                            "what": "trainer built once; per step train_epoch + validate through the API, "
                                    "wall clock (plan H2D, losses / forecasts / sMAPE D2H)"}}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        lib = REF_LIB if REF_LIB.exists() else PORT_LIB
        kind = "reference" if lib == REF_LIB else "port"
        cb = time_cpu(lib, prof, TrainConfig(batch_size=min(B, 2048), seed=7), vals, cats, a.cpu_seconds)
        cpu = {"value": cb["value"], "unit": "series/s", "cores": 1, "kind": kind, "sample": cb["sample"],
               "host_cores": cb["host_cores"], "cpu_model": cb["cpu_model"], "pinned_core": cb["pinned_core"],
               "build": cb["build"]}

    # the same step in fp64 parity mode (the reference's arithmetic), device-timed, for context
    fp64_line = None
    if world == 1 and a.precision == "fp32":
        t64 = Trainer((vals, cats), prof, TrainConfig(**{**cfg.__dict__, "precision": "fp64"}), api=api)
        for _ in range(max(1, a.warmup)):
            t64.train_epoch()
            t64.validate()
        ms64 = []
        for _ in range(max(1, a.steps)):
            flush_l2(local)
            t64.train_epoch()
            m = t64.last_device_ms()
            v64 = t64.validate()
            ms64.append(m + t64.last_device_ms())
        fp64_line = {"value": n_total * len(ms64) / (sum(ms64) / 1000.0), "unit": "series/s",
                     "ms_per_step": statistics.mean(ms64), "val_smape": v64.mean_smape, "dtype": "f64"}
        t64.close()

    if rank == 0:
        out = {
            "metric": metric, "value": value, "unit": "series/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32" if a.precision == "fp32" else "f64",
            "data": "synthetic (reference generator make_multiplicative_series, seed 41)", "config": cfg_desc,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "wall_ms_per_step": 1000.0 * statistics.mean(wall), "epoch_losses": losses,
            "val_smape": v.mean_smape, "kernels": shares, "fp64_engine": fp64_line,
            "speedup_vs_cpu": (value / cpu["value"]) if cpu else None,
        }
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
