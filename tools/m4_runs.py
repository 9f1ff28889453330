#!/usr/bin/env python3
"""BASELINE configs[3] and configs[4] on one B200 (the bench line itself is configs[1], cfg1).

    python tools/m4_runs.py sweep   [--out gpurun_out/r01_sweep.json]
    python tools/m4_runs.py mixed   [--epochs 15] [--out gpurun_out/r01_m4_mixed.json]

sweep: the paper's speedup-vs-batch curve: one training
       epoch at batch B on Quarterly-shaped data -- Q-1k for B <= 2,048 (the reference cap,
       trainer.hpp:36-37) with the reference CPU timed beside it on a bounded sample, Q-24k
       for B = 4,096 .. 48,000 (GPU only; the reference rejects B > 2,048).
mixed: the full-M4-scale run: 23,000 Yearly + 24,000 Quarterly + 48,000
       Monthly series, one model per frequency (trainer.hpp:165-170), `--epochs` epochs each,
       then cmd_evaluate scoring on the test block (sMAPE / MASE / seasonal-naive) and the
       count-weighted overall sMAPE (metrics.hpp:94-137).  Wall time end to end.
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1907_03329_b200 import _native as N  # noqa: E402
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer  # noqa: E402


def gpu_epoch_ms(api, vals, cats, prof, B, reps=3):
    # tiny batches mean tens of thousands of steps per epoch: launch eagerly instead of
    # capturing one enormous graph
    tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=B, max_batch_size=max(B, 2048),
                                                 use_graphs=B >= 64, precision="fp32"), api=api)
    for _ in range(2):
        tr.train_epoch()
    ms = []
    for _ in range(reps):
        tr.train_epoch()
        ms.append(tr.last_device_ms())
    tr.close()
    return statistics.median(ms)


def sweep(out):
    import bench  # the reference CPU timer (bounded samples)
    api = N.product_api()
    prof = FrequencyProfile.defaults(Frequency.Quarterly)
    rows = []
    v1, c1 = api.make_synthetic(41, 1000, 88, 4, 0.05)
    for B in (1, 4, 16, 64, 128, 256, 512, 1000, 2048):
        ms = gpu_epoch_ms(api, v1, c1, prof, B, reps=1 if B < 16 else 3)
        row = {"B": B, "series": 1000, "gpu_epoch_ms": ms, "gpu_series_per_s": 1000 / (ms / 1e3)}
        if bench.REF_LIB.exists():
            cb = bench.time_cpu(bench.REF_LIB, prof, TrainConfig(batch_size=B, seed=7), v1, c1, budget_s=3.0)
            row.update({"cpu_series_per_s": cb["value"], "cpu_sample": cb["sample"],
                        "speedup": row["gpu_series_per_s"] / cb["value"]})
        rows.append(row)
        print(json.dumps(row), flush=True)
    v24, c24 = api.make_synthetic(41, 24000, 88, 4, 0.05)
    for B in (2048, 4096, 8192, 16384, 32768, 48000):
        ms = gpu_epoch_ms(api, v24, c24, prof, B)
        row = {"B": B, "series": 24000, "gpu_epoch_ms": ms, "gpu_series_per_s": 24000 / (ms / 1e3),
               "cpu_reference": "Q-24k B=2048 plateau 16.2 s/epoch (SURVEY §6, reference rejects B > 2048)",
               "speedup_vs_cpu_plateau": 16.2 / (ms / 1e3)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    Path(out).write_text(json.dumps({"what": "one training epoch per point, device time (CUDA events), fp32; "
                                             "CPU = reference (oracle/_ref), 1 thread, bounded sample",
                                     "rows": rows}, indent=1))


def mixed(out, epochs):
    api = N.product_api()
    res = {}
    t_all = time.perf_counter()
    for freq, n, seed in ((Frequency.Yearly, 23000, 41), (Frequency.Quarterly, 24000, 42), (Frequency.Monthly, 48000, 43)):
        prof = FrequencyProfile.defaults(freq)
        length = prof.min_length + 2 * prof.horizon
        vals, cats = api.make_synthetic(seed, n, length, prof.seasonality_length, 0.05)
        t0 = time.perf_counter()
        tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=2048, precision="fp32"), api=api)
        dev = 0.0
        losses = []
        for _ in range(epochs):
            losses.append(tr.train_epoch())
            dev += tr.last_device_ms()
            tr.validate()
            dev += tr.last_device_ms()
        ev = tr.evaluate(True)
        wall = time.perf_counter() - t0
        res[freq.name] = {"series": n, "length": length, "epochs": epochs, "wall_s": wall, "device_ms": dev,
                          "final_train_loss": losses[-1], "test_smape": ev.mean_smape, "test_mase": ev.mean_mase,
                          "naive_test_smape": float(ev.totals[3] / ev.totals[6])}
        tr.close()
        print(freq.name, json.dumps(res[freq.name]), flush=True)
    total = sum(r["series"] for r in res.values())
    overall = sum(r["test_smape"] * r["series"] for r in res.values()) / total
    summary = {"what": f"M4-scale mixed run on 1 B200: one model per frequency, {epochs} epochs + validate each, "
                       "then evaluate on the test block; synthetic M4-shaped data (reference generator)",
               "total_series": total, "wall_s": time.perf_counter() - t_all,
               "series_epochs_per_s": total * epochs / (time.perf_counter() - t_all),
               "weighted_test_smape": overall, "per_frequency": res}
    Path(out).write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: v for k, v in summary.items() if k != "per_frequency"}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["sweep", "mixed"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--epochs", type=int, default=15)
    a = ap.parse_args()
    sys.path.insert(0, str(ROOT))
    if a.mode == "sweep":
        sweep(a.out or "gpurun_out/r01_sweep.json")
    else:
        mixed(a.out or "gpurun_out/r01_m4_mixed.json", a.epochs)
