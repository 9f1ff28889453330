#!/usr/bin/env python3
"""§8(f) row 1: the general dilated LSTM stack (forward_stack over a sequence) at M4 shapes.

For each frequency profile (M4 defaults: dilations, H) and T in 16..72 at B = 2,048: the
shared-memory-resident inference kernel (k_seq_fwd_fast) vs the per-step global-memory kernel
(k_seq_forward, ESRNN_SEQ_NAIVE=1), device time from CUDA events, output agreement, and the
fraction of the FP32 FFMA peak on the live-gate FLOPs
    sum over layers of 2 * B * T * (in_l + H) * 4H  (+ the head, negligible)
(recurrent products skipped for t < d are counted as the kernel skips them).

    python tools/seqstack_bench.py [--precision fp32] > gpurun_out/seqstack.json
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1907_03329_b200 import _native as N  # noqa: E402
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile, TrainConfig, Trainer  # noqa: E402


def flops(prof, T, B):
    H = prof.hidden_size
    dil = [d for b in prof.dilation_blocks for d in b]
    tot = 0.0
    for l, d in enumerate(dil):
        k = prof.input_window + 6 if l == 0 else H
        tot += 2.0 * B * T * k * 4 * H + 2.0 * B * max(T - d, 0) * H * 4 * H
    return tot + 2.0 * B * H * H + 2.0 * B * H * prof.horizon


def main():
    prec = "fp64" if "--precision" in sys.argv and sys.argv[sys.argv.index("--precision") + 1] == "fp64" else "fp32"
    api = N.product_api()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12 / (2 if prec == "fp64" else 1)
    rows = []
    B = 2048
    for freq in (Frequency.Yearly, Frequency.Quarterly, Frequency.Monthly):
        prof = FrequencyProfile.defaults(freq)
        length = prof.min_length + 2 * prof.horizon
        vals, cats = api.make_synthetic(41, 64, length, prof.seasonality_length, 0.05)
        tr = Trainer((vals, cats), prof, TrainConfig(seed=7, batch_size=64, precision=prec), api=api)
        for T in (16, 32, 72):
            x = np.random.default_rng(T).uniform(0.5, 1.5, size=(T, B, prof.input_window + 6))
            res = {}
            ob = np.random.default_rng(T + 1).normal(size=(B, prof.horizon))
            for mode in ("fast", "naive"):
                if mode == "naive":
                    os.environ["ESRNN_SEQ_NAIVE"] = "1"
                else:
                    os.environ.pop("ESRNN_SEQ_NAIVE", None)
                tr.forward_stack(x)  # warm-up
                ms = []
                for _ in range(5):
                    out = tr.forward_stack(x)
                    ms.append(tr.last_device_ms())
                tr.forward_stack(x, ob)  # warm-up of the adjoint path
                msb = []
                for _ in range(3):
                    tr.forward_stack(x, ob)
                    msb.append(tr.last_device_ms())
                res[mode] = (float(np.median(ms)), out, float(np.median(msb)))
            os.environ.pop("ESRNN_SEQ_NAIVE", None)
            f = flops(prof, T, B)
            fast_ms, naive_ms = res["fast"][0], res["naive"][0]
            diff = float(np.max(np.abs(res["fast"][1] - res["naive"][1])))
            row = {"frequency": freq.name, "T": T, "B": B, "H": prof.hidden_size, "precision": prec,
                   "fast_ms": fast_ms, "naive_ms": naive_ms, "speedup": naive_ms / fast_ms,
                   "gflop": f / 1e9, "fast_tflops": f / fast_ms / 1e9, "frac_ffma_peak": f / fast_ms / 1e9 / peak,
                   "max_abs_diff_fast_vs_naive": diff,
                   "fwd_bwd_fast_ms": res["fast"][2], "fwd_bwd_naive_ms": res["naive"][2],
                   "fwd_bwd_speedup": res["naive"][2] / res["fast"][2],
                   "fwd_bwd_frac_ffma_peak": 3 * f / res["fast"][2] / 1e9 / peak}
            rows.append(row)
            print(json.dumps(row), file=sys.stderr, flush=True)
        tr.close()
    print(json.dumps({"what": "forward_stack B=2048 (inference), device ms (CUDA events)", "peak_tflops": peak,
                      "rows": rows}))


if __name__ == "__main__":
    main()
