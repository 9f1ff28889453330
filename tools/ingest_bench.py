#!/usr/bin/env python3
"""§8(f) row 4 timing: M4-scale CSV ingestion into the engine's upload layout vs the
reference's data path.

Generates an M4-shaped train CSV + info CSV (default 100,000 series: 48,000 Monthly,
24,000 Quarterly, 23,000 Yearly and 5,000 short Yearly rows that equalize_lengths drops;
lengths drawn around the M4 per-frequency medians; the reference's parse_frequency knows
only Yearly / Quarterly / Monthly), then per frequency times
  engine     esrnn_ingest_m4_csv (all host threads): parse + info join + filter + stats +
             equalise into the pinned upload block,
  reference  the reference's own parse_m4_train_csv / parse_info_csv / apply_info / filter /
             length_stats / equalize_lengths (oracle/_ref, single-threaded) and, separately,
             its JSON bundle round trip save_prepared + load_prepared (commands.hpp:30-74),
and checks the two datasets are identical.

    python tools/ingest_bench.py [n_series] > gpurun_out/ingest.json
"""
import ctypes as C
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1907_03329_b200 import _native as N  # noqa: E402
from paper_1907_03329_b200.ingest import ingest_m4_csv  # noqa: E402
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile  # noqa: E402

CATS = ["Demographic", "Finance", "Industry", "Macro", "Micro", "Other"]


def write_m4(d: Path, n: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    groups = [("Monthly", 0.48, 216, 108), ("Quarterly", 0.24, 92, 88), ("Yearly", 0.23, 31, 25),
              ("Yearly", 0.05, 18, 12)]  # short Yearly rows: dropped by equalize_lengths
    freqs, lens = [], []
    for name, frac, med, lo in groups:
        k = int(round(n * frac))
        freqs += [name] * k
        lens += list(np.maximum(lo - 10, rng.lognormal(np.log(med), 0.5, size=k).astype(int)))
    freqs, lens = freqs[:n], np.array(lens[:n])
    maxlen = int(lens.max())
    tr, info = d / "train.csv", d / "info.csv"
    with open(tr, "w") as f:
        f.write(",".join(f'"V{i + 1}"' for i in range(maxlen + 1)) + "\n")
        for i in range(n):
            v = np.exp(rng.normal(7.0, 0.8) + np.cumsum(rng.normal(0, 0.03, size=lens[i])))
            f.write(f'"X{i}",' + ",".join(f'"{x:.6g}"' for x in v) + ',""' * (maxlen - lens[i]) + "\n")
    with open(info, "w") as f:
        f.write("M4id,category,Frequency,Horizon,SP,StartingDate\n")
        for i in range(n):
            f.write(f"X{i},{CATS[i % 6]},12,18,{freqs[i]},01-01-00 12:00\n")
    return tr, info, tr.stat().st_size


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    eng = N.product_api()
    ref = N.NativeApi(ROOT / "oracle" / "_ref" / "libesrnn_ref.so")
    ref.lib.esrnn_ref_bundle_roundtrip.argtypes = [C.c_void_p, C.c_int32, C.c_char_p]
    ref.lib.esrnn_ref_bundle_roundtrip.restype = C.c_int64
    with tempfile.TemporaryDirectory() as td:
        d = Path(td)
        t0 = time.perf_counter()
        tr, info, nbytes = write_m4(d, n)
        gen_s = time.perf_counter() - t0
        rows = []
        for freq in (Frequency.Yearly, Frequency.Quarterly, Frequency.Monthly):
            prof = FrequencyProfile.defaults(freq)
            ingest_m4_csv(tr, info, prof, api=eng).close()  # page cache warm
            te = []
            for _ in range(3):
                t0 = time.perf_counter()
                a = ingest_m4_csv(tr, info, prof, api=eng)
                te.append(time.perf_counter() - t0)
                if _ < 2:
                    a.close()
            t0 = time.perf_counter()
            b = ingest_m4_csv(tr, info, prof, api=ref)
            tr_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            got = ref.lib.esrnn_ref_bundle_roundtrip(b._h, int(freq), str(d / "bundle.json").encode())
            rt_s = time.perf_counter() - t0
            same = (a.n == b.n and np.array_equal(a.values, b.values) and np.array_equal(a.categories, b.categories)
                    and a.ids == b.ids)
            rows.append({"frequency": freq.name, "kept": a.n, "length": a.length, "raw_count": a.raw_count,
                         "engine_s": min(te), "reference_parse_equalize_s": tr_s,
                         "reference_bundle_roundtrip_s": rt_s, "bundle_series": got,
                         "speedup_vs_reference_parse": tr_s / min(te),
                         "speedup_vs_reference_prepare_plus_load": (tr_s + rt_s) / min(te), "identical": bool(same)})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            a.close()
            b.close()
    print(json.dumps({"what": "M4-shaped CSV ingestion", "series": n, "csv_bytes": nbytes, "host_threads": os.cpu_count(),
                      "generate_s": gen_s, "rows": rows}))


if __name__ == "__main__":
    main()
