#!/usr/bin/env python3
"""Summarise ncu captures for profiles/ (run here, on the CPU box, over gpurun_out/ files).

    python tools/ncu_summary.py full  <rep.ncu-rep> [...]   # --set full capture: SOL, DRAM bytes, stalls
    python tools/ncu_summary.py launches <launches.csv>       # per-kernel launch list: count, mean, share
    python tools/ncu_summary.py traffic <out.json> <config> <rep.ncu-rep> [...]
        # per-kernel DRAM bytes per launch (read + write) for bench.py's roofline.traffic
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"# {path}"]
    for v in rows[2:]:
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        out.append(f"## {d.get('Kernel Name', '?')[:110]}  (ID {d.get('ID')})")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:70s} {d[k]:>16s} {u.get(k, '')}")
        st = []
        for h, x in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(x.replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(a for a, _ in st) or 1.0
        st.sort(reverse=True)
        out.append("  stall samples: " + ", ".join(f"{n} {a / tot * 100:.1f}%" for a, n in st[:8]))
    print("\n".join(out))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    unit = ""
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                unit = d["Metric Unit"]
                agg.setdefault(d["Kernel Name"].split("(")[0][:80], []).append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values()) or 1.0
    print(f"# {path}: per-kernel launch list (cold-cache, serialised; compare shares)")
    print(f"{'kernel':80s} {'launches':>8s} {'mean_' + unit:>12s} {'share':>7s}")
    for k, v in agg.items():
        print(f"{k:80s} {len(v):8d} {sum(v) / len(v):12.1f} {sum(v) / tot * 100:6.1f}%")


def traffic(out, config, paths):
    import json
    res = {}
    for path in paths:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for v in rows[2:]:
            d, u = dict(zip(hdr, v)), dict(zip(hdr, units))
            name = d["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1].split()[-1]
            b = sum(float(d[k].replace(",", "")) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            res.setdefault(name, []).append(b)
    doc = {"config": config, "source": [str(p) for p in paths],
           "what": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full",
           "kernels": {k: sum(v) / len(v) for k, v in res.items()}}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc))


if __name__ == "__main__":
    mode, *paths = sys.argv[1:]
    if mode == "traffic":
        traffic(paths[0], paths[1], paths[2:])
    else:
        for p in paths:
            (full if mode == "full" else launches)(p)
