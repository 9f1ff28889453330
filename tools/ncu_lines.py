#!/usr/bin/env python3
"""Warp-stall samples per CUDA source line of one ncu capture (needs -lineinfo and
--import-source on):  python tools/ncu_lines.py <rep.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, idx, agg = "?", None, {}
line_key = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        idx = r.index("Warp Stall Sampling (All Samples)")
        continue
    if idx is None or len(r) <= idx:
        continue
    if r[0] not in ("", "-"):  # a CUDA source line: its samples are the sum of its SASS rows
        line_key = (cur, int(r[0]), r[1].strip()[:100])
        try:
            agg[line_key] = agg.get(line_key, 0) + int(r[idx])
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print(f"{rep}: {tot} warp-stall samples")
for (f, ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v:7d} {100 * v / tot:5.1f}%  {f}:{ln}  {src}")
