#!/usr/bin/env python3
"""Summarise a bench.py JSON line: python tools/bench_line.py file.json [label]"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k = d.get("kernels", {})
e = d.get("e2e") or {}
print(sys.argv[2] if len(sys.argv) > 2 else "", "value", round(d["value"]), "ms", round(d["ms_per_step"], 3),
      "e2e", round(e.get("value", 0)), {n: round(v["avg_us"], 1) for n, v in k.items()})
