#!/bin/bash
# one GPU iteration: phase clocks (eager + graphs), gpu tests, bench summary
python tools/phase_clocks.py 2>&1 | tail -6
GRAPHS=1 python tools/phase_clocks.py 2>&1 | tail -1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_iter.json").read().strip().splitlines()[-1])
print("value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"]),
      {k: round(v["ms"] / v["launches"] * 1e3, 1) for k, v in d["kernels"].items()})
PY
