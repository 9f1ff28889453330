#!/bin/bash
# quick GPU iteration: gpu tests, tile phase clocks, e2e host phases, cfg1 bench summary
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/phase_clocks.py 2>&1 | tail -6 | head -3
ESRNN_DEBUG_HOST=1 python tools/e2e_phases.py 2>&1 | tail -4
python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
tail -3 gpurun_out/bench_iter.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_iter.json").read().strip().splitlines()[-1])
e = d.get("e2e") or {}
print("value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "e2e", round(e.get("value", 0)),
      [round(x, 2) for x in e.get("ms_per_step", [])],
      {k: round(v["ms"] / v["launches"] * 1e3, 1) for k, v in d["kernels"].items()})
PY
