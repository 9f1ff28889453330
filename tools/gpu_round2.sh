#!/bin/bash
# GPU iteration: the full -m gpu suite (or the tests named in $TESTS), then a cfg1 bench line.
set -o pipefail
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-1500} python -m pytest ${TESTS:-tests} -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt
if [ -z "$NO_BENCH" ]; then
  timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err || tail -20 gpurun_out/bench.err
  python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "e2e", round((d.get("e2e") or {}).get("value", 0)),
      "cpu", round((d.get("cpu_baseline") or {}).get("value", 0)), "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"], 4))
for k, v in d["kernels"].items():
    print(f"  {k:28s} {v['avg_us']:8.2f} us x {v['launches_per_step']:6.0f}  share {v['share']:.3f}  frac {v['frac']:.4f} {v['unit']}")
print("fp64", d.get("fp64_engine"), "clocks", d.get("clocks"))
PY
fi
