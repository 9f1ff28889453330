#!/bin/bash
# Quick GPU iteration (under gpurun): selected gpu tests ($TESTS, default all) + bench lines
# for the configs given as arguments (default cfg1), summarised.
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-1500} python -m pytest ${TESTS:-tests} -m gpu -q -rA ${PYTEST_ARGS} > gpurun_out/quick_pytest.txt 2>&1
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/quick_pytest.txt | tail -15
for c in ${@:-cfg1}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/quick_$c.json 2> gpurun_out/quick_$c.err || tail -5 gpurun_out/quick_$c.err
  python - "$c" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/quick_{sys.argv[1]}.json").read().strip().splitlines()[-1])
e = d.get("e2e") or {}
print(sys.argv[1], "value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "e2e", round(e.get("value", 0)),
      "smape", round(d["val_smape"], 4), "clk", d["clocks"]["sm_mhz"] if d.get("clocks") else None)
for k, v in d["kernels"].items():
    print(f"   {k:26s} {v['avg_us']:8.2f}us x{v['launches_per_step']:7.1f} share {v['share']:.3f} frac {v['frac']:.4f}")
PY
done
