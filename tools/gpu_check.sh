#!/bin/bash
# quick GPU iteration: gpu tests, then bench summaries (args: bench configs, default cfg1)
T="$(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"
for c in ${@:-cfg1}; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/chk_$c.json 2> gpurun_out/chk_$c.err || tail -5 gpurun_out/chk_$c.err
  python - "$c" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/chk_{sys.argv[1]}.json").read().strip().splitlines()[-1])
e = d.get("e2e") or {}
print(sys.argv[1], "value", round(d["value"]), "ms", round(d["ms_per_step"], 3), "e2e", round(e.get("value", 0)),
      "smape", round(d["val_smape"], 4), {k: round(v["ms"] / v["launches"] * 1e3, 1) for k, v in d["kernels"].items()})
PY
done
echo "TESTS: $T"
