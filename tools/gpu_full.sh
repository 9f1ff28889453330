#!/bin/bash
# Full GPU evidence pass: gpu tests, smoke, bench (cfg1 with CPU baseline, cfg2, cfg3),
# reference arm, ncu launch list and one ncu --set full capture of the step kernel.
# Usage (under gpurun): bash tools/gpu_full.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest gpu rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/${TAG}_smoke.txt
timeout 600 python bench.py > gpurun_out/${TAG}_bench_cfg1.json 2> gpurun_out/${TAG}_bench_cfg1.err; echo "bench cfg1 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "bench ref rc=$?"
for c in cfg2 cfg3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 200 -c 2 \
  -o gpurun_out/${TAG}_tile python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu_tile.log 2>&1; echo "ncu tile rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_grad_finish -s 200 -c 2 \
  -o gpurun_out/${TAG}_finish python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu_finish.log 2>&1; echo "ncu finish rc=$?"
for f in gpurun_out/${TAG}_bench_*.json; do echo "== $f"; tail -1 $f | cut -c1-600; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_adam -s 200 -c 2 \
  -o gpurun_out/${TAG}_adam python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu_adam.log 2>&1; echo "ncu adam rc=$?"
