#!/bin/bash
# Round-2 GPU evidence pass (under gpurun): gpu tests, smoke, bench lines (cfg1 with the
# CPU baseline, the reference arm, cfg2, cfg3), the cfg1 launch list, and ncu --set full
# captures of every step kernel at cfg1 plus k_tile / k_forecast_scan at cfg3.
# Usage: bash tools/gpu_r02.sh TAG [quick]
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
lscpu > gpurun_out/${TAG}_lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=20 > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest gpu rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/${TAG}_smoke.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg1.json 2> gpurun_out/${TAG}_bench_cfg1.err; echo "bench cfg1 rc=$?"
[ "$2" = "quick" ] && exit 0
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "bench ref rc=$?"
for c in cfg2 cfg3; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
for k in k_tile k_grad_finish k_adam k_forecast_scan; do
  skip=200; [ $k = k_forecast_scan ] && skip=2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/${TAG}_cfg1_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/${TAG}_ncu_cfg1_$k.log 2>&1; echo "ncu cfg1 $k rc=$?"
done
for k in k_tile k_grad_finish k_adam k_forecast_scan; do
  skip=20; [ $k = k_forecast_scan ] && skip=1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/${TAG}_cfg3_$k python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
    > gpurun_out/${TAG}_ncu_cfg3_$k.log 2>&1; echo "ncu cfg3 $k rc=$?"
done
# the tensor-core weight-gradient blocks at the sweep end (B = 48,000)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_grad_finish -s 3 -c 1 \
  -o gpurun_out/${TAG}_sweep48000_k_grad_finish python bench.py --config sweep48000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu_sweep.log 2>&1; echo "ncu sweep48000 k_grad_finish rc=$?"
python tools/ncu_summary.py full gpurun_out/${TAG}_sweep48000_*.ncu-rep > gpurun_out/${TAG}_ncu_full_sweep48000.txt 2>&1
timeout 600 python bench.py --config sweep48000 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_sweep48000.json 2>/dev/null
# summaries on the box (the reps exceed gpurun's 64 MiB return limit); keep only k_tile's rep
python tools/ncu_summary.py full gpurun_out/${TAG}_cfg1_*.ncu-rep > gpurun_out/${TAG}_ncu_full_cfg1.txt 2>&1
python tools/ncu_summary.py full gpurun_out/${TAG}_cfg3_*.ncu-rep > gpurun_out/${TAG}_ncu_full_cfg3.txt 2>&1
python tools/ncu_summary.py traffic gpurun_out/${TAG}_ncu_traffic_cfg1.json cfg1 gpurun_out/${TAG}_cfg1_*.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py traffic gpurun_out/${TAG}_ncu_traffic_cfg3.json cfg3 gpurun_out/${TAG}_cfg3_*.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt 2>&1
rm -f gpurun_out/${TAG}_cfg1_k_grad_finish.ncu-rep gpurun_out/${TAG}_cfg1_k_adam.ncu-rep gpurun_out/${TAG}_cfg1_k_forecast_scan.ncu-rep \
      gpurun_out/${TAG}_cfg3_*.ncu-rep gpurun_out/${TAG}_sweep48000_*.ncu-rep gpurun_out/${TAG}_launches.csv
du -sh gpurun_out
for f in gpurun_out/${TAG}_bench_*.json; do echo "== $f"; tail -1 $f | cut -c1-400; done
