#!/bin/bash
# compute-sanitizer over tools/repro_batch.py (round-2 kernels: fp32 ES blocks, tensor-core dW
# path on the 8,192-window steps; two-tile K2 CTAs, TMA-staged K3 GEMM, opt-in q-strip GEMM)
mkdir -p gpurun_out
out=gpurun_out/r02i_sanitizers.txt
: > $out
run() { echo "compute-sanitizer --tool $1 python tools/repro_batch.py $2 $3 $4" >> $out;
        timeout 1200 compute-sanitizer --tool $1 python tools/repro_batch.py $2 $3 $4 2>&1 | grep -E "SUMMARY|Invalid|Race|Barrier|error" | head -5 >> $out; }
run memcheck quarterly fp32
run racecheck quarterly fp32
run synccheck quarterly fp32
run memcheck monthly fp32
run racecheck monthly fp32
run memcheck yearly fp32
run memcheck monthly fp64
run memcheck quarterly fp32 big
run racecheck quarterly fp32 big
echo "ESRNN_GEMM_WIDE=1 compute-sanitizer --tool memcheck python tools/repro_batch.py quarterly fp32" >> $out
ESRNN_GEMM_WIDE=1 timeout 1200 compute-sanitizer --tool memcheck python tools/repro_batch.py quarterly fp32 2>&1 | grep -E "SUMMARY|Invalid|Race|Barrier|error" | head -5 >> $out
echo "ESRNN_GEMM_WIDE=1 compute-sanitizer --tool racecheck python tools/repro_batch.py quarterly fp32" >> $out
ESRNN_GEMM_WIDE=1 timeout 1200 compute-sanitizer --tool racecheck python tools/repro_batch.py quarterly fp32 2>&1 | grep -E "SUMMARY|Invalid|Race|Barrier|error" | head -5 >> $out
cat $out
