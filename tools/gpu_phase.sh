#!/bin/bash
# k_tile / k_grad_finish per-phase clock64 stamps and step-5 spans (ESRNN_DEBUG_CLOCKS), per frequency.
# Usage: bash tools/gpu_phase.sh TAG [frequencies...]; extra env (e.g. ESRNN_NO_PDL=1) passes through
TAG=${1:-phase}; shift
FREQS=${@:-Quarterly Yearly Monthly}
mkdir -p gpurun_out
for f in $FREQS; do
  GRAPHS=1 timeout 300 python tools/phase_clocks.py $f > gpurun_out/${TAG}_$f.txt 2>&1; echo "$f rc=$?"
  grep "esrnn dbg" gpurun_out/${TAG}_$f.txt | grep -v "timeline\|scan block\|reduce block0 start" | tail -8
done
