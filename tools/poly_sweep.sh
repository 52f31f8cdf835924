#!/bin/bash
# Rebuild the CUDA layer with each FA_POLY (pairs of 8 on the FMA pipe) and time
# the 32K attention block period and the bidirectional TTFT. Run on the GPU box.
set -e
cd "$(dirname "$0")/.."
for P in ${POLYS:-2 3 4}; do
  touch paper_2410_03065_b200/csrc/cuda/cake_cuda.cu
  make -s cuda NVCC="nvcc -DFA_POLY=$P" > /dev/null 2>&1
  echo "FA_POLY=$P"
  T=32768 python tools/attn_trace.py 2>&1 | awk '/^0 +[0-9]+ \|/ {n++; t[n]=$NF} END {printf "  block period %.0f cycles (blocks 20..60)\n", (t[61]-t[21])/40}'
  T=32768 REPS=2 MODE=cake python tools/profile_step.py 2>&1 | tail -1 | sed 's/^/  /'
done
