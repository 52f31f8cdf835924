#!/bin/bash
# A/B of compile-time variants of the CUDA layer on the GPU box:
#   DEFS="-DX=0;-DX=1" CMD="python tools/..." tools/ab_build.sh
cd "$(dirname "$0")/.."
IFS=';' read -ra VARIANTS <<< "$DEFS"
for D in "${VARIANTS[@]}"; do
  touch paper_2410_03065_b200/csrc/cuda/cake_cuda.cu
  make -s cuda NVCC="nvcc $D" > /dev/null 2>&1 || { echo "build failed: $D"; continue; }
  echo "== $D"
  bash -c "$CMD" 2>&1 | sed 's/^/  /'
done
