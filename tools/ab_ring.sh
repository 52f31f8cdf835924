#!/bin/bash
# A/B of the GEMM operand-ring budget (CAKE_GEMM_RING_KB): at <= ~110 KB two
# GEMM CTAs fit one SM, so a dependent launch's CTAs are resident (prologue,
# weight prefetch) before the predecessor's CTAs exit.
cd "$(dirname "$0")/.."
DEFS="${DEFS:--DCAKE_GEMM_RING_KB=200;-DCAKE_GEMM_RING_KB=108}" \
CMD="T=8192 REPS=3 python tools/profile_step.py; python tools/gemm_ksweep.py 4096 128 2 0" tools/ab_build.sh
