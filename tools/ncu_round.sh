#!/bin/bash
# One profiling pass on the GPU box (1 GPU): the launch list of a compute-only
# 8B step (per-kernel device time; cold-cache and serialised, so compare
# shares) and full ncu captures of the top kernels, taken inside a 16K
# compute-only tier build (chunks 0..31) at the launch offsets below.
set -x
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r01}
mkdir -p $OUT
export T=8192 REPS=1
python tools/profile_step.py > $OUT/${TAG}_step_noprof.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launch_summary.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launch_summary.txt
export T=16384 REPS=0
# gemm2: 2 launches per layer (QKV, gate/up) -> skip 1280 = chunk 20; gemm_tc: O, down
ncu --set full --clock-control none --import-source on -k regex:gemm2_tc_kernel -s 1280 -c 2 -o $OUT/${TAG}_gemm2 -f python tools/profile_step.py > $OUT/${TAG}_gemm2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1280 -c 2 -o $OUT/${TAG}_gemm_tc -f python tools/profile_step.py > $OUT/${TAG}_gemm_tc.log 2>&1
# attention: chunks 0-15 (prefix < 8K) one-tile kernel, 16-31 two-tile kernel; capture prefix ~6K and ~12K
ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 380 -c 1 -o $OUT/${TAG}_attn1 -f python tools/profile_step.py > $OUT/${TAG}_attn1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fa4_kernel -s 300 -c 1 -o $OUT/${TAG}_attn2 -f python tools/profile_step.py > $OUT/${TAG}_attn2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_permute -s 4 -c 1 -o $OUT/${TAG}_scatter -f python tools/profile_step.py > $OUT/${TAG}_scatter.log 2>&1
