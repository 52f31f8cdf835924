#!/bin/bash
# One profiling pass on the GPU box: launch list of a compute-only 8K step and
# full ncu captures of the top kernels at chunk 12 (prefix 6K) of the tier build.
set -x
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r01}
mkdir -p $OUT
export T=8192 REPS=1
python tools/profile_step.py > $OUT/${TAG}_step_noprof.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launch_summary.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launch_summary.txt
export REPS=0
for k in attn_tc_kernel gemm2_tc_kernel gemm_tc_kernel rmsnorm_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-400} -c 2 -o $OUT/${TAG}_$k -f python tools/profile_step.py > $OUT/${TAG}_$k.log 2>&1
done
