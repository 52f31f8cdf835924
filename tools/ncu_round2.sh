#!/bin/bash
# Round-2 profiling pass on the GPU box (1 GPU): the launch list of a
# compute-only 8K step (per-kernel device time; cold-cache and serialised, so
# compare shares), the launch list of one bidirectional 32K run's first-token
# step, and full ncu captures of the top kernels inside a 16K compute-only
# tier build (chunks 0..31) at the launch offsets below.
set -x
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r02}
mkdir -p $OUT
export T=8192 REPS=1
python tools/profile_step.py > $OUT/${TAG}_step_noprof.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv python tools/profile_step.py > /dev/null 2>&1
python tools/launch_summary.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launch_summary.txt
export T=16384 REPS=0
# the M = 512 projections (gemm2_tc: gate/up N-256; gemm2c_tc: QKV N-192, O / down N-128 in pair clusters):
# 4 launches per layer -> skip 20 chunks x 32 layers x 4 = 2560 for chunk 20, layer 0
ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 2560 -c 4 -o $OUT/${TAG}_gemm2 -f python tools/profile_step.py > $OUT/${TAG}_gemm2.log 2>&1
# attention: chunk 28 (prefix 14K), layer 5
ncu --set full --clock-control none --import-source on -k regex:"attn_(tc|alt)_kernel" -s 901 -c 1 -o $OUT/${TAG}_attn2 -f python tools/profile_step.py > $OUT/${TAG}_attn2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_permute -s 4 -c 1 -o $OUT/${TAG}_scatter -f python tools/profile_step.py > $OUT/${TAG}_scatter.log 2>&1
