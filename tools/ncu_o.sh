for v in 0 8; do
ncu --set full --clock-control none -k regex:gemm -s 6 -c 1 -o gpurun_out/o_v$v -f python tools/gemm_sweep.py $v o > /dev/null 2>&1
done
python tools/gemm_sweep.py 0,8 o,down
