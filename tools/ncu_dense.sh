# ncu --set full of lx_linear engine(s) at the QKV projection shape (args: modes)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:gemm_sm100" -c 1 -f -o gpurun_out/ncu_dense_m${1:-5} python tools/dense_one.py ${1:-5} > gpurun_out/ncu_dense.log 2>&1
echo ncu rc=$?; tail -2 gpurun_out/ncu_dense.log
