set -x
mkdir -p gpurun_out
for spec in "fc1:gemm_sm100_kernel<3, 2" "fc2:gemm_sm100_kernel<4, 3" "attnfwd:bsattn_fwd_tc_kernel" "dkdv:bsattn_dkdv_tc_kernel" "dq:bsattn_dq_tc_kernel" "colgrad:colgrad_partial_kernel" "lnbwd:ln_bwd_kernel"; do
  name=${spec%%:*}; k=${spec#*:}
  timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:${k}" -s 2 -c 1 -f -o gpurun_out/r01_${name} python tools/profile_step.py > gpurun_out/ncu_${name}.log 2>&1
  tail -2 gpurun_out/ncu_${name}.log
done
ls -la gpurun_out/*.ncu-rep
