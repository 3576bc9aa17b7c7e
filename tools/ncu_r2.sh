# Round-2 ncu evidence: launch list of one cfg3 step + --set full of the hot kernels. bash tools/ncu_r2.sh
set -u
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/r2_launches.csv python tools/ncu_step.py cfg3 > gpurun_out/r2_launches.log 2>&1
echo launches rc=$?
for k in bsattn_dkdv_pp bsattn_dq_pp bsattn_fwd_tc bsattn_prep "gemm_sm100_kernel<3, 2, 512" "gemm_sm100_kernel<3, 4, 512" "gemm_sm100_kernel<4, 3" "gemm_sm100_kernel<4, 5" "gemm_sm100_kernel<0, 0" "gemm_sm100_kernel<0, 6" ln_fwd_warp rowproj_mma2 colgrad_group attn_pattern; do
  tag=$(echo "$k" | tr -c 'a-zA-Z0-9' '_' | cut -c1-40)
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:${k}" --launch-skip 2 -c 1 -f \
    -o gpurun_out/r2_full_${tag} python tools/ncu_step.py cfg3 > gpurun_out/r2_full_${tag}.log 2>&1
  echo "$k rc=$?"
done
