# Round-2 ncu evidence at the current build: launch list of one cfg3 step (time + DRAM bytes per launch) and
# --set full of the hot kernels, summarised. bash tools/ncu_r2.sh TAG
set -u
tag=${1:-r2}
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/${tag}_launches.csv python tools/ncu_step.py cfg3 > gpurun_out/${tag}_launches.log 2>&1
echo launches rc=$?
python tools/summarize_launches.py gpurun_out/${tag}_launches.csv 45 > gpurun_out/${tag}_launches.txt
python tools/traffic_db.py gpurun_out/${tag}_launches.csv cfg3 > gpurun_out/${tag}_ncu_traffic.json
: > gpurun_out/${tag}_ncu_full.txt
for k in bsattn_dkdv_ds bsattn_dq_ds bsattn_fwd_tc bsattn_prep "gemm_sm100_kernel<.int.3, .int.2, .int.512" "gemm_sm100_kernel<.int.3, .int.4, .int.512" "gemm_sm100_kernel<.int.4, .int.3" "gemm_sm100_kernel<.int.4, .int.5" "gemm_sm100_kernel<.int.6, .int.0" "gemm_sm100_kernel<.int.6, .int.6" attn_pattern ln_fwd_warp rowproj_smem colgrad_group ce_kernel; do
  t=$(echo "$k" | tr -c 'a-zA-Z0-9' '_' | cut -c1-40)
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "regex:${k}" --launch-skip 2 -c 1 -f \
    -o gpurun_out/${tag}_full_${t} python tools/ncu_step.py cfg3 > gpurun_out/${tag}_full_${t}.log 2>&1
  echo "$k rc=$?"
  echo "=== $k (gpurun_out/${tag}_full_${t}.ncu-rep) ===" >> gpurun_out/${tag}_ncu_full.txt
  python tools/ncu_hot.py gpurun_out/${tag}_full_${t}.ncu-rep 12 >> gpurun_out/${tag}_ncu_full.txt 2>&1
done
rm -f gpurun_out/${tag}_full_*.ncu-rep
