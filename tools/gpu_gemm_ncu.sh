set -u
mkdir -p gpurun_out
timeout 300 python tools/gemm_trace.py 0.15 --default > gpurun_out/gt.txt 2>&1; echo trace rc=$?; cat gpurun_out/gt.txt
: > gpurun_out/r2g_ncu_full.txt
for k in "gemm_sm100_kernel<.int.3, .int.2, .int.512" "gemm_sm100_kernel<.int.3, .int.4, .int.512" "gemm_sm100_kernel<.int.4, .int.3" "gemm_sm100_kernel<.int.4, .int.5" "gemm_sm100_kernel<.int.6, .int.0" "gemm_sm100_kernel<.int.6, .int.6"; do
  t=$(echo "$k" | tr -c 'a-zA-Z0-9' '_' | cut -c1-40)
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "regex:${k}" --launch-skip 2 -c 1 -f \
    -o gpurun_out/r2g_full_${t} python tools/ncu_step.py cfg3 > gpurun_out/r2g_full_${t}.log 2>&1
  echo "$k rc=$?"
  echo "=== $k (gpurun_out/r2g_full_${t}.ncu-rep) ===" >> gpurun_out/r2g_ncu_full.txt
  python tools/ncu_hot.py gpurun_out/r2g_full_${t}.ncu-rep 12 >> gpurun_out/r2g_ncu_full.txt 2>&1
done
rm -f gpurun_out/r2g_full_*.ncu-rep
