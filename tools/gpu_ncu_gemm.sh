# ncu --set full summaries of the engine's GEMM kernels in one cfg3 step. bash tools/gpu_ncu_gemm.sh TAG
set -u
tag=${1:-r2g}; mkdir -p gpurun_out
: > gpurun_out/${tag}_ncu_full.txt
for k in "gemm_sm100_kernel<.int.3, .int.2, .int.512" "gemm_sm100_kernel<.int.3, .int.4, .int.512" "gemm_sm100_kernel<.int.4, .int.3" "gemm_sm100_kernel<.int.4, .int.5" "gemm_sm100_kernel<.int.6, .int.0" "gemm_sm100_kernel<.int.6, .int.6" "gemm_sm100_kernel<.int.0, .int.8" pack_rows ce_rescale; do
  t=$(echo "$k" | tr -c 'a-zA-Z0-9' '_' | cut -c1-40)
  n=2; case "$k" in *int.0,*|ce_rescale) n=0;; esac
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "regex:${k}" --launch-skip $n -c 1 -f \
    -o gpurun_out/${tag}_full_${t} python tools/ncu_step.py cfg3 > gpurun_out/${tag}_full_${t}.log 2>&1
  echo "$k rc=$?"
  echo "=== $k (gpurun_out/${tag}_full_${t}.ncu-rep) ===" >> gpurun_out/${tag}_ncu_full.txt
  python tools/ncu_hot.py gpurun_out/${tag}_full_${t}.ncu-rep 12 >> gpurun_out/${tag}_ncu_full.txt 2>&1
done
rm -f gpurun_out/${tag}_full_*.ncu-rep
