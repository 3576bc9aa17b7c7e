# kineto graph-step breakdown under two env settings. usage: bash tools/gpu_kab.sh TAG "ENV_A" "ENV_B"
set -u
tag=$1; mkdir -p gpurun_out
for v in "$2" "$3"; do
  env $v timeout 300 python tools/kineto_step.py --graph > gpurun_out/${tag}_k.txt 2>&1
  echo "== $v"; grep -v Warn gpurun_out/${tag}_k.txt | head -28
done
