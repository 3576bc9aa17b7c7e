# GEMM barrier polling A/B: dense projection + lm_head shapes and the MLP GEMMs, LX_GEMM_SPIN=0/1
mkdir -p gpurun_out
for sp in 0 1; do
  echo "== LX_GEMM_SPIN=$sp"
  LX_GEMM_SPIN=$sp timeout 300 python tools/dense_trace.py 6144 0 1 2 3
  LX_GEMM_SPIN=$sp timeout 300 python tools/dense_trace.py 50272 0 1
  LX_GEMM_SPIN=$sp timeout 300 python tools/gemm_trace.py --default
done > gpurun_out/spin.txt 2>&1
cat gpurun_out/spin.txt
