# DEBUG epilogue ablation (LX_GEMM_SPIN bits: 2 skip global stores, 4 skip TMEM loads after the first chunk)
for sp in 0 2 4 6; do echo "== LX_GEMM_SPIN=$sp"; LX_GEMM_SPIN=$sp timeout 300 python tools/dense_trace.py 6144 5; done > gpurun_out/epi.txt 2>&1
cat gpurun_out/epi.txt
