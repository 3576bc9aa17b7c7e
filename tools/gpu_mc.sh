# dense GEMM engines vs cuBLAS: gemm tests (all engines) + projection-shape probe + clock64 timelines
mkdir -p gpurun_out
[ -n "$SKIP_TESTS" ] || timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/mc_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/mc_pytest.log
[ -n "$SKIP_PROBE" ] || timeout 300 python tools/linear_probe.py 0 > gpurun_out/mc_probe.txt 2>&1; echo probe rc=$?; cat gpurun_out/mc_probe.txt
timeout 300 python tools/dense_trace.py 6144 0 5 > gpurun_out/mc_trace.txt 2>&1; timeout 300 python tools/dense_trace.py 50272 0 5 >> gpurun_out/mc_trace.txt 2>&1; cat gpurun_out/mc_trace.txt
