timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k 'regex:gemm_sm100_kernel<3, 2' -s 2 -c 1 -f -o gpurun_out/v4_fc1 python tools/profile_step.py > gpurun_out/ncu_fc1.log 2>&1; echo fc1 rc=$?
