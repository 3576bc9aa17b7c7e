# One GPU session: gpu tests, smoke, bench, ncu launch list, ncu --set full of the hot kernels.
# usage: bash tools/gpu_round.sh TAG [skip-tests]
set -u
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${tag}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1; echo build rc=$?
if [ "${2:-}" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo pytest rc=$?
  tail -3 gpurun_out/${tag}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo smoke rc=$?
fi
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench rc=$?
cat gpurun_out/${tag}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${tag}_launches.csv python tools/profile_step.py > gpurun_out/${tag}_launches.log 2>&1; echo launches rc=$?
python tools/summarize_launches.py gpurun_out/${tag}_launches.csv 30 > gpurun_out/${tag}_launches.txt 2>&1
head -32 gpurun_out/${tag}_launches.txt
bash tools/ncu_full.sh ${tag} fc1:'gemm_sm100_kernel<(\(int\))?3, (\(int\))?2,' attnfwd:bsattn_fwd_tc_kernel dkdv:bsattn_dkdv_pp_kernel dq:bsattn_dq_pp_kernel colgrad:colgrad_group_kernel lnf:ln_fwd_warp mask:'gemm_sm100_kernel<(\(int\))?0, (\(int\))?6,'
