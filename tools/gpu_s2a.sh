# round-2 session-2 baseline: gpu tests, bench, dense projection probe, kineto graph breakdown
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s2a_pytest.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/s2a_pytest.log | tail -30
timeout 600 python bench.py > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/s2a_bench.json')); print({k:d.get(k) for k in ('value','speedup_vs_dense_torch','dense_torch_ms','dense_same_kernels_ms')}, d['e2e']['value'])"
tail -3 gpurun_out/s2a_bench.err
timeout 300 python tools/linear_probe.py 0 5 > gpurun_out/s2a_linear.txt 2>&1; echo probe rc=$?; cat gpurun_out/s2a_linear.txt | tail -8
timeout 300 python tools/kineto_step.py --graph > gpurun_out/s2a_kineto.txt 2>&1; echo kineto rc=$?; head -40 gpurun_out/s2a_kineto.txt
