# full GPU validation at the current build: all gpu tests, smoke, bench line. usage: bash tools/gpu_full.sh TAG
set -u
tag=${1:-full}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo pytest rc=$?
grep -E "passed|failed" gpurun_out/${tag}_pytest.log | tail -2; grep -E "^FAILED|^ERROR" gpurun_out/${tag}_pytest.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/${tag}_bench.json')); print({k:d.get(k) for k in ('value','speedup_vs_dense_torch','dense_torch_ms','dense_same_kernels_ms')}, d['e2e']['value'], d['k1'])"
