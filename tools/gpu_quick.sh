# Quick GPU check: build, selected gpu tests, bench line. usage: bash tools/gpu_quick.sh TAG [pytest -k expr]
set -u
tag=${1:-q}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1; echo build rc=$?
if [ -n "${2:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$2" > gpurun_out/${tag}_pytest.log 2>&1; echo pytest rc=$?
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo pytest rc=$?
fi
tail -15 gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench rc=$?
cat gpurun_out/${tag}_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ('value','e2e','speedup_vs_dense_torch','dense_torch_ms','gpu_launches_per_step')})"
tail -3 gpurun_out/${tag}_bench.err
