# Round-2 GPU check: gpu tests + one bench line. usage: bash tools/gpu_r2.sh TAG [pytest -k expr] [bench args...]
set -u
tag=${1:-q}; kexpr=${2:-}; shift 2 2>/dev/null || shift $#
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ "$kexpr" != "none" ]; then
  if [ -n "$kexpr" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1
  else timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; fi
  echo pytest rc=$?; tail -8 gpurun_out/${tag}_pytest.log
fi
timeout 900 python bench.py --skip-cfg1 "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench rc=$?
python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/${tag}_bench.json").read().strip().splitlines()[-1])
    print({k:d.get(k) for k in ("value","e2e","speedup_vs_dense_torch","dense_torch_ms","dense_same_kernels_ms","gpu_launches_per_step")})
    print(d["config"].get("mlp_block_sparsity"), d["config"].get("attn_block_sparsity"), d.get("clocks"))
    for k in d.get("kernels") or []: print(k)
except Exception as e: print("bench parse failed", e)
PY
tail -5 gpurun_out/${tag}_bench.err
