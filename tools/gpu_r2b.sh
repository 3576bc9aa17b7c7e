set -u
mkdir -p gpurun_out
python tools/parity_report.py > gpurun_out/r2b_parity.txt 2>&1; echo parity rc=$?
cat gpurun_out/r2b_parity.txt | tail -60
timeout 600 python -m pytest tests/test_gpu_model.py -q > gpurun_out/r2b_pytest.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|Error" gpurun_out/r2b_pytest.log | tail -12
timeout 900 python bench.py --skip-cfg1 --skip-cpu > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench rc=$?
python - <<PY
import json
d=json.loads(open("gpurun_out/r2b_bench.json").read().strip().splitlines()[-1])
print({k:d.get(k) for k in ("value","speedup_vs_dense_torch","dense_torch_ms","dense_same_kernels_ms")}, d["e2e"]["value"])
print(d["config"].get("mlp_block_sparsity"), d["config"].get("attn_block_sparsity"))
for k in d.get("kernels") or []: print(k["kernel"], k["ms_per_launch"], k["frac"], k["total_ms"])
PY
tail -3 gpurun_out/r2b_bench.err
