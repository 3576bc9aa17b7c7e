set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1; echo build rc=$?; tail -2 gpurun_out/r2c_build.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2c_pytest.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/r2c_pytest.log | tail -30
python tools/parity_report.py > gpurun_out/r2c_parity.txt 2>&1; echo parity rc=$?
grep -A40 "batched item 0" gpurun_out/r2c_parity.txt | head -40
timeout 600 python bench_ops.py --ops attn --reps 10 > gpurun_out/r2c_ops.jsonl 2> gpurun_out/r2c_ops.err; echo ops rc=$?
python - <<PY
import json
for l in open("gpurun_out/r2c_ops.jsonl"):
    d=json.loads(l)
    print(d.get("op"),d.get("phase"),d.get("sparsity"),d.get("attn_blk"),d.get("ms"),d.get("tflops") or d.get("achieved"),d.get("speedup_vs_same_kernel_dense"),d.get("mma_tiles_fwd_dq"),d.get("mma_tiles_dkdv"))
PY
tail -3 gpurun_out/r2c_ops.err
