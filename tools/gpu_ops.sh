set -u
mkdir -p gpurun_out
timeout 900 python bench_ops.py --reps 10 > gpurun_out/ops.jsonl 2> gpurun_out/ops.err; echo ops rc=$?
python - <<PY
import json
for l in open("gpurun_out/ops.jsonl"):
    d=json.loads(l)
    print({k: d[k] for k in d if k not in ("config",)})
PY
tail -3 gpurun_out/ops.err
