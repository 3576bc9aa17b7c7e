# A/B of an env toggle on the cfg3 bench line. usage: bash tools/gpu_ab.sh TAG "ENV_A" "ENV_B" [pytest -k expr]
set -u
tag=$1; mkdir -p gpurun_out
if [ -n "${4:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$4" > gpurun_out/${tag}_pytest.log 2>&1; echo pytest rc=$?
  tail -3 gpurun_out/${tag}_pytest.log
fi
for i in 1 2; do
for v in "$2" "$3"; do
  env $v timeout 600 python bench.py --skip-cpu --skip-cfg1 --skip-dense > gpurun_out/${tag}_b.json 2> gpurun_out/${tag}_b.err
  echo "$v run$i: $(python -c "import json; d=json.load(open('gpurun_out/${tag}_b.json')); print(d['value'], d['e2e']['value'])")"
done; done
