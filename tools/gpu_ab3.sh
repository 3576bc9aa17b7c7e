# A/B/C of env settings on the cfg3 bench line (2 rounds). usage: bash tools/gpu_ab3.sh TAG "ENV_A" "ENV_B" "ENV_C"
set -u
tag=$1; shift; mkdir -p gpurun_out
for i in 1 2; do
for v in "$@"; do
  env $v timeout 600 python bench.py --skip-cpu --skip-cfg1 --skip-dense > gpurun_out/${tag}_b.json 2> gpurun_out/${tag}_b.err
  echo "$v run$i: $(python -c "import json; d=json.load(open('gpurun_out/${tag}_b.json')); print(d['value'], d['e2e']['value'])")"
done; done
