# A/B of an alternative build of the library (LX_LIB) on the cfg3 bench line. usage: bash tools/gpu_lib_ab.sh TAG LIB [pytest -k expr]
set -u
tag=$1; alt=$2; mkdir -p gpurun_out
if [ -n "${3:-}" ]; then
  LX_LIB=$alt timeout 900 python -m pytest tests -m gpu -x -q -k "$3" > gpurun_out/${tag}_pytest.log 2>&1; echo pytest rc=$?
  tail -1 gpurun_out/${tag}_pytest.log
fi
for i in 1 2 3; do
for v in paper_2510_15964_b200/libsparseft_b200.so "$alt"; do
  LX_LIB=$v timeout 600 python bench.py --skip-cpu --skip-cfg1 --skip-dense > gpurun_out/${tag}_b.json 2> gpurun_out/${tag}_b.err
  echo "$(basename $v) run$i: $(python -c "import json; d=json.load(open('gpurun_out/${tag}_b.json')); print(d['value'], d['e2e']['value'])")"
done; done
