# Extra bench lines beside the headline (BASELINE configs[0], [3], [4]): bash tools/gpu_configs.sh TAG
set -u
tag=${1:-r3}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py --skip-cpu --skip-cfg1 "$@" > gpurun_out/${tag}_bench_${name}.json 2> gpurun_out/${tag}_bench_${name}.err; echo "$name rc=$?"; tail -c 300 gpurun_out/${tag}_bench_${name}.json | head -c 300; echo; tail -2 gpurun_out/${tag}_bench_${name}.err; }
[ -n "${SKIP_CFG1:-}" ] || run cfg1 --config cfg1 --steps 20
run cfg4_lora --config cfg4 --steps 5
run cfg4_adapter --config cfg4 --peft adapter --steps 5
run cfg4_bitfit --config cfg4 --peft bitfit --steps 5
[ -n "${SKIP_CFG5:-}" ] || run cfg5_shard --config cfg5 --global-batch 1 --steps 5
