# End-of-session evidence at the current build. bash tools/gpu_final.sh TAG
set -u
tag=${1:-fin}; mkdir -p gpurun_out
bash tools/gpu_full.sh ${tag}
timeout 300 python tools/kineto_step.py --graph > gpurun_out/${tag}_kineto.txt 2>&1; echo kineto rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/${tag}_launches.csv python tools/ncu_step.py cfg3 > gpurun_out/${tag}_launches.log 2>&1
echo launches rc=$?
python tools/summarize_launches.py gpurun_out/${tag}_launches.csv 45 > gpurun_out/${tag}_launches.txt
python tools/traffic_db.py gpurun_out/${tag}_launches.csv cfg3 > gpurun_out/${tag}_ncu_traffic.json
bash tools/gpu_configs.sh ${tag}
timeout 600 python bench_ops.py --reps 10 > gpurun_out/${tag}_ops.jsonl 2> gpurun_out/${tag}_ops.err; echo ops rc=$?
