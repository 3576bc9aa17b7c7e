# ncu --set full of the attention kernels at cfg2 shapes: bash tools/ncu_attn.sh TAG [sparsity] [attn_blk]
set -u
tag=$1; sp=${2:-0.0}; ab=${3:-64}
mkdir -p gpurun_out
for spec in fwd:bsattn_fwd_tc dkdv:bsattn_dkdv_tc dq:bsattn_dq_tc; do
  name=${spec%%:*}; k=${spec#*:}
  timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:${k}" -c 1 -f \
    -o gpurun_out/${tag}_attn_${name} python tools/attn_probe.py $sp $ab > gpurun_out/ncu_attn_${name}.log 2>&1
  echo "$name rc=$?"
done
