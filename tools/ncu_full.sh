# ncu --set full captures of single launches of the step's kernels: bash tools/ncu_full.sh TAG name:regex ...
set -u
tag=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; k=${spec#*:}
  timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled -k "regex:${k}" -s 2 -c 1 -f \
    -o gpurun_out/${tag}_${name} python tools/profile_step.py > gpurun_out/ncu_${name}.log 2>&1
  echo "$name rc=$?"
done
