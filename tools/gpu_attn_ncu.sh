set -u
mkdir -p gpurun_out
python tools/attn_bench.py 24; python tools/attn_bench.py 0 dense; python tools/attn_bench.py 0 blockdiag
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -f -o gpurun_out/r2_attn_mix python tools/attn_bench.py 24 > gpurun_out/r2_attn_ncu.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/r2_attn_mix.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|Compute \(SM\) Throughput|Memory Throughput|DRAM Throughput|Registers Per Thread|Achieved Occupancy|Executed Ipc Active|Issue Slots Busy)"' | cut -d, -f5,13-16 | head -40
