set -u
timeout 300 python -m pytest tests/test_gpu_ops.py -q -x -k bsattn 2>&1 | tail -3
timeout 120 python tools/attn_bench.py 24; timeout 120 python tools/attn_bench.py 0 dense; timeout 120 python tools/attn_bench.py 0 blockdiag
timeout 120 python tools/attn_bwd_trace.py blockdiag
