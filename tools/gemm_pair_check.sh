set -x
EMM_GEMM_PAIR=2 timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -5
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -3
EMM_GEMM_PAIR=0 timeout 200 python tools/gemm_bench.py 2>&1 | tail -8
timeout 200 python tools/gemm_bench.py 2>&1 | tail -8
