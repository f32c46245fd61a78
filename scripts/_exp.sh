timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q -k "split" 2>&1 | tail -2
timeout 300 python scripts/bench_kernels.py splitk_pair 2>&1 | tail -6
