python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py -x -q 2>&1 | tail -2
WS_GEMM_ABLATE=8 python scripts/bench_kernels.py timeline 2>&1 | tail -7
python scripts/forward_probe.py 10 2>&1 | tail -2
