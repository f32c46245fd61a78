timeout 900 python -m pytest tests/test_gpu_gemm_chunks.py tests/test_gpu_gemm.py tests/test_gpu_model_parity.py -x -q -m gpu > gpurun_out/chunks2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/chunks2_tests.log
run() { echo "== $1" >> gpurun_out/chunks2.out; WS_GEMM_CHUNKS="$1" timeout 300 python scripts/gemm_probe.py 7 48,119,496 32,64,107 2>&1 | grep -o '"model": "[^"]*"\|"rows": [0-9]*\|"ms_median": [0-9.]*' | paste - - - >> gpurun_out/chunks2.out; }
run "4096:14336:1"
run ""
run "4096:14336:1"
run ""
