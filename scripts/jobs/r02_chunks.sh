timeout 900 python -m pytest tests/test_gpu_gemm_chunks.py tests/test_gpu_gemm.py -x -q -m gpu > gpurun_out/chunks_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/chunks_tests.log
run() { echo "== $1" >> gpurun_out/chunks.out; WS_GEMM_CHUNKS="$1" timeout 300 python scripts/gemm_probe.py 7 48,119,192,496 32,64,107 2>&1 | grep -o '"model": "[^"]*"\|"rows": [0-9]*\|"ms_median": [0-9.]*' | paste - - - >> gpurun_out/chunks.out; }
run ""
run "2048:8192:2"
run "2048:8192:4"
run "2048:8192:2,2048:2048:2"
run "2048:8192:4,2048:2048:2,4096:14336:2,4096:4096:2"
run ""
