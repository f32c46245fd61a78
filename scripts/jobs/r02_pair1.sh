timeout 900 bash -c 'WS_GEMM_PAIR1=1 python -m pytest tests/test_gpu_gemm_chunks.py tests/test_gpu_gemm.py -x -q -m gpu' > gpurun_out/pair1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pair1_tests.log
probe() { timeout 300 python scripts/gemm_probe.py 7 48,116,192 8,16,32 2>&1 | grep -o '"rows": [0-9]*\|"ms_median": [0-9.]*' | paste - - | tr '\n' ' '; echo; }
for rep in 1 2; do for v in 1 0; do echo "pair1=$v: $(WS_GEMM_PAIR1=$v probe)" >> gpurun_out/pair1.out; done; done
