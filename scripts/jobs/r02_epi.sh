timeout 2000 python -m pytest tests -x -q -m gpu > gpurun_out/epi_tests.log 2>&1; echo "rc=$?" >> gpurun_out/epi_tests.log
WS_GEMM_ABLATE=8 WS_TIMELINE_8B=1 WS_TIMELINE_M=535 timeout 300 python scripts/gemm_probe.py timeline > gpurun_out/epi_timeline.out 2>&1
WS_GEMM_ABLATE=8 WS_TIMELINE_M=496 timeout 300 python scripts/gemm_probe.py timeline >> gpurun_out/epi_timeline.out 2>&1
timeout 300 python scripts/gemm_probe.py 7 48,116,496 32,107 2>&1 | grep -o '"model": "[^"]*"\|"rows": [0-9]*\|"ms_median": [0-9.]*' | paste - - - > gpurun_out/epi_probe.out
