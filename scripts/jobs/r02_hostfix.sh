timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/hostfix_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/hostfix_tests.log
WS_PROFILE_HOST=1 timeout 300 python scripts/gemm_probe.py 7 48,192,496 32,107 > gpurun_out/hostfix_probe.out 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench4.json 2> gpurun_out/r02_bench4.err
