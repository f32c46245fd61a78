timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/full_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/full_gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench3.json 2> gpurun_out/r02_bench3.err
