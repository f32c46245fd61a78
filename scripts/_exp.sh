nvidia-smi --query-gpu=memory.total --format=csv
timeout 900 python bench.py --target llama3-70b --requests 128 --steps 2 --warmup 3 > gpurun_out/b70.log 2>&1; echo rc=$?; tail -3 gpurun_out/b70.log | cut -c1-1500
