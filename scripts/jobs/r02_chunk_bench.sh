timeout 1500 python -m pytest tests/test_gpu_model.py tests/test_gpu_model_parity.py tests/test_gpu_model_seam.py tests/test_gpu_gemm_chunks.py -x -q -m gpu > gpurun_out/chunkb_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/chunkb_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/chunkb_on.json 2> gpurun_out/chunkb_on.err
WS_GEMM_CHUNKS="2048:8192:1" timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/chunkb_off.json 2> gpurun_out/chunkb_off.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/chunkb_on4.json 2> gpurun_out/chunkb_on4.err
WS_GEMM_CHUNKS="2048:8192:1" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/chunkb_off4.json 2> gpurun_out/chunkb_off4.err
