nvidia-smi --query-gpu=index,name,memory.used --format=csv > gpurun_out/tp22_smi.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --target llama3-70b --requests 128 --tp 2 --steps 2 --warmup 1 > gpurun_out/tp2x2_128.json 2> gpurun_out/tp2x2_128.err
timeout 1200 python bench.py --target llama3-70b --requests 128 --tp 4 --steps 2 --warmup 1 > gpurun_out/tp4_128.json 2> gpurun_out/tp4_128.err
