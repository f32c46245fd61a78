OFF="2048:8192:1,4096:14336:1"
for rep in 1 2; do
WS_GEMM_CHUNKS="$OFF" timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/ab_off_n1_$rep.json 2>/dev/null
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/ab_on_n1_$rep.json 2>/dev/null
done
WS_GEMM_CHUNKS="$OFF" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/ab_off_n4.json 2>/dev/null
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/ab_on_n4.json 2>/dev/null
