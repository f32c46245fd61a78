for v in 32 16 8; do
WS_VERIFY_MIN=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2956$v bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/vmin_n4_$v.json 2>/dev/null
done
for v in 32 48 16; do
WS_VERIFY_MIN=$v timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/vmin_n1_$v.json 2>/dev/null
done
