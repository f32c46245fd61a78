p=29570
for v in 32 16 8 32; do
p=$((p+1))
WS_VERIFY_MIN=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/vmin4_${v}_$p.json 2>/dev/null
done
