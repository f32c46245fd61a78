p=29700
for v in 2 1 2 1; do
p=$((p+1))
WS_SHARDS=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/sh4_${v}_$p.json 2>/dev/null
python -c "import json; d=json.loads([l for l in open('gpurun_out/sh4_${v}_$p.json') if l.startswith('{')][-1]); print('shards=$v n4', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/shards.out
done
for v in 2 1; do
WS_SHARDS=$v timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/sh1_$v.json 2>/dev/null
python -c "import json; d=json.loads([l for l in open('gpurun_out/sh1_$v.json') if l.startswith('{')][-1]); print('shards=$v n1', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/shards.out
done
