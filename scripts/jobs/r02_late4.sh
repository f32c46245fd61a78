p=29600
for rep in 1 2; do
for v in 1 0; do
p=$((p+1))
WS_PDL_LATE=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/late4_${v}_$rep.json 2>/dev/null
python -c "import json; d=json.loads([l for l in open('gpurun_out/late4_${v}_$rep.json') if l.startswith('{')][-1]); print('late=$v n4', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/late4.out
done
done
