p=29650
for v in draft 0 draft 0; do
p=$((p+1))
WS_PDL_LATE=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/l2_$v.json 2>/dev/null
python -c "import json; d=json.loads([l for l in open('gpurun_out/l2_$v.json') if l.startswith('{')][-1]); print('late=$v n2', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/late2.out
done
