p=29620
for v in draft 0 draft 0; do
  WS_PDL_LATE=$v timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/lp_n1_$v.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/lp_n1_$v.json') if l.startswith('{')][-1]); print('late=$v n1', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/late_pol.out
done
for v in draft 0; do
  p=$((p+1))
  WS_PDL_LATE=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/lp_n4_$v.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/lp_n4_$v.json') if l.startswith('{')][-1]); print('late=$v n4', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/late_pol.out
done
