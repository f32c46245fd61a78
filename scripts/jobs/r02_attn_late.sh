timeout 1500 python -m pytest tests/test_gpu_model.py tests/test_gpu_model_parity.py -x -q -m gpu > gpurun_out/al_tests.log 2>&1; echo "rc=$?" >> gpurun_out/al_tests.log
p=29720
for v in 1 0 1 0; do
p=$((p+1))
WS_PDL_LATE_ATTN=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/al_${v}_$p.json 2>/dev/null
python -c "import json; d=json.loads([l for l in open('gpurun_out/al_${v}_$p.json') if l.startswith('{')][-1]); print('attn_late=$v n4', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/attn_late.out
done
