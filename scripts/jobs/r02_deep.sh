timeout 1500 python -m pytest tests/test_gpu_model_parity.py tests/test_gpu_model.py -x -q -m gpu > gpurun_out/deep_tests.log 2>&1; echo "rc=$?" >> gpurun_out/deep_tests.log
probe() { timeout 300 python scripts/gemm_probe.py 7 48,116,256,496 16,32,64,107 2>&1 | grep -o '"rows": [0-9]*\|"ms_median": [0-9.]*' | paste - - | tr '\n' ' '; echo; }
for rep in 1 2; do for v in 1 0; do echo "deep=$v: $(WS_ATTN_DEEP=$v probe)" >> gpurun_out/deep.out; done; done
p=29660
for v in 1 0; do
p=$((p+1))
WS_ATTN_DEEP=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/deep_n4_$v.json 2>/dev/null
python -c "import json; d=json.loads([l for l in open('gpurun_out/deep_n4_$v.json') if l.startswith('{')][-1]); print('deep=$v n4', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/deep.out
done
