WS_GEMM_CHUNKS="8192:14336:2" timeout 1500 python -m pytest tests/test_gpu_tp.py -x -q -m gpu > gpurun_out/tpc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tpc_tests.log
p=29680
for v in "8192:14336:2" "" "8192:14336:2" ""; do
p=$((p+1))
WS_GEMM_CHUNKS="$v" timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p bench.py --target llama3-70b --requests 128 --tp 2 --steps 2 --warmup 1 > gpurun_out/tpc_$p.json 2>/dev/null
python -c "import json; d=json.loads([l for l in open('gpurun_out/tpc_$p.json') if l.startswith('{')][-1]); print('[$v]', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['frac'],3))" >> gpurun_out/tpc.out
done
