timeout 2000 python -m pytest tests -x -q -m gpu > gpurun_out/st2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/st2_tests.log
for rep in 1 2; do
for v in 1 0; do
  echo "stage=$v prefill: $(WS_EPI_STAGE=$v timeout 300 python scripts/prefill_probe.py 64 3 2>&1 | grep -o '"ms_median": [0-9.]*' | tr '\n' ' ') probe: $(WS_EPI_STAGE=$v timeout 300 python scripts/gemm_probe.py 5 48,496 107 2>&1 | grep -o '"ms_median": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/stage2.out
  WS_EPI_STAGE=$v timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/st2_${v}_$rep.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/st2_${v}_$rep.json') if l.startswith('{')][-1]); print('stage=$v bench', round(d['value']), 'prefill', round(d['roofline']['prefill']['ms_per_forward'],1), 'verify', round(d['roofline']['ms_per_forward'],2), 'draft', round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/stage2.out
done
done
