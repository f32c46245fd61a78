timeout 1500 python -m pytest tests/test_gpu_model_parity.py tests/test_gpu_model.py tests/test_gpu_gemm.py -x -q -m gpu > gpurun_out/late_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late_tests.log
probe() { timeout 300 python scripts/gemm_probe.py 7 48,116,496 32,107 2>&1 | grep -o '"rows": [0-9]*\|"ms_median": [0-9.]*' | paste - - | tr '\n' ' '; echo; }
for rep in 1 2; do
for v in 1 0; do
  echo "late=$v probe: $(WS_PDL_LATE=$v probe)" >> gpurun_out/late_ab.out
  WS_PDL_LATE=$v timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/late_ab_${v}_$rep.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/late_ab_${v}_$rep.json') if l.startswith('{')][-1]); print('late=$v bench', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3), d['clocks']['sm_mhz'])" >> gpurun_out/late_ab.out
done
done
