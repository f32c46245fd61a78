probe() { timeout 300 python scripts/gemm_probe.py 7 48,116,496 32,107 2>&1 | grep -o '"rows": [0-9]*\|"ms_median": [0-9.]*' | paste - - | tr '\n' ' '; echo; }
for rep in 1 2; do
for v in 1 0; do
  touch paper_2602_18931_b200/csrc/kernels/gemm_tc.cu
  NVCC_APPEND_FLAGS="-DWS_EPI_STAGE=$v" python -c "from paper_2602_18931_b200 import build; build.build()" > /dev/null 2>&1
  echo "stage=$v probe: $(probe)" >> gpurun_out/epi_ab.out
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/epi_ab_${v}_$rep.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/epi_ab_${v}_$rep.json') if l.startswith('{')][-1]); print('stage=$v bench', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3), d['clocks']['sm_mhz'])" >> gpurun_out/epi_ab.out
done
done
