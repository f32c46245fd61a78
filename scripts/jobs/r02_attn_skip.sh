timeout 1500 python -m pytest tests/test_gpu_model_parity.py tests/test_gpu_model.py tests/test_gpu_model_seam.py tests/test_gpu_trace.py -x -q -m gpu > gpurun_out/as_tests.log 2>&1; echo "rc=$?" >> gpurun_out/as_tests.log
for rep in 1 2; do
for v in 1 0; do
  touch paper_2602_18931_b200/csrc/kernels/attention.cu
  NVCC_APPEND_FLAGS="-DWS_ATTN_SKIP=$v" python -c "from paper_2602_18931_b200 import build; build.build()" > /dev/null 2>&1
  echo "skip=$v prefill: $(timeout 300 python scripts/prefill_probe.py 64 3 2>&1 | grep -o '"ms_median": [0-9.]*' | tr '\n' ' ') fwd: $(timeout 300 python scripts/forward_probe.py 5 2>&1 | grep -o '"ms_median": [0-9.]*' | tr '\n' ' ')" >> gpurun_out/attn_skip.out
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/as_${v}_$rep.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/as_${v}_$rep.json') if l.startswith('{')][-1]); print('skip=$v bench', round(d['value']), round(d['roofline']['prefill']['ms_per_forward'],1))" >> gpurun_out/attn_skip.out
done
done
