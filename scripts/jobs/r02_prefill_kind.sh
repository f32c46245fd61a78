timeout 2000 python -m pytest tests -x -q -m gpu > gpurun_out/pk_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pk_tests.log
for rep in 1 2; do
for v in 0 1; do
  WS_PREFILL_CHUNKS=$v timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/pk_${v}_$rep.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/pk_${v}_$rep.json') if l.startswith('{')][-1]); m=d['model_time']; print('prefill_chunks=$v', round(d['value']), 'prefill ms/fwd', round(d['roofline']['prefill']['ms_per_forward'],1), 'draft prefill', round(m['prefill_draft_ms']), 'verify', round(d['roofline']['ms_per_forward'],2))" >> gpurun_out/pk.out
done
done
