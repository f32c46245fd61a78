for v in 0 120 96 0 120; do
  if [ "$v" = 0 ]; then e=""; else e="WS_TARGET_CTAS=$v"; fi
  env $e timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/tc_$v.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/tc_$v.json') if l.startswith('{')][-1]); print('target_ctas=$v', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/tctas.out
done
