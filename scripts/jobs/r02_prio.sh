for v in default -1 0 default -1; do
  if [ "$v" = default ]; then env_=""; else env_="WS_DRAFT_PRIO=$v"; fi
  env $env_ timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/prio_$v.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/prio_$v.json') if l.startswith('{')][-1]); print('prio=$v', round(d['value']), round(d['roofline']['ms_per_forward'],2), round(d['roofline']['frac'],3), round(d['roofline']['draft']['ms_per_forward'],3))" >> gpurun_out/prio.out
done
