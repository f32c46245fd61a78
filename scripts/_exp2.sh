python -m pytest tests -m gpu -q 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 2 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['model_time'])"; done
