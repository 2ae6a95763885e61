python tools/dev/hostcost.py
for c in 1 2 5; do python bench.py --config $c --warmup 3 --no-e2e --no-cpu-baseline | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d['config'].get('window_sweep'))"; done
