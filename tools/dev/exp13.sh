b() { python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['ms_per_step'], d['roofline']['frac'])"; }
b default
for nb in 17 18 19 20 21 22 24 26 28 32; do ABIN_V4_BANDS=$nb b bands$nb; done
ABIN_DEBUG=1 python -c "print()" 
