ABIN_RING=4 timeout 900 python -m pytest tests/test_gpu_v5.py tests/test_gpu_pack.py tests/test_gpu_rules_v5.py -x -q -m gpu 2>&1 | tail -n 1
for r in 2 4; do echo "RING $r"; ABIN_RING=$r python tools/dev/latency.py 2>&1 | tail -n 5; done
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['ms_per_step'])"
