timeout 900 python -m pytest tests/test_gpu_pack.py -x -q -m gpu > gpurun_out/t12.log 2>&1; tail -n 3 gpurun_out/t12.log
python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pack', d['value'], d['ms_per_step'], d['roofline']['frac'])"
ABIN_NO_PACK=1 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopack', d['value'], d['ms_per_step'], d['roofline']['frac'])"
python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pack', d['value'], d['ms_per_step'], d['roofline']['frac'])"
