python -m pytest tests/test_gpu_parity.py tests/test_gpu_quant5.py tests/test_gpu_v5.py -x -q -m gpu > gpurun_out/t3.log 2>&1; tail -2 gpurun_out/t3.log
for a in "--config 5 --steps 5" "--config 5 --steps 200" "--config 1 --steps 20" "--config 1 --steps 1000" "--config 5b --steps 20"; do
  python bench.py $a --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
done
python tools/dev/latency.py > gpurun_out/lat3.txt 2>&1; cat gpurun_out/lat3.txt
