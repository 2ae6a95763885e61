timeout 900 python -m pytest tests/test_gpu_small.py -x -q -m gpu > gpurun_out/t15.log 2>&1; tail -n 1 gpurun_out/t15.log
for px in 524288; do ABIN_SMALL_PX=$px python tools/dev/latency.py 2>&1 | head -1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_launch.csv python bench.py --config 1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b1s.log 2>&1
python bench.py --config 1 --warmup 3 --no-e2e --no-cpu-baseline | tail -n 1
