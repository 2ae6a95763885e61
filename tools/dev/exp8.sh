python -m pytest tests/test_gpu_bernsen.py -x -q -m gpu > gpurun_out/t8.log 2>&1; tail -n 1 gpurun_out/t8.log
python tools/dev/bern_perf.py
