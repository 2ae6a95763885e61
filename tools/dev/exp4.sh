python -m pytest tests/test_gpu_bernsen.py tests/test_gpu_parity.py -k bernsen -x -q -m gpu > gpurun_out/t4.log 2>&1; tail -5 gpurun_out/t4.log
python tools/dev/bern_perf.py
