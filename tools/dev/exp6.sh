python -m pytest tests/test_gpu_bernsen.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -k bernsen -x -q -m gpu > gpurun_out/t6.log 2>&1; tail -3 gpurun_out/t6.log
python tools/dev/bern_perf.py
ncu -f --set full --clock-control none --import-source on -k regex:k_bern -c 2 -o /tmp/bern python -c "
import sys; sys.path.insert(0,'tools/dev'); import bern_perf as b; print(b.t(4096,4096,51,51,pages=8,n=1))" > gpurun_out/bern_ncu.log 2>&1
ncu -i /tmp/bern.ncu-rep --page raw --csv > gpurun_out/bern_raw.csv 2>/dev/null
