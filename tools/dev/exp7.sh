python -m pytest tests/test_gpu_bernsen.py -x -q -m gpu > gpurun_out/t7.log 2>&1; tail -1 gpurun_out/t7.log
ABIN_BERN_GSB=1 python -m pytest tests/test_gpu_bernsen.py -x -q -m gpu > gpurun_out/t7b.log 2>&1; tail -1 gpurun_out/t7b.log
python tools/dev/bern_perf.py
echo GSB; ABIN_BERN_GSB=1 python tools/dev/bern_perf.py
ncu -f --set full --clock-control none --import-source on -k regex:k_bern_h -c 1 -o /tmp/bernh python -c "
import sys; sys.path.insert(0,'tools/dev'); import bern_perf as b; print(b.t(4096,4096,51,51,pages=8,n=1))" > gpurun_out/bern_ncu.log 2>&1
ncu -i /tmp/bernh.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/bernh_sass.csv.gz
