ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bern_launch.csv python tools/dev/bern_perf.py > /dev/null 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:k_bern -c 2 -o /tmp/bern python -c "
import sys; sys.path.insert(0,'tools/dev'); import bern_perf as b; print(b.t(4096,4096,51,51,pages=8,n=1))" > gpurun_out/bern_ncu.log 2>&1
ncu -i /tmp/bern.ncu-rep --page raw --csv > gpurun_out/bern_raw.csv 2>/dev/null
ncu -i /tmp/bern.ncu-rep --page details --csv > gpurun_out/bern_details.csv 2>/dev/null
