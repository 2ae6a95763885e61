# ncu launch list of the bench (config 3) + full capture of the moments kernel and the quantile kernel
ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
bash tools/ncu_capture.sh c3 python tools/prof_case.py 3 2 8
NCU_KERNEL=k_quantile bash tools/ncu_capture.sh c5 python tools/prof_case.py 5 2
