python tools/dev/latency.py --quantile > gpurun_out/latq.txt 2>&1
for e in 0 1 2 3 4 7; do echo "EXP $e"; ABIN_EXP_FIX=$e python tools/dev/latency.py; done > gpurun_out/lat2.txt 2>&1
ABIN_EXP_FIX=2 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launch_c1_pdl.csv python bench.py --config 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
