ncu -f --set full --cache-control none --clock-control none --import-source on -k regex:k_small -s 10 -c 1 -o /tmp/small python bench.py --config 1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/small_ncu.log 2>&1
ncu -i /tmp/small.ncu-rep --page raw --csv > gpurun_out/small_raw.csv 2>/dev/null
ncu -i /tmp/small.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/small_sass.csv.gz
