python tools/dev/latency.py > gpurun_out/lat.txt 2>&1
for v in base l2v1 l2v2 l2v4 l2v5; do
  if [ $v = base ]; then L="ABIN_X=1"; else L="ABIN_LIB=paper_1905_13038_b200/ab/libabin_$v.so"; fi
  env $L python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$v.json 2>&1
  env $L ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:k_mom5 -c 1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$v.txt 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launch_c1.csv python bench.py --config 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launch_c5.csv python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launch_c2.csv python bench.py --config 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
