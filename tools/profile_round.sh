# tools/profile_round.sh <tag>: the committed profiles for a round
#  1. the ncu launch list of the bench command (cold-cache, serialised per-launch times)
#  2. one `ncu --set full` capture of the dominant kernel in the bench's own launch configuration
#  3. the same for the quantile kernel (config 5)
tag=${1:-r01}
mkdir -p gpurun_out/prof
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_plain.json 2>&1 || { echo "bench failed"; cat gpurun_out/prof/bench_plain.json; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/${tag}_launches_c3.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:k_mom5 -c 1 -o /tmp/${tag}_c3 \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_c3.log 2>&1
ncu -i /tmp/${tag}_c3.ncu-rep --page raw --csv > gpurun_out/prof/${tag}_c3_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_c3.ncu-rep --page details --csv > gpurun_out/prof/${tag}_c3_details.csv 2>/dev/null
ncu -i /tmp/${tag}_c3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/prof/${tag}_c3_sass.csv.gz
python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:k_quant -c 1 -o /tmp/${tag}_c5 \
    python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_c5.log 2>&1
ncu -i /tmp/${tag}_c5.ncu-rep --page raw --csv > gpurun_out/prof/${tag}_c5_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_c5.ncu-rep --page details --csv > gpurun_out/prof/${tag}_c5_details.csv 2>/dev/null
ls -la gpurun_out/prof
