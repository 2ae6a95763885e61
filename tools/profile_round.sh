# tools/profile_round.sh <tag>: the committed profiles for a round
#  1. the ncu launch list of the bench command (cold-cache, serialised per-launch times)
#  2. one `ncu --set full` capture of the dominant kernel in the bench's own launch configuration
#  3. the same for the quantile kernel (config 5) and the two Bernsen kernels (config-5 page, 51 x 51)
#  4. the bench lines (configs 3, 2, 5, 5b, 1) as JSON
tag=${1:-r02}
mkdir -p gpurun_out/prof
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_plain.json 2>&1 || { echo "bench failed"; cat gpurun_out/prof/bench_plain.json; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/${tag}_launches_c3.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:k_mom5 -c 1 -o /tmp/${tag}_c3 \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_c3.log 2>&1
ncu -i /tmp/${tag}_c3.ncu-rep --page raw --csv > gpurun_out/prof/${tag}_c3_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_c3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/prof/${tag}_c3_sass.csv.gz
ncu -f --set full --clock-control none --import-source on -k regex:k_quant -c 1 -o /tmp/${tag}_c5 \
    python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_c5.log 2>&1
ncu -i /tmp/${tag}_c5.ncu-rep --page raw --csv > gpurun_out/prof/${tag}_c5_raw.csv 2>/dev/null
for k in h v; do
  ncu -f --set full --clock-control none -k regex:k_bern_$k -c 1 -o /tmp/${tag}_b$k \
      python -c "import sys; sys.path.insert(0, 'tools/dev'); import bern_perf as b; print(b.t(4096, 4096, 51, 51, n=1))" \
      > gpurun_out/prof/ncu_b$k.log 2>&1
  ncu -i /tmp/${tag}_b$k.ncu-rep --page raw --csv > gpurun_out/prof/${tag}_b${k}_raw.csv 2>/dev/null
done
for c in 3 2 5 5b 1; do
  python bench.py --config $c --warmup 3 $( [ $c = 3 ] || echo --no-e2e ) > gpurun_out/prof/${tag}_bench_c$c.log 2>&1
  tail -n 1 gpurun_out/prof/${tag}_bench_c$c.log > gpurun_out/prof/${tag}_bench_line_c$c.json
done
ls -la gpurun_out/prof
