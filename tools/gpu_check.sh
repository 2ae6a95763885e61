timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in 1 2 5; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>&1; tail -c 1500 gpurun_out/bench_c$c.json; echo; done
