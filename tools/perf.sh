# quick GPU iteration: parity tests, timing of configs, one ncu capture of config 3 (8 pages)
set -o pipefail
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in 3 4 2 1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg', $c, round(d['value'],1), d['unit'], 'frac', round(d['roofline']['frac'],4), 'ms', round(d['ms_per_step'],4), d['clocks'])"; done
if [ -n "$NCU" ]; then bash tools/ncu_capture.sh c3 python tools/prof_case.py 3 2 8 >/dev/null; python tools/ncu_stalls.py gpurun_out/c3_raw.csv; fi
