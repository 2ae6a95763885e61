# tools/ab.sh cfgs libs...: time bench configs for each variant library
cfgs=$1; shift
for lib in "$@"; do for c in $cfgs; do
ABIN_LIB=$PWD/abvar/$lib.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'cfg', $c, round(d['value'],1), d['unit'], 'frac', round(d['roofline']['frac'],4), 'ms', round(d['ms_per_step'],4))"
done; done
