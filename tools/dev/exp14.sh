timeout 900 python -m pytest tests/test_gpu_small.py -x -q -m gpu > gpurun_out/t14.log 2>&1; tail -n 3 gpurun_out/t14.log
for px in 0 524288 16000000; do echo "SMALL_PX $px"; ABIN_SMALL_PX=$px python tools/dev/latency.py; done
python -c "import __graft_entry__ as g; g.smoke()"
