mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -x -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/pytest_iter.log; tail -2 gpurun_out/pytest_iter.log
timeout 600 python tools/variant_sweep.py "SWEEP_COUNT=1" 2>&1 | tail -3
timeout 600 python tools/tick_timers.py 256 64 7:2 2>&1 | grep -v nvcc | tail -11
