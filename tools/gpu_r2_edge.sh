mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_scale.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 900 python tools/step_variants.py edge= noidx=-DDG_EXP_NOEDGEIDX 2>&1 | tail -12
timeout 600 python tools/tick_timers.py 256 64 7:2 2>&1 | grep -v nvcc | tail -12
