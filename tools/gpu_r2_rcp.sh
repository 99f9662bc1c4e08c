timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sysid.py tests/test_gpu_bench_parity.py tests/test_gpu_engine_behaviour.py -x -q -p no:cacheprovider 2>&1 | tail -3
python tools/step_variants.py rcp= head=--src=tools/ab/head_step.cu 2>&1 | tail -12
timeout 600 python tools/tick_timers.py 256 64 7:2 2>&1 | grep -v nvcc | tail -12
