mkdir -p gpurun_out
timeout 300 python tools/dense_scene_timing.py 2>&1 | tail -5
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rollout.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 300 python tools/variant_sweep.py "SWEEP_COUNT=1" 2>&1 | tail -3
