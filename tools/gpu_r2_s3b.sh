set -x
mkdir -p gpurun_out
timeout 300 python tools/device_loop_profile.py 64 300 > gpurun_out/devloop.txt 2>&1
timeout 600 python tools/tick_timers.py 256 64 8:0 7:2 > gpurun_out/tick_timers.txt 2>&1
timeout 600 python tools/tick_timers.py 256 20 7:2 >> gpurun_out/tick_timers.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_acceptance.py::test_throughput_shape 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
