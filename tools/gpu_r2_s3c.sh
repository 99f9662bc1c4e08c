set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_worldgen.py tests/test_gpu_acceptance.py -x -q -p no:cacheprovider -s 2>&1 | tail -30 > gpurun_out/pytest_worldgen.log
tail -8 gpurun_out/pytest_worldgen.log
