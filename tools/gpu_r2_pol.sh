mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_policy.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_pol.log; tail -3 gpurun_out/pytest_pol.log
timeout 300 python tools/policy_time.py 2>&1 | tail -4
bash tools/gpu_ncu_traffic.sh
