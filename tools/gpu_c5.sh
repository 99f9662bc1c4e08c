mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_policy.py -x -q -s 2>&1 | grep -E "passed|failed|Error|assert" | head -20
timeout 600 python bench.py --no-cpu --steps 50 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c5.json')); print(json.dumps(d['c5_policy_rollout']))"; tail -3 gpurun_out/bench_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:policy -s 4 -c 2 -o gpurun_out/policy -f python bench.py --steps 16 --warmup 4 --no-cpu --e2e-steps 10 > gpurun_out/ncu_policy.log 2>&1; tail -1 gpurun_out/ncu_policy.log
