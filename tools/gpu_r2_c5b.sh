mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_rollout.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python tools/policy_time.py 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 50 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; python -c "
import json; d=json.load(open('gpurun_out/bench_c5.json')); c=d['c5_policy_rollout']; print(d['value']/1e6, 'c4', d['c4_single_gpu']['value']/1e6, 'c5', c['value']/1e6, c['ms_per_tick'], c['env_ms_per_tick'], c['policy_ms_per_tick'], c['launches_per_tick'], c['policy_roofline']['frac'])"; tail -3 gpurun_out/bench_c5.err
