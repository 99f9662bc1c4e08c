mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_rollout.py tests/test_gpu_bindings.py tests/test_gpu_host_delivery.py tests/test_gpu_engine_behaviour.py -x -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2 3; do timeout 300 python tools/policy_time.py 2>&1 | tail -3; done
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_l9.json 2> gpurun_out/bench_l9.err; python -c "
import json; d=json.load(open('gpurun_out/bench_l9.json')); c=d['c5_policy_rollout']; print(d['value']/1e6, 'e2e', d['e2e']['value']/1e6, 'c4', d['c4_single_gpu']['value']/1e6, 'c5', c['value']/1e6, c['ms_per_tick'], c['policy_ms_per_tick'], c['policy_roofline']['frac'])"; tail -2 gpurun_out/bench_l9.err
