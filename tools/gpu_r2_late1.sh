mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_policy.py tests/test_gpu_rollout.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python tools/policy_time.py 2>&1 | tail -3
for i in 1 2; do timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_l1_$i.json 2> gpurun_out/bench_l1_$i.err; python -c "
import json; d=json.load(open('gpurun_out/bench_l1_$i.json')); print(d['value']/1e6, d['ms_per_step'], d['launch']['ms_incl_submit'], d['roofline']['frac'], d['roofline']['kernel_ms'], 'c4', d['c4_single_gpu']['value']/1e6, 'c5', d['c5_policy_rollout']['value']/1e6, d['clocks'])"; tail -2 gpurun_out/bench_l1_$i.err; done
